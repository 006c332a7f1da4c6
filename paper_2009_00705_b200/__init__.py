"""B200-native geometric p-multigrid Laplace solver (arXiv 2009.00705).

Thin Python binding of the C-ABI library ``libsem_pmg.so`` (include/sem_pmg.h):
argument marshalling only -- every step of the solve runs in the library's CUDA
kernels.  PyTorch provides device memory and the stream.  There is no CPU
fallback: importing this package without the built library raises ImportError.
"""
from ._capi import (  # noqa: F401
    LIB_PATH,
    SemError,
    Solver,
    default_opts,
    host_numbering,
    host_fdm,
    host_partition,
    host_reference,
    host_schwarz,
    nccl_unique_id,
    reference_nodes,
)

__all__ = ["Solver", "SemError", "reference_nodes", "default_opts", "LIB_PATH"]
