"""Build the C-ABI library libsem_pmg.so in-tree for sm_100a (nvcc)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = ["csrc/refelem.cpp", "csrc/topology.cpp", "csrc/partition.cpp", "csrc/kernels.cu", "csrc/apply_dmma.cu", "csrc/apply_warp.cu", "csrc/apply_quad.cu",
       "csrc/capi.cu", "csrc/coarse.cu", "csrc/fnpf.cu", "csrc/stage.cu", "csrc/condense.cu", "csrc/dist.cu", "csrc/fdm.cpp", "csrc/fdm.cu"]
LIB = os.path.join(HERE, "libsem_pmg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-fopenmp,-O3", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(HERE, s) for s in SRC]
    deps = srcs + [os.path.join(HERE, "csrc", h) for h in ("internal.h", "refelem.h", "topology.h", "partition.h", "setup_util.h", "fdm.h")] + \
        [os.path.join(ROOT, "include", "sem_pmg.h")]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps):
        return LIB
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(s):
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        r = subprocess.run([NVCC, "-c", s, "-o", o] + FLAGS, capture_output=True, text=True)
        return s, o, r

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
        for s, o, r in ex.map(compile_one, srcs):
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError("nvcc failed on " + s)
            objs.append(o)
    cmd = [NVCC, "-shared", "-o", LIB] + objs + ["-gencode", "arch=compute_100a,code=sm_100a",
                                                 "-Xcompiler", "-fopenmp", "-lcublas", "-lcusolver", "-lgomp", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
