"""The partitioned solve over NCCL (one process per GPU, torchrun) matches the
single-domain solve -- runs only where >= 2 GPUs are visible (the round's GPU
boxes have one; the emulated-rank tests of test_gpu_dist.py and the gloo tests
of test_dist_gloo.py cover the same orchestration there)."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)


def test_nccl_two_ranks_match_single_domain():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tools", "nccl_check.py")], capture_output=True, text=True, timeout=600)
    outs = [json.loads(l.split(" ", 1)[1]) for l in r.stdout.splitlines() if l.startswith("NCCLCHECK ")]
    assert r.returncode == 0 and len(outs) == 2, r.stderr[-2000:]
    for o in outs:
        assert o["apply_rel"] <= 1e-13 and o["solve_rel"] <= 1e-10 and abs(o["iters"] - o["iters1"]) <= 1
