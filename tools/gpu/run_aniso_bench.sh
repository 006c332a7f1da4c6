timeout 900 python -c "
import sys, json; sys.argv=[\"bench.py\"]
import bench, argparse
import paper_2009_00705_b200 as lib
a=argparse.Namespace(steps=3, warmup=2, tol=1e-8)
print(json.dumps(bench.run_aniso(a, lib, 6537.0)))
" 2>&1 | tail -2
