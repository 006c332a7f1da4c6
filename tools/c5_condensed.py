import json, sys, os
sys.path.insert(0, os.getcwd())
import bench, paper_2009_00705_b200 as lib
class A: steps=3; warmup=2; tol=1e-8
print(json.dumps(bench.run_config5(A, lib, 6470.8)))
