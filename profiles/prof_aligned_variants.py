import os, sys, json
sys.path.insert(0, os.getcwd())
import bench_secondary as bs
import paper_2603_25691_b200 as cp
ctx = cp.Context(0)
for which in ("config2", "config0"):
    o = bs.aligned(which, ctx, 20, 37.0)
    print(which, os.environ.get("CPHIFI_SANDWICH"), json.dumps({k: o[k] for k in ("solve_ms", "mttkrp_ms", "gram_ms", "decoupled_ms", "roofline_frac")}))
