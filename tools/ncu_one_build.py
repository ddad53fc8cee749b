"""Dev tool: ONE planning launch of a workload (for ncu captures).
Usage: python tools/ncu_one_build.py C4|C2|C1|C3|C5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2105_13336_b200.planner import Planner
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
P = Planner(0)
reqs = bench.workload(name, 0, 1, P)
outs = P.build_plan_groups([j for _, j, _ in reqs], [c for _, _, c in reqs], with_views=False)
print(name, "kernel_ms", outs[0]["stats"]["kernel_ms"], "alg_bytes", sum(o["stats"]["algorithmic_bytes"] for o in outs))
