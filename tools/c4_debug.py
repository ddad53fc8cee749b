"""Dev tool: one C4-family build under several TSL_* settings vs the oracle."""
import os, sys, hashlib, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_13336_b200.planner import Planner
from paper_2105_13336_b200 import workload as W
from oracle import tslo
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1
jobs = [W.c4_job(M)]
init = sum(tslo.initial_peaks(jobs).values())
cfg = {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": init * 7 // 10}
want = tslo.build_plan(jobs, cfg)["plans_json"]
P = Planner(lib_path=os.environ.get("TSL_LIB")) if os.environ.get("TSL_LIB") else Planner(0)
for setting in sys.argv[2:] or ["TSL_COOP=1", "TSL_COOP=0"]:
    env = dict(kv.split("=") for kv in setting.split(","))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    got = P.build_plan(jobs, cfg, with_views=False)
    for k, v in old.items():
        if v is None: os.environ.pop(k)
        else: os.environ[k] = v
    s = got["stats"]
    print(f"M{M} {setting:40s} ok={got['plans_json'] == want} kernel={s['kernel_ms']:.1f}ms rescored={s['rescored']} "
          f"comp={s['comp_rescored']} confmis={s['queryprof'][15]}", flush=True)
