"""Dev tool: C4 (GPT-2-medium trace) on the device planner vs the restated
oracle (small micro-batch counts) and timing at full size."""
import sys, os, time, json, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import tslo
from paper_2105_13336_b200 import workload as W
from paper_2105_13336_b200.planner import Planner
P = Planner(0)
oracle_max = int(os.environ.get("C4_ORACLE_MAX", "4"))
for M in [int(a) for a in sys.argv[1:]]:
    t = time.time(); jobs = [W.c4_job(M)]; tg = time.time() - t
    A = sum(len(op["inputs"]) + len(op["outputs"]) for op in jobs[0][0]["ops"])
    init = sum(tslo.initial_peaks(jobs).values())
    cfg = {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": init * 7 // 10}
    t = time.time(); p = P.build_plan(jobs, cfg); tp = time.time() - t
    s = p["stats"]
    line = f"M={M} A={A} gen {tg:.1f}s call {tp:.2f}s kernel {s['kernel_ms']:.1f}ms prep {s['prep_ms']:.1f}ms iters {s['loop_iterations']} evals {s['evaluations']} cands {s['candidates']} rescored {s['rescored']} swaps {p['plans_json'].count(chr(34) + 'direction')} final {p['final_merged_peak']} events/s {A / (s['kernel_ms'] / 1e3):.3g}"
    if M <= oracle_max:
        t = time.time(); o = tslo.build_plan(jobs, cfg); to = time.time() - t
        ok = p["plans_json"] == o["plans_json"] and p["reports_json"] == o["reports_json"] and p["merged_peak_history"] == o["merged_peak_history"]
        line += f" | oracle {to:.1f}s match {ok}"
    print(line, flush=True)
    print("   sha", hashlib.sha256(p["plans_json"].encode()).hexdigest()[:16], flush=True)
