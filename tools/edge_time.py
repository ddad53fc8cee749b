"""Times the larger edge.json builds on the GPU (best of 5 through build_plan,
host buffers, wall clock of the call) next to the reference's recorded time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from helpers import check_against_golden, edge_jobs, golden  # noqa: E402
from paper_2105_13336_b200.planner import Planner  # noqa: E402

P = Planner(0)
for c in golden("edge"):
    if "error" in c or c["n_accesses"] < 500:
        continue
    jobs = edge_jobs(c)
    best = 1e30
    for _ in range(5):
        t0 = time.perf_counter()
        out = P.build_plan(jobs, c["config"])
        best = min(best, time.perf_counter() - t0)
    check_against_golden(out, c)
    print(f"{c['name']:24s} accesses {c['n_accesses']:6d}  e2e {best * 1e3:8.2f} ms  reference {c['ref_ms']:8.1f} ms"
          f"  {c['ref_ms'] / (best * 1e3):6.1f}x", flush=True)
