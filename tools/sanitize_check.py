"""Representative builds for compute-sanitizer (memcheck / racecheck / synccheck):
C1, C2, C3's last arrival, a C5 shard's 15 replans in one launch, an analyze_job
call, a job above one sort tile through the cooperative launch and through the
single-CTA big path, and (full run) the executor's C3 replay, each checked against the reference fixtures or the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_check.py [quick]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from helpers import check_against_golden, config_jobs, golden  # noqa: E402
from paper_2105_13336_b200 import configs as CF, workload as W  # noqa: E402
from paper_2105_13336_b200.planner import Planner  # noqa: E402

P = Planner(0)
quick = "quick" in sys.argv[1:]
cases = {c["name"]: c for c in golden("configs") if c["ratio"] is None}
for name in ("C1", "C2", "C3.3"):
    c = cases[name]
    check_against_golden(P.build_plan(config_jobs(c), c["config"]), c)
    print(name, "ok", flush=True)
rc = next(c for c in golden("configs") if c["name"] == "C2" and c["ratio"] is not None)
check_against_golden(P.build_plan(config_jobs(rc), rc["config"]), rc)
print("C2 ratio", rc["ratio"], "ok", flush=True)
reqs = CF.requests("C5s0")
shard = [c for c in golden("configs") if c["name"].startswith("C5s0.") and c["ratio"] is None]
outs = P.build_plan_groups([r.jobs for r in reqs], [c["config"] for c in shard])
for c, o in zip(shard, outs):
    check_against_golden(o, c)
print("C5s0 (15 groups, one launch) ok", flush=True)
a = golden("analyze")[0]
P.analyze_job(a["graph"], a["latencies"], a["plan"])
print("analyze_job ok", flush=True)
if not quick:
    from oracle import tslo
    g = W.generate_workload("chain", 1, 0, 2200, "big")
    jobs = [(g, W.true_latency_table(g, 3))]
    init = sum(tslo.initial_peaks(jobs).values())
    cfg = {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": init * 7 // 10}
    want = tslo.build_plan(jobs, cfg)["plans_json"]
    for coop in ("1", "0"):
        os.environ["TSL_COOP"] = coop
        assert P.build_plan(jobs, cfg)["plans_json"] == want
        print("chain 2200 (big mode, coop=%s) ok" % coop, flush=True)
    # plan executor (tsl_exec.cu): C3's three jobs replayed together, HWM vs prediction
    c3 = cases["C3.3"]
    out = P.build_and_execute_all(config_jobs(c3), c3["config"], tick_ns=2000, iterations=1)
    assert out["merged"]["hwm"] <= out["merged"]["predicted_peak"], out["merged"]
    assert out["merged"]["verify_errors"] == 0 and out["merged"]["violations"] == 0
    print("executor C3 replay ok", flush=True)
print("SANITIZE_CHECK_DONE", flush=True)
