"""Dev tool: build + replay plans with the device executor; HWM vs predicted peak."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_13336_b200 import configs as CF
from paper_2105_13336_b200.planner import Planner
P = Planner(0)
for name in sys.argv[1:] or ["C1", "C2"]:
    for req in CF.requests(name)[-1:]:
        if name.startswith("C5"):
            from paper_2105_13336_b200 import multigpu as MG
            peaks = MG.initial_peaks(P, [int(name[3:])])
        else:
            peaks = CF.INITIAL_PEAK
        out = P.build_and_execute(req.jobs, req.config(peaks), tick_ns=int(os.environ.get("TICK_NS", 2000)),
                                  iterations=3)
        for jid, r in out["exec"].items():
            print(name, jid, json.dumps({k: r[k] for k in ("predicted_peak", "hwm", "final_footprint", "swap_outs",
                  "swap_ins", "verify_errors", "violations", "iteration_ms", "planned_iteration_ms", "kernels",
                  "total_ms")}), flush=True)
# every job of a multi-job build replayed together (one FIFO channel)
if os.environ.get("MULTI", "1") == "1":
    for name in [n for n in (sys.argv[1:] or ["C3"]) if n in ("C3",) or n.startswith("C5")]:
        req = CF.requests(name)[-1]
        if name.startswith("C5"):
            from paper_2105_13336_b200 import multigpu as MG
            peaks = MG.initial_peaks(P, [int(name[3:])])
            req = CF.requests(name)[7]  # the fullest replan: 8 resident workloads
        else:
            peaks = CF.INITIAL_PEAK
        out = P.build_and_execute_all(req.jobs, req.config(peaks), tick_ns=int(os.environ.get("TICK_NS", 2000)),
                                      iterations=3)
        m = out["merged"]
        print(name, "ALL-JOBS", json.dumps({k: m[k] for k in ("predicted_peak", "hwm", "final_footprint", "swap_outs",
              "swap_ins", "verify_errors", "violations", "iteration_ms", "planned_iteration_ms", "kernels",
              "total_ms")}), flush=True)
