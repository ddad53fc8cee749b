"""Quick parity + timing sweep of the CUDA planner against the oracle (dev tool)."""
import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref, tslo
from paper_2105_13336_b200 import configs as CF
from paper_2105_13336_b200.planner import Planner
lib = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".so") else None
names = [a for a in sys.argv[1:] if not a.endswith(".so")] or ["C1", "C2", "C3", "C5s0"]
P = Planner(0, lib_path=lib)
bad = 0
for ratio in [None, 0.1]:
    for name in names:
        for req in CF.requests(name, ratio=ratio):
            cfg = req.config(ref.initial_peaks(req.jobs))
            o = tslo.build_plan(req.jobs, cfg)
            try:
                p = P.build_plan(req.jobs, cfg)
                p = P.build_plan(req.jobs, cfg)
            except Exception as e:
                print(ratio, req.name, "ERROR", e, flush=True); bad += 1; continue
            ok = p["plans_json"] == o["plans_json"] and p["reports_json"] == o["reports_json"] \
                and p["merged_peak_history"] == o["merged_peak_history"]
            bad += not ok
            pr = P.prepare([req.jobs], cfg)
            kms = pr.run(5)
            pr.close()
            print(f"{ratio} {req.name} A={req.n_accesses} parity={ok} call={p['ms']:.3f}ms kernel={kms:.3f}ms "
                  f"oracle={o['ms']:.2f}ms stats={p['stats']}", flush=True)
print("BAD", bad)
