"""Generates tests/golden/c4.json: C4 (GPT-2-medium trace, workload.gpt2_workload)
parity digests from the restated CPU oracle (oracle/tensile_oracle.cpp).

The reference cannot plan C4 (setup + first evaluation of a
100 k-access chain take minutes, 1 M accesses did not finish in 30 min), so the
oracle -- checked byte-for-byte against the reference on every fixture and on
C4-family instances up to 16 k accesses (this script's `pin` section) -- is
the C4 parity source, labelled as such. Usage:
    python tests/golden/make_c4_golden.py pin              # reference vs oracle, small C4 instances
    python tests/golden/make_c4_golden.py M [M ...]       # oracle digests for micro_batches = M
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref, tslo  # noqa: E402
from paper_2105_13336_b200 import workload as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c4.json")


def digest(r):
    h = lambda t: hashlib.sha256(t.encode()).hexdigest()  # noqa: E731
    return {"plans_sha256": h(r["plans_json"]), "reports_sha256": h(json.dumps(r["reports_json"], sort_keys=True)),
            "history": r["merged_peak_history"], "final_merged_peak": r["final_merged_peak"],
            "swap_events": r["plans_json"].count('"direction"')}


def config_for(jobs):
    # budget: 70 % of the initial merged peak
    init = sum(tslo.initial_peaks(jobs).values())
    return {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": init * 7 // 10}, init


def main():
    data = json.load(open(OUT)) if os.path.exists(OUT) else {"source": "restated CPU oracle", "cases": {}}
    if sys.argv[1:] == ["pin"]:
        for (M, L, H) in [(1, 2, 2), (2, 2, 2), (1, 4, 4), (3, 3, 2), (1, 24, 16)]:
            jobs = [W.c4_job(M, L, H)]
            cfg, _ = config_for(jobs)
            t = time.time()
            rp, _ = ref.build_plan(jobs, cfg)
            tr = time.time() - t
            o = tslo.build_plan(jobs, cfg)
            ok = rp == o["plans_json"]
            print(f"pin M={M} L={L} H={H}: reference {tr:.1f}s, plans equal: {ok}", flush=True)
            data.setdefault("pinned", {})[f"M{M}_L{L}_H{H}"] = {"reference_equal": ok, "reference_s": round(tr, 2)}
        json.dump(data, open(OUT, "w"), indent=1)
        return
    for M in [int(a) for a in sys.argv[1:]]:
        jobs = [W.c4_job(M)]
        A = sum(len(op["inputs"]) + len(op["outputs"]) for op in jobs[0][0]["ops"])
        cfg, init = config_for(jobs)
        t = time.time()
        o = tslo.build_plan(jobs, cfg)
        dt = time.time() - t
        d = digest(o)
        d.update({"micro_batches": M, "accesses": A, "config": cfg, "initial_peak": init, "oracle_s": round(dt, 1)})
        data["cases"][f"M{M}"] = d
        json.dump(data, open(OUT, "w"), indent=1)
        print(f"M={M} A={A} oracle {dt:.1f}s swaps {d['swap_events']} final {d['final_merged_peak']}", flush=True)


if __name__ == "__main__":
    main()
