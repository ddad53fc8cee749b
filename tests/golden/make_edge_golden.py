"""Generates tests/golden/edge.json: edge-case plans of the UNMODIFIED reference.

Same driver and record format as make_golden.py (oracle/_ref/libmemsched_ref.so via
oracle/ref.py; save_plans / PeakReport digests, merged-peak history). The cases push
the inputs to their extremes: single-op jobs, zero and constant latencies, budgets of
0 / exactly the initial peak / one below it / effectively unbounded, tensor sizes near
2^40 bytes and latencies near 10^12 ticks (int64 time arithmetic), a setup cost no swap
can hide (recomputation only), bandwidth 1, max_swap_ratio 0 and 1 and entries naming
no job of the build, 40 jobs in one build,
and all 64 C5 workloads planned jointly (the reference's 4 s case). Job specs
are rebuilt by tests/helpers.edge_jobs; configs are stored concretely. Run here:

    make -C oracle ref && python tests/golden/make_edge_golden.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, HERE)

from oracle import ref  # noqa: E402
from helpers import edge_jobs  # noqa: E402
from make_golden import graph_doc, summarize  # noqa: E402

BW, SETUP = 256, 1


def cfg(budget, bw=BW, setup=SETUP, ratios=None):
    c = {"pcie_bandwidth": bw, "transfer_setup": setup, "memory_budget": int(budget)}
    if ratios is not None:
        c["max_swap_ratios"] = ratios
    return c


def gen(fam, batch, jid, depth=0, lat_seed=13, **kw):
    return dict({"gen": [fam, batch, depth, jid, lat_seed]}, **kw)


def cases():
    one = {"graph": graph_doc([("x", 4, "input"), ("y", 8, "interim")],
                              [("op", ["x"], ["y"], "forward_backward", "f")], "one"),
           "latencies": {"op": 7}}
    upd = {"graph": graph_doc([("w", 16, "parameter"), ("w_new", 16, "updated_parameter")],
                              [("U", ["w"], ["w_new"], "optimize", "update")], "upd"),
           "latencies": {"U": 3}}
    c1 = [gen("vgg16", 32, "vgg16")]
    out = []
    for b in (0, 1, 12, 100):
        out.append(("single_op.b%d" % b, [one], lambda p, b=b: cfg(b, bw=1, setup=0)))
    out.append(("single_update_op", [upd], lambda p: cfg(0, bw=2, setup=0)))
    out.append(("single_op_pair", [one, upd], lambda p: cfg(0, bw=1, setup=0)))
    for b in ("0", "70"):
        bud = (lambda p: 0) if b == "0" else (lambda p: sum(p.values()) * 7 // 10)
        out.append(("chain8_zero_latency.b" + b, [gen("chain", 1, "cz", depth=8, lat="zero")],
                    lambda p, bud=bud: cfg(bud(p), bw=4, setup=0)))
    seventy = lambda p: sum(p.values()) * 7 // 10  # noqa: E731
    out.append(("vgg16_b8_zero_odd", [gen("vgg16", 8, "vz", lat="zero_odd")], lambda p: cfg(seventy(p))))
    out.append(("resnet50_b16_const1", [gen("resnet50", 16, "rc", lat=1)], lambda p: cfg(seventy(p))))
    out.append(("C1.unbounded", c1, lambda p: cfg(1 << 50)))
    out.append(("C1.budget_eq_peak", c1, lambda p: cfg(sum(p.values()))))
    out.append(("C1.budget_peak_m1", c1, lambda p: cfg(sum(p.values()) - 1)))
    out.append(("C1.budget0", c1, lambda p: cfg(0)))
    out.append(("C2.budget0", [gen("resnet50", 64, "resnet50")], lambda p: cfg(0)))
    out.append(("C1.bw1", c1, lambda p: cfg(seventy(p), bw=1)))
    out.append(("C1.setup_huge", c1, lambda p: cfg(seventy(p), setup=10 ** 12)))
    out.append(("C1.setup_huge.r01", c1, lambda p: cfg(seventy(p), setup=10 ** 12, ratios={"vgg16": 0.1})))
    out.append(("C1.ratio0", c1, lambda p: cfg(seventy(p), ratios={"vgg16": 0.0})))
    out.append(("C1.ratio1", c1, lambda p: cfg(seventy(p), ratios={"vgg16": 1.0})))
    out.append(("C1.ratio_other_job_invalid", c1, lambda p: cfg(seventy(p), ratios={"ghost": 2.0, "vgg16": 0.5})))
    out.append(("C1.ratio_other_job_valid", c1, lambda p: cfg(seventy(p), ratios={"ghost": 0.5})))
    # non-finite ratios: NaN passes PlannerConfig::validate (config.hpp:32-34)
    # and then SwapBudget::allows (swap_planner.cpp:268-276) refuses every
    # swap of that job after the first; +inf fails validation
    nan = float("nan")
    c3 = [gen("inception_v3", 32, "inception_v3"), gen("densenet", 32, "densenet"), gen("vgg16", 32, "vgg16")]
    out.append(("C1.ratio_nan", c1, lambda p: cfg(seventy(p), ratios={"vgg16": nan})))
    out.append(("C3.ratio_nan_densenet", c3, lambda p: cfg(seventy(p), ratios={"densenet": nan})))
    out.append(("C3.ratio_nan_all", c3, lambda p: cfg(seventy(p), ratios={k: nan for k in p})))
    out.append(("C3.ratio_nan_ghost", c3, lambda p: cfg(seventy(p), ratios={"ghost": nan})))
    out.append(("C1.ratio_inf_invalid", c1, lambda p: cfg(seventy(p), ratios={"vgg16": float("inf")})))
    out.append(("chain8_size_2p36.bw1", [gen("chain", 1, "cb", depth=8, size_mul=1 << 36)],
                lambda p: cfg(seventy(p), bw=1, setup=0)))
    out.append(("vgg16_b8_size_2p30", [gen("vgg16", 8, "vb", size_mul=1 << 30)],
                lambda p: cfg(seventy(p), bw=1 << 20)))
    out.append(("chain8_lat_1e12", [gen("chain", 1, "cl", depth=8, lat=10 ** 12)],
                lambda p: cfg(seventy(p), bw=1, setup=0)))
    out.append(("chain_x40", [gen("chain", 1, "c%02d" % k, depth=3 + k % 5, lat_seed=k) for k in range(40)],
                lambda p: cfg(seventy(p), bw=4, setup=1)))
    out.append(("C5.joint64", [{"c5": k} for k in range(64)], lambda p: cfg(seventy(p))))
    return out


def main():
    res = []
    for name, specs, mk in cases():
        case = {"name": name, "jobs": specs}
        jobs = edge_jobs(case)
        case["n_accesses"] = sum(len(o["inputs"]) + len(o["outputs"]) for g, _ in jobs for o in g["ops"])
        try:
            peaks = ref.initial_peaks(jobs)
        except ref.ReferenceError_ as e:  # the reference rejects the input: record its error text
            peaks = None
            case["config"] = mk({g["job_id"]: 0 for g, _ in jobs})
            case["error"] = str(e)
        if peaks is not None:
            case["config"] = mk(peaks)
            case["initial_peaks"] = peaks
            try:
                text, r = ref.build_plan(jobs, case["config"], repeats=1)
            except ref.ReferenceError_ as e:
                case["error"] = str(e)
        if "error" in case:
            print(f"{name:28s} acc={case['n_accesses']:7d} reference error: {case['error']}", flush=True)
            res.append(case)
            continue
        case.update(summarize(text, r, keep_text=len(text) < 20000))
        print(f"{name:28s} acc={case['n_accesses']:7d} swaps={case['n_swap']:5d} rc={case['n_recompute']:4d} "
              f"hist={len(case['merged_peak_history'])} ok={case['within_budget']} {case['ref_ms']:.1f} ms "
              f"{case['diagnostic'][:60]}", flush=True)
        res.append(case)
    with open(os.path.join(HERE, "edge.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
