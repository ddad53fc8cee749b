"""Generates tests/golden/stall.json: builds where build_plan's stall rule fires.

The stall rule (orchestrator.cpp:35-41) ends the loop once iter > stall_min_iters
and the mean per-job peak moved by less than stall_epsilon (relative) over the last
three rounds. With the default stall_min_iters = 100 it never fires on the configs
(they converge in <= 11 loop iterations), so this fixture sweeps stall_min_iters
0..4 and stall_epsilon 0.05..0.9 over C1, C2, the C3 arrivals and C5 shard
replans, at max_swap_ratio 1.0 and 0.1 (recomputation passes lengthen the loop),
and keeps every case whose merged-peak history is shorter than the same build's
with the default settings -- i.e. where the rule really cut the loop. Records
are produced by the UNMODIFIED reference (oracle/_ref via oracle/ref.py), in
make_golden.summarize's format. Run here:

    make -C oracle ref && python tests/golden/make_stall_golden.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import ref  # noqa: E402
from paper_2105_13336_b200 import configs as CF  # noqa: E402
from make_golden import summarize  # noqa: E402

REQUESTS = ["C1", "C2", "C3.1", "C3.2", "C3.3", "C5s1.3", "C5s4.7", "C5s6.12"]
SWEEP = [(0, 0.05), (0, 0.9), (1, 0.2), (2, 0.5), (3, 0.05), (3, 0.9), (4, 0.3)]


def request(name: str, ratio):
    base = name.split(".")[0]
    return next(r for r in CF.requests(base, ratio=ratio) if r.name == name)


def main():
    if not ref.available():
        sys.exit("build the reference first: make -C oracle ref")
    out = []
    for name in REQUESTS:
        for ratio in (None, 0.1):
            req = request(name, ratio)
            ip = ref.initial_peaks(req.jobs)
            base_cfg = req.config(ip)
            _, base = ref.build_plan(req.jobs, base_cfg, repeats=1)
            for mi, eps in SWEEP:
                cfg = dict(base_cfg, stall_min_iters=mi, stall_epsilon=eps)
                text, res = ref.build_plan(req.jobs, cfg, repeats=1)
                fired = len(res["merged_peak_history"]) < len(base["merged_peak_history"])
                print(f"{name:8s} r={ratio} min_iters={mi} eps={eps:4} hist {len(base['merged_peak_history'])}"
                      f" -> {len(res['merged_peak_history'])} {'FIRES' if fired else ''}", flush=True)
                if fired:
                    out.append({"name": name, "ratio": ratio, "config": cfg,
                                "default_history": base["merged_peak_history"],
                                **summarize(text, res)})
    with open(os.path.join(HERE, "stall.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(len(out), "cases")


if __name__ == "__main__":
    main()
