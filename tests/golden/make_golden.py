"""Generates tests/golden/*.json from the UNMODIFIED reference.

The reference hot path is compiled from /root/reference/proj/src by
oracle/Makefile into oracle/_ref/libmemsched_ref.so (test infrastructure);
this script drives it through oracle/ref.py and records, per case, the
reference's own serialisations (save_plans text and PeakReport::to_json
text) as sha256 digests, plus the merged-peak history and a few counts.
Small cases keep their full text. Run here (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

Fixture sources (reference file:line):
  configs.json    BASELINE.json configs C1, C2, C3, C5,
                  planner settings of test_acceptance.cpp:195-202, plus the
                  max_swap_ratio 0.1 variants that exercise recomputation
  handbuilt.json  the hand-built graphs of the reference unit tests:
                  small_chain_job (test_peak.cpp:40-62), decay job
                  (test_peak.cpp:118-183), two_candidate_job
                  (test_recompute.cpp:19-38), gap_job (test_swap.cpp:157-174),
                  chain depth 3 (test_swap.cpp:230-267)
  analyze.json    analyze_job on caller plans: test_peak.cpp:66-183 cases and
                  testsup::planned_random_job seeds 0..49 (test_support.hpp:182-226)
  fuzz.json       random graphs (testsup::random_job, generator families) x
                  random planner configs
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2105_13336_b200 import configs as CF  # noqa: E402
from paper_2105_13336_b200 import workload as W  # noqa: E402


def h(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def summarize(plans_json: str, res: dict, keep_text: bool = False) -> dict:
    out = {
        "plans_sha256": h(plans_json),
        "reports_sha256": {j: h(json.dumps(r, indent=2)) for j, r in res["reports"].items()},
        "merged_peak_history": res["merged_peak_history"],
        "final_merged_peak": res["final_merged_peak"],
        "within_budget": res["within_budget"],
        "diagnostic": res["diagnostic"],
        "ref_ms": min(res["times_ms"]),
    }
    plans = json.loads(plans_json)
    out["n_swap"] = sum(len(p["swap_events"]) for p in plans.values())
    out["n_recompute"] = sum(len(p["recompute_events"]) for p in plans.values())
    if keep_text:
        out["plans_json"] = plans_json
        out["reports"] = res["reports"]
    return out


def graph_doc(tensors, ops, job_id):
    return {"job_id": job_id,
            "tensors": [{"id": i, "size": s, "kind": k} for i, s, k in tensors],
            "ops": [{"id": o, "kind": kd, "inputs": ins, "outputs": outs, "attributes": [],
                     "phase": ph} for o, ins, outs, ph, kd in ops]}


def F(o, ins, outs):
    return (o, ins, outs, "forward_backward", "f")


def handbuilt():
    G = {}
    G["small"] = (graph_doc([("x", 4, "input"), ("t1", 8, "interim"), ("t2", 2, "interim")],
                            [F("conv", ["x"], ["t1"]), F("relu", ["t1"], ["t2"])], "small"),
                  {"conv": 10, "relu": 5})
    G["decay"] = (graph_doc([("x", 4, "input"), ("t1", 8, "interim"), ("t2", 4, "interim"),
                             ("t3", 16, "interim"), ("t4", 2, "interim"), ("t5", 2, "interim"),
                             ("y", 1, "interim")],
                            [F("A", ["x"], ["t1"]), F("B", ["x"], ["t2"]), F("D", ["t2"], ["t3"]),
                             F("E", ["t3"], ["t4"]), F("E2", ["t4"], ["t5"]), F("C", ["t1", "t5"], ["y"])],
                            "decay"),
                  {"A": 10, "B": 10, "D": 10, "E": 10, "E2": 10, "C": 5})
    G["rc"] = (graph_doc([("x", 4, "input"), ("t2", 8, "interim"), ("t4", 20, "interim"),
                          ("big", 64, "interim"), ("m", 4, "interim"), ("y", 1, "interim")],
                         [F("A", ["x"], ["t2"]), F("A2", ["x"], ["t4"]), F("B", ["x"], ["big"]),
                          F("B2", ["big"], ["m"]), F("C", ["t2", "t4", "m"], ["y"])], "rc"),
               {"A": 5, "A2": 2, "B": 8, "B2": 10, "C": 5})
    for fl in (50, 4):
        G[f"gap{fl}"] = (graph_doc([("x", 4, "input"), ("t", 8, "interim"), ("u", 2, "interim"),
                                    ("v", 1, "interim")],
                                   [F("a", ["x"], ["t"]), F("b", ["x"], ["u"]), F("c", ["t", "u"], ["v"])],
                                   f"gap{fl}"),
                         {"a": 10, "b": fl, "c": 10})
    g = W.generate_workload("chain", 1, 0, 3, "wrapjob")
    G["wrapjob"] = (g, {o["id"]: 10 for o in g["ops"]})
    G["wrap"] = (graph_doc([("x", 4, "input"), ("w", 16, "parameter"), ("w_new", 16, "updated_parameter"),
                            ("g", 8, "interim")],
                           [F("F", ["x", "w"], ["g"]), ("U", ["w", "g"], ["w_new"], "optimize", "update")],
                           "wrap"),
                 {"F": 10, "U": 10})
    out = {}
    for name, (g, lat) in G.items():
        for cfg in ({"pcie_bandwidth": 4, "transfer_setup": 0, "memory_budget": 0},
                    {"pcie_bandwidth": 2, "transfer_setup": 1, "memory_budget": 0},
                    {"pcie_bandwidth": 128, "transfer_setup": 0, "memory_budget": 0},
                    {"pcie_bandwidth": 4, "transfer_setup": 0, "memory_budget": 0,
                     "max_swap_ratios": {g["job_id"]: 0.1}}):
            text, res = ref.build_plan([(g, lat)], cfg, repeats=1)
            out.setdefault(name, {"graph": g, "latencies": lat, "cases": []})["cases"].append(
                {"config": cfg, **summarize(text, res, keep_text=True)})
    return out


def analyze_cases():
    cases = []
    # small chain with the documented flags (test_peak.cpp:40-62): x's and t1's TUAs
    g = graph_doc([("x", 4, "input"), ("t1", 8, "interim"), ("t2", 2, "interim")],
                  [F("conv", ["x"], ["t1"]), F("relu", ["t1"], ["t2"])], "small")
    lat = {"conv": 10, "relu": 5}
    # accesses: conv: TUA x (0), TGA t1 (1); relu: TUA t1 (2), TGA t2 (3)
    plan = {"version": 0, "swap_events": [], "recompute_events": [], "release_flags": [0, 2]}
    cases.append({"name": "small_chain", "graph": g, "latencies": lat, "plan": plan,
                  "expect": {"memory_peak": 12, "peak_time": 0, "peak_tensors": ["t1", "x"]}})
    # decay job + t1 swap pair (test_peak.cpp:118-183): MP 32 -> 24, 21 timeline events
    g = graph_doc([("x", 4, "input"), ("t1", 8, "interim"), ("t2", 4, "interim"), ("t3", 16, "interim"),
                   ("t4", 2, "interim"), ("t5", 2, "interim"), ("y", 1, "interim")],
                  [F("A", ["x"], ["t1"]), F("B", ["x"], ["t2"]), F("D", ["t2"], ["t3"]),
                   F("E", ["t3"], ["t4"]), F("E2", ["t4"], ["t5"]), F("C", ["t1", "t5"], ["y"])], "decay")
    lat = {"A": 10, "B": 10, "D": 10, "E": 10, "E2": 10, "C": 5}
    # topo order A,B,D,E,E2,C -> accesses: A: TUA x 0, TGA t1 1; B: x 2, t2 3; D: t2 4, t3 5;
    # E: t3 6, t4 7; E2: t4 8, t5 9; C: t1 10, t5 11, y 12. Activity-analysis flags (last access
    # of each interim) plus t1's TGA, whose release the swap-out owns (test_peak.cpp:164).
    flags = [1, 4, 6, 8, 10, 11, 12]
    out = {"event_id": 0, "tensor": "t1", "direction": "out", "trigger_access": 1, "delta_time": 0,
           "wraps_iteration": False, "start_time": 10, "end_time": 11, "pair_id": 1, "serves_access": -1}
    inn = dict(out, event_id=1, direction="in", start_time=48, end_time=49, pair_id=0, serves_access=10)
    plan = {"version": 0, "swap_events": [out, inn], "recompute_events": [], "release_flags": flags}
    cases.append({"name": "decay_swap", "graph": g, "latencies": lat, "plan": plan,
                  "expect": {"memory_peak": 24}})
    for seed in range(50):
        pj = ref.planned_random_job(seed, 3, 4, 1)
        cases.append({"name": f"planned{seed}", "graph": pj["graph"], "latencies": pj["latencies"],
                      "plan": pj["plan"], "expect": {"memory_peak": pj["replay_oracle"]["peak"],
                                                     "peak_time": pj["replay_oracle"]["peak_time"],
                                                     "peak_tensors": pj["replay_oracle"]["tensors"]}})
    for c in cases:
        r = ref.analyze_job(c["graph"], c["latencies"], c["plan"])
        c["report"] = r
        for k, v in c["expect"].items():
            assert r[k] == v, (c["name"], k, r[k], v)
    return cases


def fuzz_cases(n=120):
    fams = ["vgg16", "resnet50", "inception_v3", "inception_v4", "densenet", "chain"]
    out = []
    for seed in range(n):
        rnd = random.Random(1000 + seed)
        jobs, specs = [], []
        for k in range(rnd.choice([1, 1, 2, 3])):
            if rnd.random() < 0.5:
                g, l = ref.random_job(seed * 10 + k)
                g["job_id"] = f"r{seed}_{k}"
                spec = {"graph": g, "latencies": l}
            else:
                gen = [rnd.choice(fams), rnd.choice([1, 8, 32]), rnd.randint(2, 30), f"j{k}", rnd.randint(0, 99)]
                g = W.generate_workload(gen[0], gen[1], 0, gen[2], gen[3])
                l = W.true_latency_table(g, gen[4])
                spec = {"gen": gen}  # regenerated by paper_2105_13336_b200.workload
            jobs.append((g, l))
            specs.append(spec)
        ip = ref.initial_peaks(jobs)
        cfg = {"pcie_bandwidth": rnd.choice([1, 2, 4, 16, 64, 256]), "transfer_setup": rnd.choice([0, 1, 3]),
               "memory_budget": sum(ip.values()) * rnd.choice([3, 5, 7, 9]) // 10}
        if rnd.random() < 0.3:
            cfg["max_swap_ratios"] = {g["job_id"]: rnd.choice([0.1, 0.3, 0.5, 1.0]) for g, _ in jobs}
        text, res = ref.build_plan(jobs, cfg, repeats=1)
        out.append({"seed": seed, "jobs": specs, "config": cfg,
                    **summarize(text, res)})
    return out


def config_cases():
    out = []
    for ratio in (None, 0.1):
        # every C5 shard (15 arrival/departure replans each) at both ratios
        for name in ["C1", "C2", "C3"] + [f"C5s{g}" for g in range(8)]:
            for req in CF.requests(name, ratio=ratio):
                ip = ref.initial_peaks(req.jobs)
                cfg = req.config(ip)
                text, res = ref.build_plan(req.jobs, cfg, repeats=1 if name.startswith("C5") else 3)
                out.append({"name": req.name, "ratio": ratio, "config": cfg,
                            "initial_peaks": ip, "n_accesses": req.n_accesses,
                            **summarize(text, res, keep_text=(name == "C1"))})
                print(req.name, ratio, out[-1]["final_merged_peak"], flush=True)
    return out


def main():
    if not ref.available():
        sys.exit("build the reference first: make -C oracle ref")
    if sys.argv[1:] == ["configs"]:  # regenerate configs.json only
        with open(os.path.join(HERE, "configs.json"), "w") as f:
            json.dump(config_cases(), f, indent=1)
        return
    with open(os.path.join(HERE, "analyze.json"), "w") as f:
        json.dump(analyze_cases(), f, separators=(",", ":"))
    with open(os.path.join(HERE, "handbuilt.json"), "w") as f:
        json.dump(handbuilt(), f, separators=(",", ":"))
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(config_cases(), f, indent=1)
    with open(os.path.join(HERE, "fuzz.json"), "w") as f:
        json.dump(fuzz_cases(), f, separators=(",", ":"))


if __name__ == "__main__":
    main()
