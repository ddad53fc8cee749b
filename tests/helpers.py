"""Shared test helpers: golden fixtures, job reconstruction, comparisons."""
from __future__ import annotations

import functools
import hashlib
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
EMU_LIB = os.path.join(ROOT, "tests", "emu", "build", "libtsl_emu.so")


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


@functools.lru_cache(None)
def golden(name: str):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def fuzz_jobs(case):
    from paper_2105_13336_b200 import workload as W
    jobs = []
    for spec in case["jobs"]:
        if "gen" in spec:
            fam, batch, depth, jid, lat_seed = spec["gen"]
            g = W.generate_workload(fam, batch, 0, depth, jid)
            jobs.append((g, W.true_latency_table(g, lat_seed)))
        else:
            jobs.append((spec["graph"], spec["latencies"]))
    return jobs


def config_jobs(case):
    """Jobs of a configs.json case (C1..C5 requests rebuilt by configs.py)."""
    from paper_2105_13336_b200 import configs as CF
    name = case["name"]
    base = name.split(".")[0]
    reqs = CF.requests(base, ratio=case["ratio"])
    return next(r for r in reqs if r.name == name).jobs


def check_against_golden(out: dict, case: dict):
    """out: planner/oracle build_plan dict; case: golden summary."""
    assert out["merged_peak_history"] == case["merged_peak_history"]
    assert out["final_merged_peak"] == case["final_merged_peak"]
    assert out["within_budget"] == case["within_budget"]
    assert out["diagnostic"] == case["diagnostic"]
    assert sha(out["plans_json"]) == case["plans_sha256"], "save_plans bytes differ from the reference"
    for jid, digest in case["reports_sha256"].items():
        assert sha(json.dumps(json.loads(out["reports_json"][jid]), indent=2)) == digest, f"PeakReport of {jid}"
    if "plans_json" in case:
        assert out["plans_json"] == case["plans_json"]


def ensure_oracle():
    from oracle import tslo
    if not tslo.available():
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       stdout=subprocess.DEVNULL)
    return tslo


def ensure_emu():
    """TEST-ONLY CPU emulation build of the planner (tests/emu)."""
    subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "emu")], check=True, stdout=subprocess.DEVNULL)
    return EMU_LIB


def edge_jobs(case):
    """Jobs of an edge.json case. Job specs: {"graph", "latencies"} verbatim, {"c5": k}
    (configs.c5_job), or {"gen": [family, batch, depth, job_id, lat_seed]} with optional
    "size_mul" (every tensor size x k) and "lat" ("table" | "zero" | "zero_odd" | int constant)."""
    from paper_2105_13336_b200 import configs as CF
    from paper_2105_13336_b200 import workload as W
    jobs = []
    for spec in case["jobs"]:
        if "graph" in spec:
            jobs.append((spec["graph"], spec["latencies"]))
            continue
        if "c5" in spec:
            jobs.append(CF.c5_job(spec["c5"]))
            continue
        fam, batch, depth, jid, lat_seed = spec["gen"]
        g = W.generate_workload(fam, batch, 0, depth, jid)
        mul = spec.get("size_mul", 1)
        if mul != 1:
            for t in g["tensors"]:
                t["size"] *= mul
        lat = W.true_latency_table(g, lat_seed)
        mode = spec.get("lat", "table")
        if mode == "zero":
            lat = {o: 0 for o in lat}
        elif mode == "zero_odd":
            lat = {o["id"]: (0 if i % 2 else lat[o["id"]]) for i, o in enumerate(g["ops"])}
        elif isinstance(mode, int):
            lat = {o: mode for o in lat}
        jobs.append((g, lat))
    return jobs


def check_edge(build_plan, case):
    """One edge.json case: the reference's plan, or the reference's error text."""
    import pytest
    if "error" in case:
        with pytest.raises(Exception) as e:
            build_plan(edge_jobs(case), case["config"])
        assert str(e.value) == case["error"]
    else:
        check_against_golden(build_plan(edge_jobs(case), case["config"]), case)
