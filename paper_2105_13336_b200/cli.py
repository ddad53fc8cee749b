"""`memsched plan` on the B200 planner: the reference CLI's plan subcommand
(tools/memsched_cli.cpp:136-153) as a process-level drop-in.

    python -m paper_2105_13336_b200.cli plan --config scenario.json --out DIR [--seed N]

Reads the reference's scenario document (load_scenario, scenario.cpp:37-108:
the same known fields, the same per-job entries, graph_file paths relative to
the scenario file, the same ValidationError texts), plans it the way
plan_scenario does (scenario.cpp:213-221 -> Orchestrator::plan_with_latencies
-> build_plan, one rebuild, so every plan gets version 1) and writes
DIR/plans.json (save_plans) and DIR/peaks.json (the CLI's {"job": PeakReport}
document) byte-identical to the reference CLI's. The plan diagnostic, if any,
goes to stdout; errors print "error: <text>" and exit 1 (memsched_cli.cpp:175-178).

Latency source: `latency_file` ({job: {op: ticks}}) or `predictor_file` (a
LatencyPredictor document: cold start, every op's latency predicted at the
config's cold_start_gpu_usage -- latency.py / csrc/tsl_latency.cpp).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from typing import List, Optional

KNOWN = {"pcie_bandwidth", "transfer_setup", "memory_budget", "ewma_alpha", "replan_threshold", "stall_epsilon",
         "stall_min_iters", "jobs", "iterations", "seed", "gpu_slowdown_curve", "predictor_file", "latency_file"}
JOB_KNOWN = {"graph_file", "max_swap_ratio", "launch_tick"}


class CliError(Exception):
    pass


def _resolve(base_dir: str, path: str) -> str:  # scenario.cpp:28-33
    if os.path.isabs(path) or not base_dir:
        return path
    return os.path.join(base_dir, path)


def _read(path: str) -> str:
    try:
        with open(path, "rb") as f:
            return f.read().decode()
    except OSError:
        raise CliError("cannot read file: " + path)


def _at(doc: dict, key: str):  # nlohmann json::at's message
    if key not in doc:
        raise CliError(f"[json.exception.out_of_range.403] key '{key}' not found")
    return doc[key]


def load_scenario(document: str, base_dir: str) -> dict:
    """load_scenario (scenario.cpp:37-108) -> {"config", "jobs" [(graph, entry)], "latency_file", ...}."""
    try:
        doc = json.loads(document)
    except json.JSONDecodeError as e:
        raise CliError("scenario file is not valid JSON: " + str(e))
    if not isinstance(doc, dict):
        raise CliError("scenario file must be an object")
    for key in sorted(doc):  # nlohmann objects iterate in key order
        if key not in KNOWN:
            raise CliError(f"unknown field '{key}' in scenario file")
    cfg = {"pcie_bandwidth": int(_at(doc, "pcie_bandwidth")), "transfer_setup": int(_at(doc, "transfer_setup")),
           "memory_budget": int(_at(doc, "memory_budget"))}
    for key in ("ewma_alpha", "replan_threshold", "stall_epsilon"):
        if key in doc:
            cfg[key] = float(doc[key])
    if "stall_min_iters" in doc:
        cfg["stall_min_iters"] = int(doc["stall_min_iters"])
    out = {"config": cfg, "jobs": [], "launch_ticks": [],
           "iterations": int(doc.get("iterations", 3)), "seed": int(doc.get("seed", 0)),
           "gpu_slowdown_curve": {int(k): float(v) for k, v in doc.get("gpu_slowdown_curve", {}).items()},
           "predictor_file": _resolve(base_dir, doc["predictor_file"]) if "predictor_file" in doc else "",
           "latency_file": _resolve(base_dir, doc["latency_file"]) if "latency_file" in doc else ""}
    entries = []
    for j in _at(doc, "jobs"):
        for key in sorted(j):
            if key not in JOB_KNOWN:
                raise CliError(f"unknown field '{key}' in job entry")
        entries.append({"graph_file": _resolve(base_dir, _at(j, "graph_file")),
                        "max_swap_ratio": float(j.get("max_swap_ratio", 1.0)),
                        "launch_tick": int(j.get("launch_tick", 0))})
    if not entries:
        raise CliError("scenario needs at least one job")
    ratios = {}
    for e in entries:
        try:
            g = json.loads(_read(e["graph_file"]))
        except json.JSONDecodeError as ex:
            raise CliError("graph file is not valid JSON: " + str(ex))
        ratios[g.get("job_id", "")] = e["max_swap_ratio"]
        out["jobs"].append(g)
        out["launch_ticks"].append(e["launch_tick"])
    cfg["max_swap_ratios"] = ratios
    return out


def plan_scenario(scn: dict, planner) -> tuple:
    """plan_scenario (scenario.cpp:213-221): (plans.json, peaks.json, diagnostic)."""
    if scn["latency_file"]:
        table = json.loads(_read(scn["latency_file"]))
    elif scn["predictor_file"]:
        # Orchestrator::plan_cold_start (orchestrator.cpp:118-124): every op's
        # latency from the fitted predictor at cold_start_gpu_usage
        from .latency import LatencyPredictor
        pred = LatencyPredictor.from_json(_read(scn["predictor_file"]), lib_path=planner.lib._name)
        usage = scn["config"].get("cold_start_gpu_usage", 0.5)
        table = {g.get("job_id", ""): pred.predict_latencies(g, usage) for g in scn["jobs"]}
    else:
        raise CliError("scheduled mode needs a latency source: fit a predictor (predictor_file) or supply a "
                       "latency table (latency_file)")
    jobs = []
    for g in scn["jobs"]:
        jid = g.get("job_id", "")
        if jid not in table:
            raise CliError("map::at")  # Orchestrator::rebuild's latencies_.at(job)
        jobs.append((g, {op: int(t) for op, t in table[jid].items()}))
    out = planner.build_plan(jobs, scn["config"])
    # Orchestrator::rebuild numbers every plan of its first build version 1
    plans = out["plans_json"].replace('    "version": 0,\n', '    "version": 1,\n')
    peaks = "{\n" + ",\n".join(f'"{jid}": {out["reports_json"][jid]}' for jid in sorted(out["reports_json"])) + "}\n"
    return plans, peaks, out.get("diagnostic", "")


def main(argv: Optional[List[str]] = None, planner=None) -> int:
    ap = argparse.ArgumentParser(prog="memsched")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("plan", help="Build scheduling plans for a scenario without simulating")
    p.add_argument("--config", required=True)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--out", required=True)
    p.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    try:
        if planner is None:
            from paper_2105_13336_b200.planner import Planner
            planner = Planner(a.device)
        scn = load_scenario(_read(a.config), os.path.dirname(a.config))
        plans, peaks, diag = plan_scenario(scn, planner)
        os.makedirs(a.out, exist_ok=True)
        with open(os.path.join(a.out, "plans.json"), "w") as f:
            f.write(plans)
        with open(os.path.join(a.out, "peaks.json"), "w") as f:
            f.write(peaks)
        if diag:
            print(diag)
    except Exception as e:  # memsched_cli.cpp:175-178
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
