"""Generates tests/golden/scenario_c3/: a scenario in the reference's own
format (C3's three graphs written by the reference's save_graph, their true
latency tables, the scenario document) and the reference CLI `plan` outputs
for it (load_scenario + plan_scenario through oracle/_ref, formatted as
tools/memsched_cli.cpp:136-153 writes them). Run in this container only.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "scenario_c3")


def main():
    os.makedirs(OUT, exist_ok=True)
    lat = {}
    jobs = []
    for fam in ("inception_v3", "densenet", "vgg16"):
        g_json, l_json = ref.generate_workload(fam, 32, 0, 0, fam, 13)
        with open(os.path.join(OUT, f"{fam}.graph.json"), "w") as f:
            f.write(g_json if isinstance(g_json, str) else json.dumps(g_json, indent=1))
        g = json.loads(g_json) if isinstance(g_json, str) else g_json
        lt = json.loads(l_json) if isinstance(l_json, str) else l_json
        lat[fam] = lt
        jobs.append((g, lt))
    with open(os.path.join(OUT, "latencies.json"), "w") as f:
        json.dump(lat, f, indent=1, sort_keys=True)
    peaks = ref.initial_peaks(jobs)
    scenario = {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": sum(peaks.values()) * 7 // 10,
                "latency_file": "latencies.json", "iterations": 3, "seed": 13,
                "jobs": [{"graph_file": "inception_v3.graph.json"},
                         {"graph_file": "densenet.graph.json", "max_swap_ratio": 0.5, "launch_tick": 40},
                         {"graph_file": "vgg16.graph.json", "launch_tick": 90}]}
    doc = json.dumps(scenario, indent=1)
    with open(os.path.join(OUT, "scenario.json"), "w") as f:
        f.write(doc)
    plans, peaks_doc, diag = ref.plan_scenario(doc, OUT)
    with open(os.path.join(OUT, "expected_plans.json"), "w") as f:
        f.write(plans)
    with open(os.path.join(OUT, "expected_peaks.json"), "w") as f:
        f.write(peaks_doc)
    with open(os.path.join(OUT, "expected_diagnostic.txt"), "w") as f:
        f.write(diag)
    print("wrote", OUT, len(plans), len(peaks_doc), repr(diag[:60]))


if __name__ == "__main__":
    main()
