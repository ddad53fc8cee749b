"""`memsched plan` drop-in (paper_2105_13336_b200/cli.py): the reference
CLI's plan subcommand on a scenario in the reference's own format, outputs
compared with the reference CLI's (tests/golden/scenario_c3, written by
tests/golden/make_scenario_golden.py through the unmodified reference)."""
import json
import os
import shutil

import pytest

from helpers import ensure_emu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "scenario_c3")


def _run(planner, tmp_path, scenario=None):
    from paper_2105_13336_b200 import cli
    cfg = os.path.join(GOLD, "scenario.json")
    if scenario is not None:  # a modified scenario next to copies of the graph files
        for f in os.listdir(GOLD):
            if f.endswith(".json"):
                shutil.copy(os.path.join(GOLD, f), tmp_path / f)
        cfg = str(tmp_path / "scenario.json")
        with open(cfg, "w") as fh:
            fh.write(scenario)
    out = tmp_path / "out"
    rc = cli.main(["plan", "--config", cfg, "--out", str(out)], planner=planner)
    return rc, out


def _check_outputs(out):
    for name in ("plans", "peaks"):
        with open(out / f"{name}.json") as a, open(os.path.join(GOLD, f"expected_{name}.json")) as b:
            assert a.read() == b.read(), name


def test_plan_matches_reference_cli_emu(tmp_path):
    from paper_2105_13336_b200.planner import Planner
    rc, out = _run(Planner(lib_path=ensure_emu()), tmp_path)
    assert rc == 0
    _check_outputs(out)


def _scenario(**edit):
    doc = json.load(open(os.path.join(GOLD, "scenario.json")))
    for k, v in edit.items():
        if v is None:
            doc.pop(k, None)
        else:
            doc[k] = v
    return json.dumps(doc)


@pytest.mark.parametrize("edit, text", [
    ({"bogus": 1}, "unknown field 'bogus' in scenario file"),
    ({"memory_budget": None}, "key 'memory_budget' not found"),
    ({"jobs": []}, "scenario needs at least one job"),
    ({"jobs": [{"graph_file": "vgg16.graph.json", "color": 1}]}, "unknown field 'color' in job entry"),
    ({"latency_file": None}, "scheduled mode needs a latency source"),
    ({"stall_epsilon": 2.0}, "stall_epsilon out of (0,1)"),
])
def test_scenario_errors(tmp_path, capsys, edit, text):
    from paper_2105_13336_b200.planner import Planner
    rc, _ = _run(Planner(lib_path=ensure_emu()), tmp_path, _scenario(**edit))
    assert rc == 1
    assert text in capsys.readouterr().err


@pytest.mark.gpu
def test_plan_matches_reference_cli_device(tmp_path):
    from paper_2105_13336_b200.planner import Planner
    rc, out = _run(Planner(0), tmp_path)
    assert rc == 0
    _check_outputs(out)
