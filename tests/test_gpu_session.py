"""The replan lifecycle with the device planner: run_scenario (vanilla /
passive / scheduled with the ReplanController driving Orchestrator::
replan_if_needed, every rebuild a planning-kernel launch) against the
UNMODIFIED reference's run_scenario (oracle/_ref), ModeStats and trace CSV
value for value; arrival / departure replans of a C5 shard through the
session API against the reference's build_plan."""
import json

import pytest

from test_sim import _scenario

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    from paper_2105_13336_b200.planner import Planner
    return Planner(0)


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref is not built")
    return R


@pytest.mark.parametrize("over", [{}, {"latency_scale": 0.6, "replan_threshold": 0.05, "ewma_alpha": 0.5},
                                  {"latency_scale": 1.7, "replan_threshold": 0.02, "iterations": 4,
                                   "gpu_slowdown_curve": {"2": 1.2, "3": 1.4}}],
                         ids=["c3", "c3_replans", "c3_slowdown_replans"])
def test_run_scenario_on_device_matches_reference(planner, ref, tmp_path, over):
    from paper_2105_13336_b200 import cli, orchestrator
    doc, base = _scenario(tmp_path, **over)
    ours = orchestrator.run_scenario(cli.load_scenario(doc, base), planner)
    theirs = ref.run_scenario(doc, base)
    for mode in ("vanilla", "passive", "scheduled"):
        a, b = ours["stats"][mode], json.loads(theirs["stats"][mode])
        tm = a.pop("total_mean_iteration_time"), b.pop("total_mean_iteration_time")
        assert tm[0] == pytest.approx(tm[1], rel=1e-12)
        assert a == b, mode
        assert ours["traces"][mode]["csv"] == theirs["csv"][mode], mode
    assert ours["replan_count"] == theirs["replan_count"]
    assert len(ours["rebuild_ms"]) == 1 + ours["replan_count"]


def test_session_arrivals_and_departures_c5_shard(planner, ref):
    """C5 shard 3 through ONE session: 8 arrivals then 7 departures, each a
    rebuild (one device launch) of the active set, against the reference's
    build_plan of the same set; plan versions count each job's rebuilds."""
    from paper_2105_13336_b200 import configs as CF
    from paper_2105_13336_b200.orchestrator import Orchestrator
    s = 3
    jobs = {k: CF.c5_job(k) for k in range(8 * s, 8 * s + 8)}
    peaks = ref.initial_peaks(list(jobs.values()))
    cfg = CF.planner_config(CF.budget_of(list(peaks.values())) // 2)
    orch = Orchestrator(planner, cfg)
    active, rebuilds = [], {}
    for want in CF.c5_shard_events(s):
        for k in want:
            if k not in active:
                orch.add_job(*jobs[k])
        for k in list(active):
            if k not in want:
                orch.remove_job("w%02d" % k)
        active = list(want)
        got = orch.rebuild()
        for k in want:
            rebuilds[k] = rebuilds.get(k, 0) + 1
        text, res = ref.build_plan([jobs[k] for k in want], cfg)
        assert got["merged_peak_history"] == res["merged_peak_history"]
        plans = json.loads(text)
        for jid, p in plans.items():
            mine = got["jobs"][jid]["plan"]
            assert mine["release_flags"] == p["release_flags"], jid
            assert [(e["event_id"], e["start_time"]) for e in mine["swap_events"]] == \
                [(e["event_id"], e["start_time"]) for e in p["swap_events"]], jid
            assert mine["version"] == rebuilds[int(jid[1:])], jid
    assert len(orch.rebuild_ms) == len(CF.c5_shard_events(s))
