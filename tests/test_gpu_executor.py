"""Plan executor (north-star item 5; reference analogue: the scheduled mode of
memsched::simulate, simulator.cpp:112-569): replaying a plan on the device
with real pinned-host cudaMemcpyAsync swaps must reproduce the planner's
predicted peak as the executor allocator's high-water mark, move every tensor
through host memory intact (swapped-out device slots are poisoned), and keep
the planned iteration length (test_simulator.cpp:71-110 checks the same on
the reference's simulated executor: scheduled peak == final_merged_peak)."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def planner():
    from paper_2105_13336_b200.planner import Planner
    return Planner(0)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_replay_matches_prediction(planner, name):
    from paper_2105_13336_b200 import configs as CF
    req = CF.requests(name)[-1]
    out = planner.build_and_execute(req.jobs, req.config(CF.INITIAL_PEAK), tick_ns=2000, iterations=3)
    for jid, r in out["exec"].items():
        assert r["verify_errors"] == 0, jid
        assert r["violations"] == 0, jid
        assert r["hwm"] == r["predicted_peak"], (jid, r["hwm"], r["predicted_peak"])
        plan = __import__("json").loads(out["plan"]["plans_json"])[jid]
        n_out = sum(1 for e in plan["swap_events"] if e["direction"] == "out")
        assert r["swap_outs"] == 3 * n_out and r["swap_ins"] == 3 * n_out
        for ms in r["iteration_ms"]:
            assert abs(ms - r["planned_iteration_ms"]) / r["planned_iteration_ms"] < 0.02


def test_replay_with_recomputation(planner):
    """max_swap_ratio 0.1 makes the planner recompute; the replay runs the
    regeneration steps and still meets the predicted peak."""
    from paper_2105_13336_b200 import configs as CF
    req = CF.requests("C2", ratio=0.1)[0]
    out = planner.build_and_execute(req.jobs, req.config(CF.INITIAL_PEAK), tick_ns=2000, iterations=2)
    plan = __import__("json").loads(out["plan"]["plans_json"])["resnet50"]
    assert plan["recompute_events"]
    r = out["exec"]["resnet50"]
    assert r["verify_errors"] == 0 and r["violations"] == 0
    assert r["hwm"] == r["predicted_peak"]
