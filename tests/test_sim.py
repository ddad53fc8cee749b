"""The tick-level executor model (csrc/tsl_sim.cpp: simulate in vanilla /
scheduled / passive mode, the SimController hook) and the replan lifecycle
(csrc/tsl_session.cpp: Orchestrator) against the UNMODIFIED reference
(oracle/_ref: simulate, run_scenario), value for value: every trace row (the
CSV), transfers, blocked ticks, passive fetches, violations, iteration times,
plan versions, ModeStats. The host code is the same in the CUDA library and
the CPU emulation build these tests load; tests/test_gpu_session.py repeats
the scenario runs with the device planner."""
import json
import os
import shutil

import pytest

from helpers import GOLDEN, ensure_emu, golden

from paper_2105_13336_b200 import cli, orchestrator, sim
from paper_2105_13336_b200 import configs as CF
from paper_2105_13336_b200 import workload as W


@pytest.fixture(scope="module")
def lib():
    return ensure_emu()


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref (the reference compiled from its sources) is not built")
    return R


def _same(a, b):
    for k in ("peak", "blocked_ticks", "passive_swap_count", "transfers", "safety_violations", "passive_events", "csv"):
        assert a[k] == b[k], k
    for ja, jb in zip(a["jobs"], b["jobs"]):
        assert ja == jb, ja["job_id"]


def _plans(ref, req, ratio=None):
    cfg = req.config(ref.initial_peaks(req.jobs))
    if ratio:
        cfg["max_swap_ratios"] = {g["job_id"]: ratio for g, _ in req.jobs}
    text, _ = ref.build_plan(req.jobs, cfg)
    return json.loads(text), cfg


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
@pytest.mark.parametrize("mode", ["vanilla", "scheduled", "passive"])
def test_simulate_matches_reference(lib, ref, name, mode):
    req = CF.requests(name)[-1]
    plans, cfg = _plans(ref, req)
    jobs = [(g, W.true_latency_table(g, 7), 25 * k) for k, (g, _) in enumerate(req.jobs)]
    if mode != "scheduled":
        plans = sim.baseline_plans(jobs, lib)
    kw = dict(mode=mode, iterations=3, memory_budget=cfg["memory_budget"], pcie_bandwidth=256, transfer_setup=1,
              slowdown={2: 1.25, 3: 1.5})
    _same(sim.simulate(jobs, plans, lib_path=lib, **kw), ref.simulate(jobs, plans, dict(kw)))


def test_simulate_recompute_plans(lib, ref):
    """Plans with recomputation events (max_swap_ratio 0.1): regeneration steps."""
    for name in ("C2", "C3"):
        req = CF.requests(name)[-1]
        plans, cfg = _plans(ref, req, ratio=0.1)
        assert any(p["recompute_events"] for p in plans.values())
        jobs = [(g, W.true_latency_table(g, 0), 0) for g, _ in req.jobs]
        kw = dict(mode="scheduled", iterations=2, pcie_bandwidth=256, transfer_setup=1)
        _same(sim.simulate(jobs, plans, lib_path=lib, **kw), ref.simulate(jobs, plans, dict(kw)))


def test_simulate_tight_passive_budget_and_violations(lib, ref):
    """Passive mode below the working set (LRU thrashing), and a plan whose
    swap-out never returns the tensor (safety violations + materialization)."""
    req = CF.requests("C3")[-1]
    jobs = [(g, W.true_latency_table(g, 3), 0) for g, _ in req.jobs]
    base = sim.baseline_plans(jobs, lib)
    kw = dict(mode="passive", iterations=2, memory_budget=45000, pcie_bandwidth=64, transfer_setup=2)
    _same(sim.simulate(jobs, base, lib_path=lib, **kw), ref.simulate(jobs, base, dict(kw)))
    plans, _ = _plans(ref, req)
    broken = json.loads(json.dumps(plans))
    for p in broken.values():  # drop every swap-in: outs without their ins
        p["swap_events"] = [e for e in p["swap_events"] if e["direction"] == "out"]
    kw = dict(mode="scheduled", iterations=1, pcie_bandwidth=256, transfer_setup=1)
    a = sim.simulate(jobs, broken, lib_path=lib, **kw)
    assert a["safety_violations"] or a["passive_swap_count"]
    _same(a, ref.simulate(jobs, broken, dict(kw)))


def test_controller_installs_plans_at_iteration_boundaries(lib, ref):
    """The SimController hook: a plan returned at job A's boundary applies to A
    at once and to B at B's next boundary (plan_versions per iteration)."""
    req = CF.requests("C3")[1]
    plans, _ = _plans(ref, req)
    jobs = [(g, W.true_latency_table(g, 0), 0) for g, _ in req.jobs]
    v2 = {j: dict(p, version=7) for j, p in plans.items()}
    seen = []

    def ctrl(job, it, observed):
        seen.append((job, it, len(observed)))
        return v2 if (job, it) == ("inception_v3", 0) else None

    t = sim.simulate(jobs, plans, mode="scheduled", iterations=3, pcie_bandwidth=256, transfer_setup=1,
                     controller=ctrl, lib_path=lib)
    vers = {j["job_id"]: j["plan_versions"] for j in t["jobs"]}
    assert vers["inception_v3"] == [0, 7, 7]
    assert vers["densenet"][-1] == 7
    assert ("inception_v3", 0, len(jobs[0][0]["ops"])) in seen


def test_errors_match_reference(lib, ref):
    g, _ = CF.requests("C1")[0].jobs[0]
    jobs = [(g, W.true_latency_table(g, 0), 0)]
    for kw, text in ((dict(iterations=0), "iterations must be at least 1"),
                     (dict(slowdown={1: 0.5}), "slowdown multipliers must be >= 1"),
                     (dict(ticks_per_iteration_limit=10), "iteration tick limit exceeded for job vgg16")):
        with pytest.raises(Exception) as e:
            sim.simulate(jobs, {}, lib_path=lib, **kw)
        assert str(e.value) == text
        with pytest.raises(Exception) as e2:
            ref.simulate(jobs, {}, dict(kw))
        assert str(e2.value) == text


def test_metrics_formula():
    v = {"peak": 100, "jobs": [{"job_id": "a", "iteration_times": [10, 20]}]}
    e = {"peak": 60, "jobs": [{"job_id": "a", "iteration_times": [18, 18]}]}
    m = sim.compute_metrics(v, e)
    assert m["msr"] == pytest.approx(0.4) and m["eor"] == pytest.approx(0.2) and m["cbr"] == pytest.approx(2.0)
    assert sim.compute_metrics(v, v)["cbr"] == float("inf")


def _scenario(tmp_path, **over):
    """scenario_c3 (tests/golden) with overrides; latencies scaled so the
    simulator's true latencies drift from the planning estimates."""
    d = tmp_path / "scn"
    shutil.copytree(os.path.join(GOLDEN, "scenario_c3"), d)
    doc = json.loads((d / "scenario.json").read_text())
    scale = over.pop("latency_scale", None)
    if scale is not None:
        lat = json.loads((d / "latencies.json").read_text())
        lat = {j: {o: max(0, int(t * scale)) for o, t in ops.items()} for j, ops in lat.items()}
        (d / "latencies.json").write_text(json.dumps(lat))
    doc.update(over)
    (d / "scenario.json").write_text(json.dumps(doc))
    return (d / "scenario.json").read_text(), str(d)


@pytest.mark.parametrize("over", [{}, {"latency_scale": 0.6, "replan_threshold": 0.05, "ewma_alpha": 0.5},
                                  {"latency_scale": 1.7, "replan_threshold": 0.02, "iterations": 4,
                                   "gpu_slowdown_curve": {"2": 1.2, "3": 1.4}}],
                         ids=["c3", "c3_replans", "c3_slowdown_replans"])
def test_run_scenario_matches_reference(lib, ref, tmp_path, over):
    """run_scenario (scenario.cpp:223-262): vanilla / passive / scheduled with
    the replan controller -- every mode's ModeStats and trace CSV, the plans."""
    from paper_2105_13336_b200.planner import Planner
    doc, base = _scenario(tmp_path, **over)
    ours = orchestrator.run_scenario(cli.load_scenario(doc, base), Planner(lib_path=lib))
    theirs = ref.run_scenario(doc, base)
    for mode in ("vanilla", "passive", "scheduled"):
        a, b = ours["stats"][mode], json.loads(theirs["stats"][mode])
        tm = a.pop("total_mean_iteration_time"), b.pop("total_mean_iteration_time")
        assert tm[0] == pytest.approx(tm[1], rel=1e-12)
        assert a == b, mode
        assert ours["traces"][mode]["csv"] == theirs["csv"][mode], mode
    assert ours["replan_count"] == theirs["replan_count"]
    if over:
        assert ours["replan_count"] > 0
    assert len(ours["rebuild_ms"]) == 1 + ours["replan_count"]


def test_orchestrator_lifecycle(lib, ref):
    """Arrival / departure replans with per-job plan versions (orchestrator.cpp:96-110)."""
    from paper_2105_13336_b200.planner import Planner
    req = CF.requests("C3")[-1]
    ip = ref.initial_peaks(req.jobs)
    cfg = req.config(ip)
    orch = orchestrator.Orchestrator(Planner(lib_path=lib), cfg)
    (g0, l0), (g1, l1), (g2, l2) = req.jobs
    orch.add_job(g0, l0)
    r1 = orch.rebuild()
    assert r1["jobs"]["inception_v3"]["plan"]["version"] == 1
    orch.add_job(g1, l1)
    orch.add_job(g2, l2)
    r2 = orch.rebuild()
    text, res = ref.build_plan(req.jobs, cfg)
    assert r2["merged_peak_history"] == res["merged_peak_history"]
    assert {j: v["plan"]["version"] for j, v in r2["jobs"].items()} == {"inception_v3": 2, "densenet": 1, "vgg16": 1}
    orch.remove_job("densenet")
    r3 = orch.rebuild()
    assert sorted(r3["jobs"]) == ["inception_v3", "vgg16"]
    # no drift: no replan; a 50 % drift replans and EWMA-corrects the estimates
    assert orch.replan_if_needed({"vgg16": l2}) is None
    doubled = {o: 2 * t for o, t in l2.items()}
    new = orch.replan_if_needed({"vgg16": doubled})
    assert new is not None and orch.replan_count == 1
    alpha = cfg.get("ewma_alpha", 0.3)
    op = next(iter(l2))
    assert orch.latencies("vgg16")[op] == round(alpha * 2 * l2[op] + (1 - alpha) * l2[op])
    assert new["vgg16"]["version"] == 3
