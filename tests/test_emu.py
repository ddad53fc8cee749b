"""Algorithm checks on CPU through the TEST-ONLY emulation build
(tests/emu: the product's tsl_plan.cuh + tsl_host.cpp compiled for the host
with a one-thread execution context). The product library never contains
this build; the GPU tests (test_gpu_parity.py) check the CUDA build itself.
"""
import json

import pytest

from helpers import check_against_golden, check_edge, config_jobs, ensure_emu, fuzz_jobs, golden
from paper_2105_13336_b200 import abi, workload as W
from paper_2105_13336_b200.planner import Planner, ValidationError


@pytest.fixture(scope="module")
def emu():
    return Planner(lib_path=ensure_emu())


@pytest.mark.parametrize("case", [c for c in golden("configs") if c["name"].split(".")[0] in ("C1", "C2", "C3")
                                  or c["name"] in ("C5s0.7", "C5s0.14", "C5s1.7", "C5s3.5")],
                         ids=lambda c: f"{c['name']}-r{c['ratio']}")
def test_configs(emu, case):
    check_against_golden(emu.build_plan(config_jobs(case), case["config"]), case)


@pytest.mark.parametrize("case", golden("fuzz")[::2], ids=lambda c: f"seed{c['seed']}")
def test_fuzz(emu, case):
    check_against_golden(emu.build_plan(fuzz_jobs(case), case["config"]), case)


@pytest.mark.parametrize("case", golden("stall"), ids=lambda c: f"{c['name']}-r{c['ratio']}-"
                         f"{c['config']['stall_min_iters']}-{c['config']['stall_epsilon']}")
def test_stall_rule(emu, case):
    """Builds where the stall rule (orchestrator.cpp:35-41) fires."""
    check_against_golden(emu.build_plan(config_jobs(case), case["config"]), case)


@pytest.mark.parametrize("window", [1, 5, 64])
def test_speculation_windows(emu, window, monkeypatch):
    """Swap passes speculating in windows of the candidate order (the busy
    structure advanced between windows) plan exactly what one pass-wide
    speculation plans: the reference's fixtures, byte for byte."""
    monkeypatch.setenv("TSL_SPEC_WINDOW", str(window))
    cases = [c for c in golden("configs") if c["name"] in ("C1", "C2", "C3.3", "C5s2.7")]
    for case in cases:
        check_against_golden(emu.build_plan(config_jobs(case), case["config"]), case)
    for case in golden("fuzz")[1::6]:
        check_against_golden(emu.build_plan(fuzz_jobs(case), case["config"]), case)


def test_handbuilt(emu):
    for name, spec in golden("handbuilt").items():
        for case in spec["cases"]:
            check_against_golden(emu.build_plan([(spec["graph"], spec["latencies"])], case["config"]), case)


def test_analyze(emu):
    for c in golden("analyze"):
        r = emu.analyze_job(c["graph"], c["latencies"], c["plan"])
        assert json.loads(r["report_json"]) == c["report"], c["name"]


def _chain():
    g = W.generate_workload("chain", 1, 0, 3, "cj")
    return g, W.true_latency_table(g, 1)


# (mutation, expected ValidationError text) -- texts from graph.cpp:49-119,
# access.cpp:33-38, config.hpp:25-35
ERRORS = [
    (lambda g, l, c: g["tensors"][1].update(size=0), "nonpositive size for tensor a01"),
    (lambda g, l, c: g["tensors"].append(dict(g["tensors"][0])), "duplicate tensor id x"),
    (lambda g, l, c: g["ops"].append(dict(g["ops"][0])), "duplicate op id f01"),
    (lambda g, l, c: g["ops"][1]["outputs"].append("a01"), "tensor a01 has more than one producer"),
    (lambda g, l, c: g["tensors"].append({"id": "zz", "size": 1, "kind": "interim"}), "tensor zz has no producing op"),
    (lambda g, l, c: l.pop("b02"), "missing latency entry for op b02"),
    (lambda g, l, c: l.update(f02=-1), "negative latency for op f02"),
    (lambda g, l, c: c.update(pcie_bandwidth=0), "pcie_bandwidth must be positive"),
    (lambda g, l, c: c.update(transfer_setup=-1), "transfer_setup must be nonnegative"),
    (lambda g, l, c: c.update(memory_budget=-5), "memory_budget must be nonnegative"),
    (lambda g, l, c: c.update(stall_epsilon=2.0), "stall_epsilon out of (0,1)"),
    (lambda g, l, c: c.update(max_swap_ratios={"cj": 1.5}), "max swap ratio for cj out of (0,1]"),
]


@pytest.mark.parametrize("mutate,msg", ERRORS, ids=[m for _, m in ERRORS])
def test_validation_errors(emu, mutate, msg):
    g, l = _chain()
    cfg = {"pcie_bandwidth": 4, "transfer_setup": 0, "memory_budget": 0}
    mutate(g, l, cfg)
    with pytest.raises(ValidationError) as e:
        emu.build_plan([(g, l)], cfg)
    assert str(e.value) == msg


def test_cycle_detected(emu):
    g = {"job_id": "cyc", "tensors": [{"id": "a", "size": 1, "kind": "interim"},
                                      {"id": "b", "size": 1, "kind": "interim"}],
         "ops": [{"id": "p", "kind": "f", "inputs": ["b"], "outputs": ["a"], "attributes": [], "phase": "forward_backward"},
                 {"id": "q", "kind": "f", "inputs": ["a"], "outputs": ["b"], "attributes": [], "phase": "forward_backward"}]}
    with pytest.raises(ValidationError, match="cycle detected in graph of job cyc"):
        emu.build_plan([(g, {"p": 1, "q": 1})], {"pcie_bandwidth": 1, "transfer_setup": 0, "memory_budget": 0})


def test_empty_build(emu):
    out = emu.build_plan([], {"pcie_bandwidth": 1, "transfer_setup": 0, "memory_budget": 0})
    assert out["plans_json"] == "null\n" and out["merged_peak_history"] == []


def test_groups_equal_single_calls(emu):
    from paper_2105_13336_b200 import configs as CF
    reqs = CF.requests("C3")
    cfgs = [r.config(CF.INITIAL_PEAK) for r in reqs]
    # one shared config: use the last request's budget for all three groups
    outs = emu.build_plan_groups([r.jobs for r in reqs], cfgs[-1])
    for r, o in zip(reqs, outs):
        single = emu.build_plan(r.jobs, cfgs[-1])
        assert o["plans_json"] == single["plans_json"]
        assert o["merged_peak_history"] == single["merged_peak_history"]


@pytest.mark.parametrize("shape", [(1, 2, 2), (3, 3, 2), (1, 24, 16)], ids=lambda s: f"M{s[0]}L{s[1]}H{s[2]}")
def test_c4_family_matches_oracle(emu, shape):
    """C4-family traces (GPT-2-medium generator), including jobs above one
    sort tile, against the restated oracle."""
    from helpers import ensure_oracle
    tslo = ensure_oracle()
    jobs = [W.c4_job(*shape)]
    init = sum(tslo.initial_peaks(jobs).values())
    cfg = {"pcie_bandwidth": 256, "transfer_setup": 1, "memory_budget": init * 7 // 10}
    got, want = emu.build_plan(jobs, cfg), tslo.build_plan(jobs, cfg)
    assert got["plans_json"] == want["plans_json"]
    assert got["reports_json"] == want["reports_json"]
    assert got["merged_peak_history"] == want["merged_peak_history"]


@pytest.mark.parametrize("case", golden("edge"), ids=lambda c: c["name"])
def test_edge_cases(emu, case):
    """Extreme inputs (tests/golden/make_edge_golden.py): single-op jobs, zero and
    constant latencies, budgets 0 / = peak / unbounded, ~2^40-byte tensors, 10^12-tick
    latencies, recompute-only setups, ratio-map errors, 40 jobs and all 64 C5 workloads
    in one build -- the reference's plans byte for byte, or its error text."""
    check_edge(emu.build_plan, case)


@pytest.mark.parametrize("block", range(6))
def test_live_reference_fuzz(emu, block):
    """The GPU suite's live differential fuzz (test_gpu_live_reference.py) through the
    emulation build: the same fresh seeds against the unmodified reference library."""
    from oracle import ref
    import test_gpu_live_reference as live
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    live.test_live_reference_fuzz(emu, ref, block)
