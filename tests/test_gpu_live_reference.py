"""Live differential fuzz on the GPU against the UNMODIFIED reference.

oracle/_ref/libmemsched_ref.so is the reference's hot path compiled from its own
sources (oracle/Makefile); it travels with the repo, so the round-end GPU run can
compare random cases directly with it -- no fixture in between. Cases mix
the reference's own random_job (test_support.hpp) and generator families
(workload.cpp) with random bandwidth, setup, budget and coupled swap ratios.
150 cases use the fixed seeds 20000-20149 (outside every committed fixture);
50 more are drawn fresh on every run from a time-derived base seed (or
TSL_FUZZ_SEED), which the test prints and names in any failure.
"""
import json
import os
import random
import time

import pytest

pytestmark = pytest.mark.gpu

FAMS = ["vgg16", "resnet50", "inception_v3", "inception_v4", "densenet", "chain"]


@pytest.fixture(scope="module")
def planner():
    from paper_2105_13336_b200.planner import Planner
    return Planner(0)


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref (the reference compiled from its sources) is not built")
    return R


def _case(ref, seed):
    from paper_2105_13336_b200 import workload as W
    rnd = random.Random(seed)
    kind = rnd.random()
    jobs = []
    for k in range(rnd.choice([1, 1, 2, 3])):
        if kind < 0.5:
            g, lat = ref.random_job(seed * 10 + k)
            g["job_id"] = "r%d_%d" % (seed, k)
        else:
            g = W.generate_workload(rnd.choice(FAMS), rnd.choice([1, 8, 32]), 0, rnd.randint(2, 30), "j%d" % k)
            lat = W.true_latency_table(g, rnd.randint(0, 99))
        jobs.append((g, lat))
    peaks = ref.initial_peaks(jobs)
    cfg = {"pcie_bandwidth": rnd.choice([1, 2, 4, 16, 64, 256]), "transfer_setup": rnd.choice([0, 1, 3]),
           "memory_budget": sum(peaks.values()) * rnd.choice([3, 5, 7, 9]) // 10}
    if rnd.random() < 0.3:
        cfg["max_swap_ratios"] = {g["job_id"]: rnd.choice([0.1, 0.3, 0.5, 1.0]) for g, _ in jobs}
    return jobs, cfg


def _check_seeds(planner, ref, seeds):
    for seed in seeds:
        jobs, cfg = _case(ref, seed)
        try:
            text, res = ref.build_plan(jobs, cfg, repeats=1)
        except ref.ReferenceError_ as e:
            with pytest.raises(Exception) as got:
                planner.build_plan(jobs, cfg)
            assert str(got.value) == str(e), seed
            continue
        out = planner.build_plan(jobs, cfg)
        assert out["plans_json"] == text, f"seed {seed}: save_plans differs"
        assert out["merged_peak_history"] == res["merged_peak_history"], seed
        assert out["within_budget"] == res["within_budget"] and out["diagnostic"] == res["diagnostic"], seed
        for jid, rep in res["reports"].items():
            assert json.loads(out["reports_json"][jid]) == rep, f"seed {seed}: PeakReport of {jid}"


@pytest.mark.parametrize("block", range(6))
def test_live_reference_fuzz(planner, ref, block):
    """25 cases per block (fixed seeds 20000 + 25*block ...): save_plans text,
    PeakReports, merged history, budget flag and diagnostic equal the reference's."""
    _check_seeds(planner, ref, range(20000 + 25 * block, 20000 + 25 * (block + 1)))


def test_live_reference_fresh_seeds(planner, ref):
    """50 cases from a base seed drawn at run time (TSL_FUZZ_SEED to replay)."""
    base = int(os.environ.get("TSL_FUZZ_SEED", int(time.time()) % 1_000_000_000 + 10 ** 9))
    print(f"fresh fuzz base seed {base}")
    _check_seeds(planner, ref, range(base, base + 50))
