"""The cold-start latency predictor (csrc/tsl_latency.cpp): LatencyPredictor
fit / predict / JSON (latency.cpp:11-149) and predict_latencies
(orchestrator.cpp:72-87).

The reference's fit needs Eigen, which is absent here, so `fit` is pinned to
what it computes -- the minimum-norm least-squares solution of the design
[features, usage^2, 1] (completeOrthogonalDecomposition().solve) -- through
numpy.linalg.lstsq, and to the reference unit tests' own expectations
(test_latency.cpp:65-140, on the reference's own sample generators). JSON
text, predict_latencies and the CLI's cold-start plan compare with the
UNMODIFIED reference (oracle/_ref)."""
import json
import math
import os

import numpy as np
import pytest

from helpers import GOLDEN, ensure_emu

from paper_2105_13336_b200.latency import LatencyPredictor
from paper_2105_13336_b200 import workload as W


@pytest.fixture(scope="module")
def lib():
    return ensure_emu()


@pytest.fixture(scope="module")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref is not built")
    return R


def _lstsq(samples, kind):
    rows = [(v, y) for k, v, y in samples if k == kind]
    X = np.array([list(v) + [v[-1] ** 2, 1.0] for v, _ in rows])
    y = np.array([y for _, y in rows])
    beta = np.linalg.lstsq(X, y, rcond=None)[0]
    fit = X @ beta
    ss_tot = float(((y - y.mean()) ** 2).sum())
    r2 = 1.0 - float(((y - fit) ** 2).sum()) / ss_tot if ss_tot > 0 else 1.0
    return beta, r2


def test_reference_unit_expectations(lib, ref):
    """test_latency.cpp:65-110 on the reference's own linear_samples."""
    p = LatencyPredictor.fit(ref.linear_samples(0.0, 1), lib)
    assert p.r2("k") >= 0.99
    assert p.predict("k", [100.0, 0.3]) == pytest.approx(205.0, rel=1e-9)
    assert LatencyPredictor.fit(ref.linear_samples(0.1, 7), lib).r2("k") >= 0.9
    back = LatencyPredictor.from_json(LatencyPredictor.fit(ref.linear_samples(0.0, 3), lib).to_json(), lib)
    q = LatencyPredictor.fit(ref.linear_samples(0.0, 3), lib)
    assert back.predict("k", [42.0, 0.7]) == pytest.approx(q.predict("k", [42.0, 0.7]))
    with pytest.raises(Exception, match="no fitted model for op kind zz"):
        back.predict("zz", [1.0])
    with pytest.raises(Exception, match="feature width mismatch for op kind k"):
        back.predict("k", [1.0, 2.0, 3.0])
    clamp = LatencyPredictor.fit([("k", [float(i), 0.5], -5.0 * i + 1.0) for i in range(1, 11)], lib)
    assert clamp.predict("k", [100.0, 0.5]) == 0.0


@pytest.mark.parametrize("samples,text", [
    ([("k", [1.0, 0.5], 7.0)], "insufficient samples for op kind k"),
    ([("k", [1.0, 0.5], 7.0), ("k", [1.0, 0.5], 8.0)], "degenerate (all-identical) features for op kind k"),
    ([("k", [1.0, 0.5], 7.0), ("k", [1.0], 8.0)], "inconsistent feature width for op kind k")])
def test_fit_rejects_degenerate_inputs(lib, samples, text):
    with pytest.raises(Exception) as e:
        LatencyPredictor.fit(samples, lib)
    assert str(e.value) == text


@pytest.mark.parametrize("family,noise", [("vgg16", 0.0), ("resnet50", 0.05), ("densenet", 0.1), ("chain", 0.0)])
def test_fit_is_the_min_norm_least_squares_solution(lib, ref, family, noise):
    """On the reference's generate_training_samples (workload.cpp:211-248):
    predictions and R^2 of the min-norm least-squares fit, rank-deficient
    kinds included (constant attribute columns duplicate the intercept)."""
    g = W.generate_workload(family, 8, 0, 6, "j")
    samples = ref.training_samples(g, 5, 12, noise)
    p = LatencyPredictor.fit(samples, lib)
    for kind in sorted({k for k, _, _ in samples}):
        beta, r2 = _lstsq(samples, kind)
        assert p.r2(kind) == pytest.approx(r2, rel=1e-6, abs=1e-9)
        for k, v, _ in samples:
            if k != kind:
                continue
            want = max(0.0, float(np.dot(list(v) + [v[-1] ** 2], beta[:-1]) + beta[-1]))
            assert p.predict(kind, v) == pytest.approx(want, rel=1e-6, abs=1e-6 * max(1.0, abs(want)))


def test_json_text_matches_reference(lib, ref):
    """to_json(from_json(doc)) == the reference's text for the same document
    (nlohmann's number formatting: integers, fractions, exponents, signs)."""
    rng = np.random.default_rng(3)
    vals = [0.0, 1.0, -2.5, 1e-7, 123456789.0, 1e16, 3.14159265358979, -1e-300, 2.5e21, 0.1, 1234567890123456.0]
    vals += list(rng.normal(size=20) * 10.0 ** rng.integers(-9, 18, size=20))
    doc = {"a": {"coefficients": vals[:12], "intercept": vals[12], "r2": 0.5},
           "b.k": {"coefficients": vals[13:], "intercept": -0.0, "r2": 1.0}}
    text = json.dumps(doc)
    assert LatencyPredictor.from_json(text, lib).to_json() == ref.predictor_roundtrip(text)
    samples = ref.training_samples(W.generate_workload("vgg16", 8, 0, 0, "v"), 1, 6, 0.05)
    fitted = LatencyPredictor.fit(samples, lib).to_json()
    assert LatencyPredictor.from_json(fitted, lib).to_json() == ref.predictor_roundtrip(fitted) == fitted


@pytest.mark.parametrize("usage", [0.0, 0.5, 0.9])
def test_predict_latencies_matches_reference(lib, ref, usage):
    g = W.generate_workload("inception_v3", 8, 0, 0, "i")
    doc = LatencyPredictor.fit(ref.training_samples(g, 2, 8, 0.0), lib).to_json()
    assert LatencyPredictor.from_json(doc, lib).predict_latencies(g, usage) == ref.predict_latencies(g, doc, usage)


def test_cli_cold_start_plan_matches_reference(lib, ref, tmp_path):
    """`memsched plan` with a predictor_file: Orchestrator::plan_cold_start,
    plans.json / peaks.json byte-identical to the reference CLI's."""
    import shutil
    from paper_2105_13336_b200 import cli
    from paper_2105_13336_b200.planner import Planner
    d = tmp_path / "scn"
    shutil.copytree(os.path.join(GOLDEN, "scenario_c3"), d)
    # one predictor per feature layout: the scenario keeps its vgg16 job
    g = json.loads((d / "vgg16.graph.json").read_text())
    (d / "predictor.json").write_text(LatencyPredictor.fit(ref.training_samples(g, 11, 6, 0.02), lib).to_json())
    doc = json.loads((d / "scenario.json").read_text())
    doc.pop("latency_file")
    doc["jobs"] = [j for j in doc["jobs"] if j["graph_file"] == "vgg16.graph.json"]
    doc["predictor_file"] = "predictor.json"
    (d / "scenario.json").write_text(json.dumps(doc))
    text = (d / "scenario.json").read_text()
    out = tmp_path / "out"
    assert cli.main(["plan", "--config", str(d / "scenario.json"), "--out", str(out)], planner=Planner(lib_path=lib)) == 0
    plans, peaks, diag = ref.plan_scenario(text, str(d))
    assert (out / "plans.json").read_text() == plans
    assert (out / "peaks.json").read_text() == peaks
