"""paper_2105_13336_b200.workload (the trace generator used by bench.py and
the multi-GPU driver) reproduces the reference generator (workload.cpp)
byte for byte."""
import json

import pytest

from paper_2105_13336_b200 import workload as W


@pytest.mark.parametrize("fam,batch,depth", [("vgg16", 32, 0), ("resnet50", 64, 0), ("inception_v3", 32, 0),
                                             ("inception_v4", 32, 0), ("densenet", 32, 0), ("chain", 1, 3),
                                             ("chain", 8, 17), ("vgg16", 1, 0)])
def test_generator_matches_reference(fam, batch, depth):
    from oracle import ref
    if not ref.available():
        pytest.skip("reference library not built here (oracle/_ref)")
    g_ref, lat_ref = ref.generate_workload(fam, batch, 0, depth, "j", 13, 0.5)
    g = W.generate_workload(fam, batch, 0, depth, "j")
    # attributes are doubles in the reference document
    for o in g_ref["ops"]:
        o["attributes"] = [float(a) for a in o["attributes"]]
    assert json.dumps(g, sort_keys=True) == json.dumps(g_ref, sort_keys=True)
    assert W.true_latency_table(g, 13) == lat_ref


def test_config_sizes():
    from paper_2105_13336_b200 import configs as CF
    assert CF.requests("C1")[0].n_accesses == 175
    assert CF.requests("C2")[0].n_accesses == 565
    assert [r.n_accesses for r in CF.requests("C3")] == [536, 1201, 1376]
    assert sum(r.n_accesses for r in CF.requests("C5") if r.name.endswith(".7")) == 32550


def test_c4_generator_shape():
    """C4: GPT-2 medium, 24 layers, 16 heads, ~1 M accesses at
    the default 70 micro-batches; every moment parameter is read before its
    update (see workload.gpt2_workload)."""
    from paper_2105_13336_b200 import workload as W
    g = W.gpt2_workload(layers=2, heads=2, micro_batches=2)
    kinds = {t["id"]: t["kind"] for t in g["tensors"]}
    ups = [o for o in g["ops"] if o["kind"] == "update"]
    assert len(ups) == 2 * 12 * 3
    for o in ups:  # exactly one parameter in, one updated parameter out
        assert sum(kinds[t] == "parameter" for t in o["inputs"]) == 1
        assert [kinds[t] for t in o["outputs"]] == ["updated_parameter"]
    full = W.gpt2_workload()
    A = sum(len(o["inputs"]) + len(o["outputs"]) for o in full["ops"])
    assert 0.95e6 < A < 1.05e6
