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
