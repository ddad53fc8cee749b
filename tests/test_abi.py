"""The drop-in boundary: the CUDA planner library loads on a CPU-only host
and exports every entry point include/tensile_b200.h declares, with struct
layouts identical between C and the ctypes mirror (abi.py). No compute call
is made here (no GPU)."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from helpers import ROOT
from paper_2105_13336_b200 import abi

HEADER = os.path.join(ROOT, "include", "tensile_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tsl_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    import __graft_entry__ as ge
    return ge.build_cuda()


def test_exports_every_declared_symbol(lib_path):
    names = declared_functions()
    assert len(names) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(tsl_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, f"not exported: {missing}"
    lib = ctypes.CDLL(lib_path)  # loads without a GPU (cudart is linked statically)
    for n in names:
        assert hasattr(lib, n)


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_ctypes(tmp_path):
    structs = {"tsl_config": abi.TslConfig, "tsl_job_desc": abi.TslJobDesc, "tsl_job_view": abi.TslJobView,
               "tsl_plan_desc": abi.TslPlanDesc, "tsl_stats": abi.TslStats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for cname, ct in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in ct._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(c)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for cname, ct in structs.items():
        assert int(got[cname]) == ctypes.sizeof(ct), cname
        for fname, _ in ct._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(ct, fname).offset, f"{cname}.{fname}"


def test_no_device_fails_loudly(lib_path):
    """Without a CUDA device the planner refuses (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2105_13336_b200.planner import Planner, PlannerError
    with pytest.raises(PlannerError):
        Planner(0, lib_path=lib_path)
