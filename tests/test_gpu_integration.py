"""The reference's OWN acceptance checklist (test_acceptance.cpp, unmodified)
linked against the B200 planner through integration/memsched_orchestrator_b200.cpp
must report exactly what it reports against the reference's CPU orchestrator.
The binaries are built here by integration/Makefile (they need the reference
sources) and travel with the tree; the test skips when they are absent."""
import os
import re
import subprocess

import pytest

from helpers import ROOT

pytestmark = pytest.mark.gpu
BUILD = os.path.join(ROOT, "integration", "build")


def run(name):
    exe = os.path.join(BUILD, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (make -C integration)")
    p = subprocess.run(["stdbuf", "-o0", exe], capture_output=True, text=True, timeout=600, cwd=BUILD)
    return [re.sub(r"\(\d+\.\d+s\)", "", l) for l in p.stdout.splitlines() if l.startswith("[")]


def test_reference_acceptance_on_b200():
    ref = run("acceptance_ref")
    ours = run("acceptance_b200")
    assert len(ref) >= 8
    assert ours == ref
    assert all(l.startswith("[PASS]") for l in ours)
