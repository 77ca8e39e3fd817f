"""INTEGRATION.md's `Algorithm::gpu` binding, compiled for real (oracle/gpu_dropin.cpp
against the unmodified reference objects and the engine library): the
reference's acceptance criteria 5-7 (proj/tests/acceptance.cpp:105-233) run
through it, its argument errors are the reference's exception types, and in
reference-order mode it reproduces plnmf::iterate() bit for bit."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "gpu_dropin"


@pytest.mark.gpu
@pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/gpu_dropin not built (needs /root/reference)")
def test_reference_acceptance_through_the_gpu_dropin(gpu):
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=900)
    print(res.stdout)
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    assert len(lines) == 5, res.stdout + res.stderr
    assert all(ln.startswith("PASS") for ln in lines), res.stdout
    assert res.returncode == 0
