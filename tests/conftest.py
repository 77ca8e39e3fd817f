"""Shared test setup.

`gpu`-marked tests are the parity tests proper: they drive the CUDA engine
through its C-ABI (libplnmf_gpu.so, via ctypes) and compare against the
oracle (oracle/: the C restatement and the compiled reference).  Everything
else runs on CPU.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); calls the engine through the C-ABI")


def _ensure_built():
    from paper_1904_07935_b200 import build as b
    if not b.LIB.exists():
        b.build()
    if not (ROOT / "oracle" / "liboracle.so").exists():
        b.build_oracle()


_ensure_built()


@pytest.fixture(scope="session")
def gpu():
    from paper_1904_07935_b200 import plnmf as P
    n = P.device_count()
    assert n > 0, "gpu tests need a CUDA device; the engine has no CPU fallback"
    return P
