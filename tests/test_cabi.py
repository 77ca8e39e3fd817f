"""The C-ABI boundary on CPU: the library loads, exports every symbol
include/plnmf_gpu.h declares, and its host-side logic (config validation,
tiling, init_factors, the synthetic generator, error mapping) behaves like the
reference — no compute call needs a GPU here."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from _helpers import Restated as R, bits_equal
from paper_1904_07935_b200 import _lib as L
from paper_1904_07935_b200 import plnmf as P

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "plnmf_gpu.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(plnmf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("plnmf_gpu_create_csr", "plnmf_gpu_iterate", "plnmf_gpu_iterate_host", "plnmf_init_factors",
                 "plnmf_gpu_precompute_h_products", "plnmf_gpu_update_w", "plnmf_gpu_evaluate_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (plnmf_[a-z0-9_]+)", out))
    for name in declared_functions():
        assert name in exported, f"{name} declared in include/plnmf_gpu.h but not exported"
        getattr(lib, name)  # resolvable through ctypes
        assert name in L.SIGNATURES, f"{name} missing from the ctypes binding"


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(L.LIB_PATH)], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_abi_version_and_defaults():
    lib = L.lib()
    assert lib.plnmf_gpu_abi_version() == 1
    c = L.Config()
    lib.plnmf_config_default(C.byref(c))
    # proj/include/plnmf/config.hpp:11-22
    assert (c.rank, c.epsilon, c.max_iters, c.rel_tol, c.seed, c.error_every, c.tile_size) == \
        (2, 1e-16, 100, 1e-6, 0, 1, 0)


@pytest.mark.parametrize("field,value,msg", [("rank", 0, "rank must be >= 1"), ("epsilon", 0.0, "epsilon must be > 0"),
                                             ("max_iters", -1, "max_iters must be >= 0"),
                                             ("rel_tol", -1e-3, "rel_tol must be >= 0"),
                                             ("error_every", 0, "error_every must be >= 1"),
                                             ("tile_size", 3, "tile_size must be in")])
def test_config_validation_messages(field, value, msg):
    """SolverConfig::validate, proj/src/config.cpp:7-15 (same messages)."""
    cfg = P.SolverConfig(rank=2)
    setattr(cfg, field, value)
    with pytest.raises(P.InvalidArgument, match=re.escape(msg)):
        cfg.validate()


def test_plan_tiles_layouts_and_errors():
    """test_engine_tiled.cpp:46-85"""
    assert [(t.begin, t.end) for t in P.plan_tiles(16, 16).tiles] == [(0, 16)]
    four = P.plan_tiles(16, 4)
    assert four.gamma() == 4 and all(t.width() == 4 for t in four.tiles)
    rem = P.plan_tiles(160, 15)
    assert rem.gamma() == 11 and rem.tiles[10].width() == 10 and rem.tiles[10].end == 160
    rng = np.random.default_rng(1)
    for _ in range(50):
        k = int(rng.integers(1, 201))
        t = int(rng.integers(1, k + 1))
        tiles = P.plan_tiles(k, t).tiles
        assert tiles[0].begin == 0 and tiles[-1].end == k
        assert all(a.end == b.begin for a, b in zip(tiles, tiles[1:]))
    for bad in [(8, 0), (8, 9)]:
        with pytest.raises(P.InvalidArgument):
            P.plan_tiles(*bad)


@pytest.mark.parametrize("v,d,k,seed,eps", [(12, 9, 4, 99, 1e-16), (20, 15, 3, 0, 1e-3), (1, 1, 1, 2**64 - 1, 0.5)])
def test_init_factors_bit_identical_to_reference_stream(v, d, k, seed, eps):
    """proj/src/solver.cpp:43-51; test_engine_reference.cpp:30-56"""
    f = P.init_factors(v, d, P.SolverConfig(rank=k, seed=seed, epsilon=eps))
    w, ht = R.init_factors(v, d, k, seed=seed, eps=eps)
    assert bits_equal(f.w, w) and bits_equal(f.ht, ht)
    assert f.w.min() >= eps and f.w.max() < 1.0
    g = P.init_factors(v, d, P.SolverConfig(rank=k, seed=seed + 1 if seed < 2**64 - 1 else 0, epsilon=eps))
    assert not bits_equal(f.w, g.w)
    with pytest.raises(P.InvalidArgument):
        P.init_factors(0, 5, P.SolverConfig(rank=k))


def test_synthetic_generator_is_deterministic_and_well_formed():
    a = P.synth_csr(5000, 3000, 0.004, 20)
    b = P.synth_csr(5000, 3000, 0.004, 20)
    assert (a.row_ptr == b.row_ptr).all() and (a.col_idx == b.col_idx).all() and bits_equal(a.values, b.values)
    assert a.row_ptr[0] == 0 and (np.diff(a.row_ptr) >= 0).all()
    for v in range(0, 5000, 97):
        cols = a.col_idx[a.row_ptr[v]:a.row_ptr[v + 1]]
        assert (np.diff(cols) > 0).all() and (cols < 3000).all()
    assert (a.values >= 0.1).all() and (a.values <= 2.0).all()
    assert bits_equal(a.values, a.values.astype(np.float32).astype(np.float64))  # fp32-representable
    expect = 5000 * 3000 * 0.004
    assert abs(a.nnz() - expect) < 5 * np.sqrt(expect)
    c = P.synth_csr(5000, 3000, 0.004, 21)
    assert c.nnz() != a.nnz() or not (c.col_idx == a.col_idx).all()
    full = P.synth_csr(3, 4, 1.0, 0)
    assert full.nnz() == 12


def test_engine_fails_loudly_without_a_gpu():
    """No CPU fallback: without a device, creating an engine is a CUDA error."""
    if P.device_count() > 0:
        pytest.skip("a GPU is present")
    m = P.synth_csr(10, 10, 0.5, 1)
    with pytest.raises(P.DeviceError, match="no CUDA device"):
        P.Engine(P.InputMatrix(m), 2)
    f = P.init_factors(10, 10, P.SolverConfig(rank=2))
    with pytest.raises(P.DeviceError):
        P.iterate(P.InputMatrix(m), f, P.SolverConfig(rank=2), P.Algorithm.reference)


def test_iterate_argument_checks_precede_device_work():
    m = P.synth_csr(10, 8, 0.5, 1)
    f = P.init_factors(10, 8, P.SolverConfig(rank=3))
    with pytest.raises(P.InvalidArgument, match="tile_size in \\[1, rank\\]"):
        P.iterate(P.InputMatrix(m), f, P.SolverConfig(rank=3, tile_size=0), P.Algorithm.tiled)
    with pytest.raises(P.InvalidArgument, match="factor dimensions"):
        P.iterate(P.InputMatrix(m), f, P.SolverConfig(rank=4), P.Algorithm.reference)
