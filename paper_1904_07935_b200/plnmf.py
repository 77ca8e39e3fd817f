"""Python mirror of the reference's public interface, backed by the B200 engine.

Same names, argument meaning and error behaviour as the C++ reference
(proj/include/plnmf/*.hpp), so code written against ``plnmf::`` reads the same:

=====================================  ==========================================
reference (C++)                        here
=====================================  ==========================================
SolverConfig, validate()               SolverConfig, .validate()   config.hpp:11-22
Algorithm{reference, tiled}            Algorithm.reference / .tiled config.hpp:9
CsrMatrix, validate()                  CsrMatrix                    csr_matrix.hpp:10-21
DenseMatrix (col-major)                numpy float64, Fortran order dense_matrix.hpp:33
InputMatrix                            InputMatrix                  input_matrix.hpp:11-34
FactorPair {w, ht}                     FactorPair                   workspace.hpp:32-35
init_factors(v, d, cfg)                init_factors                 solver.hpp:29
iterate(a, factors, cfg, alg)          iterate (factors updated in place) solver.hpp:35-36
TilingPlan / plan_tiles                TilingPlan / plan_tiles      tiling.hpp:9-24
precompute_{h,w}_products, update_*    Engine methods               hals.hpp, tiled.hpp
relative_error_{gram,direct}           Engine.evaluate_error / .relative_error_direct
=====================================  ==========================================

Exceptions: std::invalid_argument -> InvalidArgument (a ValueError),
std::runtime_error -> NonFiniteObjective / RuntimeError, std::domain_error ->
DomainError (a ValueError, as std::domain_error is a logic_error).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ValueError):
    """std::domain_error"""


class NonFiniteObjective(RuntimeError):
    """std::runtime_error thrown by iterate() on a non-finite objective"""


class DeviceError(RuntimeError):
    """CUDA failure inside the engine (no reference counterpart)"""


class ParseError(RuntimeError):
    """plnmf::ParseError (proj/include/plnmf/matrix_market.hpp:12-19): "source:line: what" """

    @property
    def line(self) -> int:
        try:
            return int(str(self).rsplit(": ", 1)[0].rsplit(":", 1)[1])
        except (IndexError, ValueError):
            return 0


_STATUS = {1: InvalidArgument, 2: NonFiniteObjective, 3: DomainError, 4: DeviceError, 5: DeviceError, 6: ParseError}


def _check(status: int) -> None:
    if status != 0:
        msg = L.lib().plnmf_last_error().decode(errors="replace")
        raise _STATUS.get(status, RuntimeError)(msg)


def _f64p(a: np.ndarray):
    return a.ctypes.data_as(L.P_f64)


def _i64p(a: np.ndarray):
    return a.ctypes.data_as(L.P_i64)


class Algorithm(enum.IntEnum):
    reference = 0  # "fast-hals"
    tiled = 1      # "pl-nmf"


class Math(enum.IntEnum):
    exact = 0  # separate rn multiply/add in the reference's order (bitwise where the order is shared)
    fused = 1  # fma in the same order
    reference_order = 2  # exact + the reference's own W-norm and error-dot order (bitwise trajectories)
    tensor = 3  # exact, but dense-A products on the tensor cores (Ozaki u8 tcgen05 GEMMs)


@dataclass
class SolverConfig:
    rank: int = 2
    epsilon: float = 1e-16
    max_iters: int = 100
    rel_tol: float = 1e-6
    seed: int = 0
    error_every: int = 1
    deterministic: bool = False
    tile_size: int = 0

    def to_c(self) -> L.Config:
        return L.Config(int(self.rank), float(self.epsilon), int(self.max_iters), float(self.rel_tol),
                        int(self.seed) & (2**64 - 1), int(self.error_every), int(bool(self.deterministic)),
                        int(self.tile_size))

    def validate(self) -> None:
        c = self.to_c()
        _check(L.lib().plnmf_config_validate(C.byref(c)))


@dataclass
class TileRange:
    begin: int
    end: int

    def width(self) -> int:
        return self.end - self.begin


@dataclass
class TilingPlan:
    tile_size: int = 0
    tiles: List[TileRange] = field(default_factory=list)

    def gamma(self) -> int:
        return len(self.tiles)


def plan_tiles(k: int, tile_size: int) -> TilingPlan:
    """proj/src/tiling.cpp:8-18"""
    g = C.c_int64(0)
    _check(L.lib().plnmf_plan_tiles(k, tile_size, None, None, C.byref(g)))
    b = np.zeros(g.value, np.int64)
    e = np.zeros(g.value, np.int64)
    _check(L.lib().plnmf_plan_tiles(k, tile_size, _i64p(b), _i64p(e), C.byref(g)))
    return TilingPlan(tile_size, [TileRange(int(x), int(y)) for x, y in zip(b, e)])


@dataclass
class CsrMatrix:
    rows: int
    cols: int
    row_ptr: np.ndarray  # int64[rows+1]
    col_idx: np.ndarray  # int64[nnz], strictly increasing per row
    values: np.ndarray   # float64[nnz], finite, >= 0

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    def nnz(self) -> int:
        return int(self.values.size)

    def to_dense(self) -> np.ndarray:
        """densify (proj/src/matrix_market.cpp:237-242)."""
        m = np.zeros((self.rows, self.cols), order="F")
        for v in range(self.rows):
            for e in range(self.row_ptr[v], self.row_ptr[v + 1]):
                m[v, self.col_idx[e]] += self.values[e]
        return m


def synth_csr(rows: int, cols: int, density: float, seed: int = 20) -> CsrMatrix:
    """Synthetic non-negative CSR of SURVEY.md 8(d) (values U(0.1, 2.0), fp32-representable)."""
    rp = np.zeros(rows + 1, np.int64)
    nnz = C.c_int64(0)
    _check(L.lib().plnmf_synth_csr(rows, cols, density, seed, _i64p(rp), None, None, C.byref(nnz)))
    ci = np.zeros(nnz.value, np.int64)
    val = np.zeros(nnz.value, np.float64)
    _check(L.lib().plnmf_synth_csr(rows, cols, density, seed, _i64p(rp), _i64p(ci), _f64p(val), C.byref(nnz)))
    return CsrMatrix(rows, cols, rp, ci, val)


class InputMatrix:
    """A (V x D): a CsrMatrix or a dense array (kept column-major, as the reference)."""

    def __init__(self, m):
        if isinstance(m, CsrMatrix):
            self._csr, self._dense = m, None
        else:
            self._csr, self._dense = None, np.asfortranarray(np.asarray(m, dtype=np.float64))
            if self._dense.ndim != 2:
                raise InvalidArgument("DenseMatrix: expected a 2-D array")
        self._engines = {}

    def rows(self) -> int:
        return self._csr.rows if self._csr is not None else self._dense.shape[0]

    def cols(self) -> int:
        return self._csr.cols if self._csr is not None else self._dense.shape[1]

    def is_sparse(self) -> bool:
        return self._csr is not None

    def csr(self) -> CsrMatrix:
        return self._csr

    def dense(self) -> np.ndarray:
        return self._dense

    def engine(self, rank: int, device: int = 0, math: Math = Math.exact) -> "Engine":
        """The device copy of this matrix for a given rank (created once, cached)."""
        key = (rank, device)
        eng = self._engines.get(key)
        if eng is None:
            eng = Engine(self, rank, device)
            self._engines[key] = eng
        eng.set_math(math)
        return eng


@dataclass
class FactorPair:
    w: np.ndarray   # V x K, float64, column-major
    ht: np.ndarray  # D x K, float64, column-major


def init_factors(v: int, d: int, config: SolverConfig) -> FactorPair:
    """proj/src/solver.cpp:43-51 — bit-identical mt19937_64 stream, W first."""
    c = config.to_c()
    w = np.zeros((max(v, 0), max(config.rank, 0)), order="F")
    ht = np.zeros((max(d, 0), max(config.rank, 0)), order="F")
    _check(L.lib().plnmf_init_factors(v, d, C.byref(c), _f64p(w), _f64p(ht)))
    return FactorPair(w, ht)


@dataclass
class PhaseTimes:
    precompute_h: float = 0.0
    update_h: float = 0.0
    precompute_w: float = 0.0
    update_w: float = 0.0
    phase1: float = 0.0
    phase2: float = 0.0
    phase3: float = 0.0
    normalize: float = 0.0
    error_eval: float = 0.0

    @staticmethod
    def from_c(p) -> "PhaseTimes":
        return PhaseTimes(*(getattr(p, n) for n in PhaseTimes.__dataclass_fields__))


@dataclass
class TraceRecord:
    iteration: int
    rel_error: float
    elapsed_s: float
    phases: PhaseTimes


@dataclass
class ConvergenceTrace:
    initial_error: float = 0.0
    records: List[TraceRecord] = field(default_factory=list)
    totals: PhaseTimes = field(default_factory=PhaseTimes)
    total_seconds: float = 0.0
    update_macs: int = 0


@dataclass
class ErrorReport:
    frobenius_sq: float
    relative: float
    cancellation: bool = False


class _TraceBuf:
    def __init__(self, cap: int):
        self.recs = (L.TraceRecordC * max(cap, 1))()
        self.c = L.TraceC()
        self.c.capacity = max(cap, 1)
        self.c.records = self.recs

    def result(self) -> ConvergenceTrace:
        t = self.c
        recs = [TraceRecord(int(r.iteration), r.rel_error, r.elapsed_s, PhaseTimes.from_c(r.phases))
                for r in self.recs[: t.n_records]]
        return ConvergenceTrace(t.initial_error, recs, PhaseTimes.from_c(t.totals), t.total_seconds,
                                int(t.update_macs))


_PRODUCT = {"p": 0, "q": 1, "r": 2, "s": 3, "column_norms": 4}


class MatrixMarket:
    """A parsed Matrix Market file (read_matrix_market, proj/src/matrix_market.cpp):
    parsed on the host with the reference's rules and messages; the CSR is
    assembled on the device when an engine is created from it."""

    def __init__(self, path: Optional[str] = None, text: Optional[str] = None, source: str = "<string>"):
        self._h = C.c_void_p()
        if path is not None:
            _check(L.lib().plnmf_mm_read(str(path).encode(), C.byref(self._h)))
        else:
            _check(L.lib().plnmf_mm_read_string(text.encode(), source.encode(), C.byref(self._h)))
        r, c, n, sp = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _check(L.lib().plnmf_mm_info(self._h, C.byref(r), C.byref(c), C.byref(n), C.byref(sp)))
        self.rows, self.cols, self.entries, self.sparse = r.value, c.value, n.value, bool(sp.value)

    def engine(self, rank: int, device: int = 0) -> "Engine":
        h = C.c_void_p()
        _check(L.lib().plnmf_gpu_create_mm(device, self._h, rank, C.byref(h)))
        return Engine._adopt(h, rank)

    def __del__(self):
        try:
            if self._h:
                L.lib().plnmf_mm_free(self._h)
        except Exception:
            pass


def read_matrix_market(path: str) -> MatrixMarket:
    """proj/include/plnmf/matrix_market.hpp:25-29"""
    return MatrixMarket(path=path)


class Engine:
    """One device copy of A plus device-resident factors and workspace.

    The step API mirrors proj/include/plnmf/hals.hpp and tiled.hpp; products
    P, Q, R, S and the last column norms are readable (column-major numpy),
    like UpdateWorkspace's fields (workspace.hpp:39-55).
    """

    def __init__(self, a: InputMatrix, rank: int, device: int = 0):
        self._h = C.c_void_p()
        lib = L.lib()
        if a.is_sparse():
            m = a.csr()
            _check(lib.plnmf_gpu_create_csr(device, m.rows, m.cols, m.nnz(), _i64p(m.row_ptr),
                                            _i64p(m.col_idx), _f64p(m.values), rank, C.byref(self._h)))
        else:
            d = a.dense()
            _check(lib.plnmf_gpu_create_dense(device, d.shape[0], d.shape[1], _f64p(d), rank, C.byref(self._h)))
        self._info(rank)

    def _info(self, rank):
        self.rank = rank
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        n2 = C.c_double()
        _check(L.lib().plnmf_gpu_input_info(self._h, C.byref(r), C.byref(c), C.byref(n), C.byref(n2)))
        self.v, self.d, self.nnz, self.norm_sq = r.value, c.value, n.value, n2.value

    @classmethod
    def _adopt(cls, handle, rank) -> "Engine":
        eng = cls.__new__(cls)
        eng._h = handle
        eng._info(rank)
        return eng

    @classmethod
    def synthetic(cls, rows: int, cols: int, density: float, seed: int, rank: int, device: int = 0) -> "Engine":
        """An engine on the SURVEY.md 8(d) synthetic CSR generated on the device
        (the stream of synth_csr; nothing of A is built on the host)."""
        h = C.c_void_p()
        _check(L.lib().plnmf_gpu_create_synthetic(device, rows, cols, float(density), int(seed), rank, C.byref(h)))
        return cls._adopt(h, rank)

    def get_csr(self) -> CsrMatrix:
        rp = np.zeros(self.v + 1, np.int64)
        ci = np.zeros(max(self.nnz, 1), np.int64)
        val = np.zeros(max(self.nnz, 1))
        _check(L.lib().plnmf_gpu_get_csr(self._h, _i64p(rp), _i64p(ci), _f64p(val)))
        return CsrMatrix(self.v, self.d, rp, ci[: self.nnz], val[: self.nnz])

    def get_csr_rows(self, rows, transposed: bool = False) -> CsrMatrix:
        """The given rows of A (or of the device-built A^T) as a CSR."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rp = np.zeros(len(rows) + 1, np.int64)
        t = int(bool(transposed))
        _check(L.lib().plnmf_gpu_get_csr_rows(self._h, t, _i64p(rows), len(rows), _i64p(rp), None, None))
        ci = np.zeros(max(int(rp[-1]), 1), np.int64)
        val = np.zeros(max(int(rp[-1]), 1))
        _check(L.lib().plnmf_gpu_get_csr_rows(self._h, t, _i64p(rows), len(rows), _i64p(rp), _i64p(ci), _f64p(val)))
        return CsrMatrix(len(rows), self.v if transposed else self.d, rp, ci[: rp[-1]], val[: rp[-1]])

    def get_rows(self, name: str, rows) -> np.ndarray:
        """Rows of W / Ht / P / R (len(rows) x K)."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros((len(rows), self.rank))
        which = {"w": 0, "ht": 1, "p": 6, "r": 7}[name]
        _check(L.lib().plnmf_gpu_get_rows(self._h, which, _i64p(rows), len(rows), _f64p(out)))
        return out

    def close(self):
        if self._h:
            L.lib().plnmf_gpu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_math(self, math: Math) -> None:
        _check(L.lib().plnmf_gpu_set_math(self._h, int(math)))

    def force_streaming(self, on: bool = True) -> None:
        """Verification hook: tiled updates take the streaming plan (stream.cu)."""
        _check(L.lib().plnmf_gpu_force_streaming(self._h, int(bool(on))))

    def force_spmm_blocks(self, operand_rows: int) -> None:
        """Verification hook: column-blocked SpMMs (spmm.cu) with blocks of
        `operand_rows` operand rows (0: automatic, operands beyond ~96 MB)."""
        _check(L.lib().plnmf_gpu_force_spmm_blocks(self._h, int(operand_rows)))

    def set_reference_threads(self, n: int) -> None:
        """Math.reference_order: the reference's OpenMP team size (its tiled
        norm partials depend on it, proj/src/tiled.cpp:97-99)."""
        _check(L.lib().plnmf_gpu_set_reference_threads(self._h, int(n)))

    # ---- factors
    def set_factors(self, f: FactorPair) -> None:
        w = np.asfortranarray(f.w, dtype=np.float64)
        ht = np.asfortranarray(f.ht, dtype=np.float64)
        if w.shape != (self.v, self.rank) or ht.shape != (self.d, self.rank):
            raise InvalidArgument("iterate: factor dimensions do not match input and rank")
        _check(L.lib().plnmf_gpu_set_factors(self._h, _f64p(w), _f64p(ht)))

    def get_factors(self) -> FactorPair:
        w = np.zeros((self.v, self.rank), order="F")
        ht = np.zeros((self.d, self.rank), order="F")
        _check(L.lib().plnmf_gpu_get_factors(self._h, _f64p(w), _f64p(ht)))
        return FactorPair(w, ht)

    def init_factors(self, config: SolverConfig) -> None:
        c = config.to_c()
        _check(L.lib().plnmf_gpu_init_factors(self._h, C.byref(c)))

    # ---- step API
    def precompute_h_products(self) -> None:
        _check(L.lib().plnmf_gpu_precompute_h_products(self._h))

    def precompute_w_products(self) -> None:
        _check(L.lib().plnmf_gpu_precompute_w_products(self._h))

    def update_h(self, config: SolverConfig, algorithm: Algorithm) -> None:
        c = config.to_c()
        _check(L.lib().plnmf_gpu_update_h(self._h, C.byref(c), int(algorithm)))

    def update_w(self, config: SolverConfig, algorithm: Algorithm) -> None:
        c = config.to_c()
        _check(L.lib().plnmf_gpu_update_w(self._h, C.byref(c), int(algorithm)))

    def evaluate_error(self) -> ErrorReport:
        out = np.zeros(3)
        _check(L.lib().plnmf_gpu_evaluate_error(self._h, _f64p(out)))
        return ErrorReport(float(out[0]), float(out[1]), bool(out[2]))

    def relative_error_direct(self) -> ErrorReport:
        out = np.zeros(2)
        _check(L.lib().plnmf_gpu_relative_error_direct(self._h, _f64p(out)))
        return ErrorReport(float(out[0]), float(out[1]))

    def _shape(self, name: str):
        return {"p": (self.v, self.rank), "q": (self.rank, self.rank), "r": (self.d, self.rank),
                "s": (self.rank, self.rank), "column_norms": (self.rank,)}[name]

    def get_product(self, name: str) -> np.ndarray:
        out = np.zeros(self._shape(name), order="F")
        _check(L.lib().plnmf_gpu_get_product(self._h, _PRODUCT[name], _f64p(out)))
        return out

    def set_product(self, name: str, value: np.ndarray) -> None:
        arr = np.asfortranarray(value, dtype=np.float64)
        if arr.shape != self._shape(name):
            raise InvalidArgument(f"set_product: {name} must have shape {self._shape(name)}")
        _check(L.lib().plnmf_gpu_set_product(self._h, _PRODUCT[name], _f64p(arr)))

    # ---- loop
    def iterate(self, config: SolverConfig, algorithm: Algorithm) -> ConvergenceTrace:
        c = config.to_c()
        buf = _TraceBuf(config.max_iters)
        _check(L.lib().plnmf_gpu_iterate(self._h, C.byref(c), int(algorithm), C.byref(buf.c)))
        return buf.result()

    def run_iterations(self, config: SolverConfig, algorithm: Algorithm, n: int) -> float:
        c = config.to_c()
        ms = C.c_double()
        _check(L.lib().plnmf_gpu_run_iterations(self._h, C.byref(c), int(algorithm), n, C.byref(ms)))
        return ms.value

    def phase_ms(self) -> dict:
        """Device ms per step of the last run_iterations call (summed over its iterations)."""
        out = np.zeros(4)
        _check(L.lib().plnmf_gpu_phase_ms(self._h, _f64p(out)))
        return dict(zip(("precompute_h", "update_h", "precompute_w", "update_w"), map(float, out)))

    def best_integer_tile(self, config: SolverConfig, candidates=None):
        """GPU counterpart of best_integer_tile (proj/src/cost_model.cpp:131-142):
        the candidate T whose tiled H + W update from the current factors is
        fastest on this device (measured; the factors are left unchanged).
        Returns (best T, {T: update ms})."""
        c = config.to_c()
        cand = list(candidates) if candidates else []
        arr = (C.c_int32 * max(1, len(cand)))(*cand)
        times = (C.c_double * max(9, len(cand)))()
        best = C.c_int32()
        _check(L.lib().plnmf_gpu_best_integer_tile(self._h, C.byref(c), arr, len(cand), C.byref(best), times))
        if not cand:
            cand = [t for t in (1, 2, 4, 8, 12, 16, 20, 24, 32) if t <= config.rank]
        return best.value, {t: times[i] for i, t in enumerate(cand)}

    def time_kernel(self, config: SolverConfig, which: int, reps: int) -> float:
        c = config.to_c()
        ms = C.c_double()
        _check(L.lib().plnmf_gpu_time_kernel(self._h, C.byref(c), which, reps, C.byref(ms)))
        return ms.value

    def stats(self) -> dict:
        s = L.StatsC()
        _check(L.lib().plnmf_gpu_get_stats(self._h, C.byref(s)))
        return {"kernel_launches": int(s.kernel_launches), "persistent_ctas": int(s.persistent_ctas),
                "sm_count": int(s.sm_count), "device_bytes": int(s.device_bytes),
                "w_plan": int(s.w_plan), "h_plan": int(s.h_plan)}

    def synchronize(self) -> None:
        _check(L.lib().plnmf_gpu_synchronize(self._h))


def iterate(a: InputMatrix, factors: FactorPair, config: SolverConfig, algorithm: Algorithm,
            device: int = 0, math: Math = Math.exact) -> ConvergenceTrace:
    """proj/src/solver.cpp:53-115 on the GPU; `factors` is updated in place."""
    config.validate()
    if (factors.w.shape != (a.rows(), config.rank) or factors.ht.shape != (a.cols(), config.rank)):
        raise InvalidArgument("iterate: factor dimensions do not match input and rank")
    if algorithm == Algorithm.tiled and not (1 <= config.tile_size <= config.rank):
        raise InvalidArgument("iterate: tiled algorithm needs tile_size in [1, rank]")
    eng = a.engine(config.rank, device, math)
    w = np.asfortranarray(factors.w, dtype=np.float64).copy(order="F")
    ht = np.asfortranarray(factors.ht, dtype=np.float64).copy(order="F")
    c = config.to_c()
    buf = _TraceBuf(config.max_iters)
    _check(L.lib().plnmf_gpu_iterate_host(eng._h, C.byref(c), int(algorithm), _f64p(w), _f64p(ht), C.byref(buf.c)))
    factors.w, factors.ht = w, ht
    return buf.result()


def device_count() -> int:
    return int(L.lib().plnmf_gpu_device_count())
