"""TEST INFRASTRUCTURE ONLY — never imported by the product package.

ctypes wrappers of
  * ``liboracle.so``            the C restatement of the reference arithmetic
                                (plnmf_oracle.c; each function cites its reference file:line)
  * ``_ref/libplnmf_ref.so``    the UNMODIFIED reference library compiled from
                                /root/reference/proj/src plus ref_shim.cpp
                                (built by oracle/Makefile; travels to the GPU box
                                as a prebuilt file, /root/reference does not).

All matrices are numpy float64 in Fortran (column-major) order, exactly the
reference's DenseMatrix layout; CSR arrays are int64 / float64.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libplnmf_ref.so"

i64, u64, f64, cint = C.c_int64, C.c_uint64, C.c_double, C.c_int
P_i64, P_f64, P_u64 = C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_uint64)
vp = C.c_void_p


def f64p(a):
    return None if a is None else a.ctypes.data_as(P_f64)


def i64p(a):
    return None if a is None else a.ctypes.data_as(P_i64)


def F(a):
    return np.asfortranarray(a, dtype=np.float64)


# ============================================================ C restatement
_ora = None

_ORA_SIGS = {
    "ora_init_factors": (None, [i64, i64, i64, u64, f64, P_f64, P_f64]),
    "ora_transpose": (None, [i64, i64, i64, P_i64, P_i64, P_f64, P_i64, P_i64, P_f64]),
    "ora_spmm": (None, [i64, i64, P_i64, P_i64, P_f64, P_f64, i64, P_f64]),
    "ora_gram": (None, [i64, i64, P_f64, P_f64]),
    "ora_update_h_reference": (None, [i64, i64, f64, P_f64, P_f64, P_f64]),
    "ora_update_w_reference": (None, [i64, i64, f64, P_f64, P_f64, P_f64, P_f64]),
    "ora_update_tiled": (None, [i64, i64, i64, f64, cint, cint, cint, P_f64, P_f64, P_f64, P_f64]),
    "ora_relative_error_gram": (None, [f64, i64, i64, i64, P_f64, P_f64, P_f64, P_f64, P_f64]),
    "ora_relative_error_direct_csr": (None, [i64, i64, P_i64, P_i64, P_f64, f64, i64, P_f64, P_f64, P_f64]),
    "ora_norm_sq": (f64, [i64, P_f64]),
    "ora_factor_deviation": (f64, [i64, P_f64, P_f64]),
    "ora_synth_csr": (cint, [i64, i64, f64, u64, P_i64, P_i64, P_f64, P_i64]),
}


def synth_csr(rows, cols, density, seed=20):
    """The SURVEY.md 8(d) synthetic CSR (oracle/synth.c, the same stream as the
    engine's plnmf_synth_csr) as (row_ptr, col_idx, values) int64/int64/f64."""
    rp = np.zeros(rows + 1, np.int64)
    nnz = C.c_int64()
    if ora().ora_synth_csr(rows, cols, density, seed, i64p(rp), None, None, C.byref(nnz)):
        raise ValueError("synth_csr: bad arguments")
    ci = np.zeros(nnz.value, np.int64)
    val = np.zeros(nnz.value)
    ora().ora_synth_csr(rows, cols, density, seed, i64p(rp), i64p(ci), f64p(val), C.byref(nnz))
    return rp, ci, val


def ora():
    global _ora
    if _ora is None:
        if not ORACLE_SO.exists():
            raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle`")
        h = C.CDLL(str(ORACLE_SO))
        for n, (r, a) in _ORA_SIGS.items():
            getattr(h, n).restype = r
            getattr(h, n).argtypes = a
        _ora = h
    return _ora


class Restated:
    """The C restatement, one method per reference function."""

    @staticmethod
    def init_factors(v, d, k, seed=0, eps=1e-16):
        w = np.zeros((v, k), order="F")
        ht = np.zeros((d, k), order="F")
        ora().ora_init_factors(v, d, k, seed, eps, f64p(w), f64p(ht))
        return w, ht

    @staticmethod
    def transpose(rows, cols, rp, ci, val):
        nnz = len(val)
        trp = np.zeros(cols + 1, np.int64)
        tci = np.zeros(nnz, np.int64)
        tval = np.zeros(nnz)
        ora().ora_transpose(rows, cols, nnz, i64p(rp), i64p(ci), f64p(val), i64p(trp), i64p(tci), f64p(tval))
        return trp, tci, tval

    @staticmethod
    def spmm(rows, cols, rp, ci, val, x):
        x = F(x)
        y = np.zeros((rows, x.shape[1]), order="F")
        ora().ora_spmm(rows, cols, i64p(rp), i64p(ci), f64p(val), f64p(x), x.shape[1], f64p(y))
        return y

    @staticmethod
    def gram(m):
        m = F(m)
        g = np.zeros((m.shape[1], m.shape[1]), order="F")
        ora().ora_gram(m.shape[0], m.shape[1], f64p(m), f64p(g))
        return g

    @staticmethod
    def update_h_reference(ht, r, s, eps=1e-16):
        ht = F(ht).copy(order="F")
        ora().ora_update_h_reference(ht.shape[0], ht.shape[1], eps, f64p(ht), f64p(F(r)), f64p(F(s)))
        return ht

    @staticmethod
    def update_w_reference(w, p, q, eps=1e-16):
        w = F(w).copy(order="F")
        norms = np.zeros(w.shape[1])
        ora().ora_update_w_reference(w.shape[0], w.shape[1], eps, f64p(w), f64p(F(p)), f64p(F(q)), f64p(norms))
        return w, norms

    @staticmethod
    def update_tiled(mat, coeff, add, tile, eps=1e-16, is_w=True, nthreads=1):
        mat = F(mat).copy(order="F")
        norms = np.zeros(mat.shape[1])
        ora().ora_update_tiled(mat.shape[0], mat.shape[1], tile, eps, int(is_w), int(is_w), nthreads,
                               f64p(mat), f64p(F(coeff)), f64p(F(add)), f64p(norms))
        return mat, norms

    @staticmethod
    def relative_error_gram(a2, w, p, q, s):
        out = np.zeros(3)
        w = F(w)
        ora().ora_relative_error_gram(a2, w.shape[0], 0, w.shape[1], f64p(w), f64p(F(p)), f64p(F(q)),
                                      f64p(F(s)), f64p(out))
        return out

    @staticmethod
    def relative_error_direct_csr(rows, cols, rp, ci, val, a2, w, ht):
        out = np.zeros(2)
        w = F(w)
        ora().ora_relative_error_direct_csr(rows, cols, i64p(rp), i64p(ci), f64p(val), a2, w.shape[1], f64p(w),
                                            f64p(F(ht)), f64p(out))
        return out

    @staticmethod
    def norm_sq(val):
        val = np.ascontiguousarray(val, dtype=np.float64)
        return ora().ora_norm_sq(len(val), f64p(val))

    @staticmethod
    def factor_deviation(ref, other):
        ref, other = F(ref), F(other)
        return ora().ora_factor_deviation(ref.size, f64p(ref), f64p(other))


# ============================================================ compiled reference
_ref = None

_REF_SIGS = {
    "ref_last_error": (C.c_char_p, []),
    "ref_max_threads": (cint, []),
    "ref_set_threads": (None, [cint]),
    "ref_input_csr": (vp, [i64, i64, i64, P_i64, P_i64, P_f64]),
    "ref_input_dense": (vp, [i64, i64, P_f64]),
    "ref_input_free": (None, [vp]),
    "ref_input_norm_sq": (f64, [vp]),
    "ref_input_nnz": (i64, [vp]),
    "ref_read_mm": (cint, [C.c_char_p, P_i64, P_i64, P_i64, C.POINTER(cint), P_i64, P_i64, P_f64]),
    "ref_spmm": (cint, [i64, i64, i64, P_i64, P_i64, P_f64, P_f64, i64, P_f64]),
    "ref_transpose": (cint, [i64, i64, i64, P_i64, P_i64, P_f64, P_i64, P_i64, P_f64]),
    "ref_gram": (cint, [i64, i64, P_f64, P_f64]),
    "ref_gemm": (cint, [f64, P_f64, i64, i64, cint, P_f64, i64, i64, cint, f64, P_f64, i64, i64]),
    "ref_init_factors": (cint, [i64, i64, i64, u64, f64, P_f64, P_f64]),
    "ref_plan_tiles": (cint, [i64, i64, P_i64, P_i64, P_i64]),
    "ref_model_tile_size": (f64, [i64, u64]),
    "ref_best_integer_tile": (i64, [i64, i64, i64, u64]),
    "ref_session_create": (vp, [vp, i64]),
    "ref_session_free": (None, [vp]),
    "ref_session_get": (cint, [vp, cint, P_f64]),
    "ref_session_set": (cint, [vp, cint, P_f64]),
    "ref_session_macs": (u64, [vp]),
    "ref_session_phase_times": (None, [vp, P_f64]),
    "ref_session_precompute_h": (cint, [vp, P_f64, i64]),
    "ref_session_precompute_w": (cint, [vp, P_f64, i64]),
    "ref_session_update_h": (cint, [vp, P_f64, i64, f64, i64]),
    "ref_session_update_w": (cint, [vp, P_f64, i64, f64, i64]),
    "ref_init_new_accumulator": (cint, [P_f64, i64, i64, P_f64, P_f64, cint]),
    "ref_phase1": (cint, [P_f64, i64, i64, P_f64, i64, P_f64]),
    "ref_phase2": (cint, [P_f64, i64, i64, P_f64, P_f64, i64, i64, cint, f64, P_f64, P_f64]),
    "ref_phase3": (cint, [P_f64, i64, i64, P_f64, i64, i64]),
    "ref_relative_error_gram": (cint, [f64, P_f64, i64, P_f64, i64, i64, P_f64, P_f64, P_f64, P_f64]),
    "ref_relative_error_direct": (cint, [vp, P_f64, P_f64, i64, P_f64]),
    "ref_factor_deviation": (f64, [P_f64, P_f64, i64, i64]),
    "ref_iterate": (cint, [vp, P_f64, P_f64, i64, f64, i64, f64, u64, i64, i64, cint, P_f64, P_i64,
                           P_f64, P_f64, P_u64]),
}


class RefError(Exception):
    pass


def have_ref() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise ImportError(f"{REF_SO} missing: run `make -C oracle` where /root/reference exists")
        h = C.CDLL(str(REF_SO))
        for n, (r, a) in _REF_SIGS.items():
            getattr(h, n).restype = r
            getattr(h, n).argtypes = a
        _ref = h
    return _ref


def _rc(code):
    if code != 0:
        raise RefError(code, ref().ref_last_error().decode())


class RefInput:
    """plnmf::InputMatrix owned by the reference library."""

    def __init__(self, rows, cols, rp=None, ci=None, val=None, dense=None):
        if dense is not None:
            self.dense = F(dense)
            self.h = ref().ref_input_dense(rows, cols, f64p(self.dense))
        else:
            self.rp, self.ci, self.val = (np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int64),
                                          np.ascontiguousarray(val, np.float64))
            self.h = ref().ref_input_csr(rows, cols, len(self.val), i64p(self.rp), i64p(self.ci), f64p(self.val))
        if not self.h:
            raise RefError(1, ref().ref_last_error().decode())
        self.rows, self.cols = rows, cols

    @property
    def norm_sq(self):
        return ref().ref_input_norm_sq(self.h)

    def __del__(self):
        try:
            ref().ref_input_free(self.h)
        except Exception:
            pass


class RefSession:
    """InputMatrix + UpdateWorkspace of the reference, driven step by step
    (the lockstep pattern of `plnmf compare`, proj/tools/plnmf.cpp:317-327)."""

    PRODUCTS = {"p": 0, "q": 1, "r": 2, "s": 3, "column_norms": 4}

    def __init__(self, a: RefInput, k: int):
        self.a, self.k = a, k
        self.h = ref().ref_session_create(a.h, k)

    def __del__(self):
        try:
            ref().ref_session_free(self.h)
        except Exception:
            pass

    def _shape(self, name):
        return {"p": (self.a.rows, self.k), "q": (self.k, self.k), "r": (self.a.cols, self.k),
                "s": (self.k, self.k), "column_norms": (self.k,)}[name]

    def get(self, name):
        out = np.zeros(self._shape(name), order="F")
        _rc(ref().ref_session_get(self.h, self.PRODUCTS[name], f64p(out)))
        return out

    def set(self, name, value):
        _rc(ref().ref_session_set(self.h, self.PRODUCTS[name], f64p(F(value))))

    def precompute_h(self, w):
        _rc(ref().ref_session_precompute_h(self.h, f64p(F(w)), self.k))

    def precompute_w(self, ht):
        _rc(ref().ref_session_precompute_w(self.h, f64p(F(ht)), self.k))

    def update_h(self, ht, eps=1e-16, tile=0):
        ht = F(ht).copy(order="F")
        _rc(ref().ref_session_update_h(self.h, f64p(ht), self.k, eps, tile))
        return ht

    def update_w(self, w, eps=1e-16, tile=0):
        w = F(w).copy(order="F")
        _rc(ref().ref_session_update_w(self.h, f64p(w), self.k, eps, tile))
        return w

    def macs(self):
        return int(ref().ref_session_macs(self.h))

    def one_iteration(self, w, ht, eps=1e-16, tile=0):
        """run_one_iteration of proj/tests/test_engine_tiled.cpp:30-42."""
        self.precompute_h(w)
        ht = self.update_h(ht, eps, tile)
        self.precompute_w(ht)
        w = self.update_w(w, eps, tile)
        return w, ht


def ref_init_factors(v, d, k, seed=0, eps=1e-16):
    w = np.zeros((v, k), order="F")
    ht = np.zeros((d, k), order="F")
    _rc(ref().ref_init_factors(v, d, k, seed, eps, f64p(w), f64p(ht)))
    return w, ht


def ref_spmm(rows, cols, rp, ci, val, x):
    x = F(x)
    y = np.zeros((rows, x.shape[1]), order="F")
    _rc(ref().ref_spmm(rows, cols, len(val), i64p(rp), i64p(ci), f64p(val), f64p(x), x.shape[1], f64p(y)))
    return y


def ref_transpose(rows, cols, rp, ci, val):
    nnz = len(val)
    trp, tci, tval = np.zeros(cols + 1, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz)
    _rc(ref().ref_transpose(rows, cols, nnz, i64p(rp), i64p(ci), f64p(val), i64p(trp), i64p(tci), f64p(tval)))
    return trp, tci, tval


def ref_gram(m):
    m = F(m)
    g = np.zeros((m.shape[1], m.shape[1]), order="F")
    _rc(ref().ref_gram(m.shape[0], m.shape[1], f64p(m), f64p(g)))
    return g


def ref_plan_tiles(k, t):
    g = C.c_int64()
    _rc(ref().ref_plan_tiles(k, t, None, None, C.byref(g)))
    b, e = np.zeros(g.value, np.int64), np.zeros(g.value, np.int64)
    _rc(ref().ref_plan_tiles(k, t, i64p(b), i64p(e), C.byref(g)))
    return list(zip(b.tolist(), e.tolist()))


def ref_read_mm(path):
    rows, cols, nnz, sp = C.c_int64(), C.c_int64(), C.c_int64(), cint()
    _rc(ref().ref_read_mm(str(path).encode(), C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(sp), None, None, None))
    if sp.value:
        rp, ci, val = np.zeros(rows.value + 1, np.int64), np.zeros(nnz.value, np.int64), np.zeros(nnz.value)
        _rc(ref().ref_read_mm(str(path).encode(), C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(sp),
                              i64p(rp), i64p(ci), f64p(val)))
        return dict(rows=rows.value, cols=cols.value, rp=rp, ci=ci, val=val)
    val = np.zeros(nnz.value)
    _rc(ref().ref_read_mm(str(path).encode(), C.byref(rows), C.byref(cols), C.byref(nnz), C.byref(sp), None, None,
                          f64p(val)))
    return dict(rows=rows.value, cols=cols.value, dense=val.reshape((rows.value, cols.value), order="F"))


def ref_iterate(a: RefInput, w, ht, k, eps=1e-16, max_iters=100, rel_tol=1e-6, seed=0, error_every=1,
                tile=0, tiled=False):
    """plnmf::iterate; returns (w, ht, trace dict)."""
    w, ht = F(w).copy(order="F"), F(ht).copy(order="F")
    init = C.c_double()
    nrec = C.c_int64()
    recs = np.zeros((max(max_iters, 1), 12))
    totals = np.zeros(10)
    macs = C.c_uint64()
    _rc(ref().ref_iterate(a.h, f64p(w), f64p(ht), k, eps, max_iters, rel_tol, seed, error_every, tile, int(tiled),
                          C.byref(init), C.byref(nrec), f64p(recs), f64p(totals), C.byref(macs)))
    trace = dict(initial_error=init.value, records=recs[: nrec.value].copy(), total_seconds=totals[0],
                 totals=totals[1:].copy(), update_macs=int(macs.value))
    return w, ht, trace
