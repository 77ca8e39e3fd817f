"""Row/column-sharded FAST-HALS / PL-NMF over ranks.

One process per GPU.  Rank g owns the W rows [v_lo, v_hi) and the Ht rows
[d_lo, d_hi) of a balanced contiguous split, and A's matching CSR row block and
CSR-of-A^T row block.  Per iteration (the reference's order,
proj/src/solver.cpp:79-108):

  1. every rank broadcasts its W rows into the full W buffer   (W all-gather)
  2. R_g = A^T[d_lo:d_hi, :] W,  S_g = W_g^T W_g                (local kernels)
     S = S_0 + S_1 + ... in rank order                          (all-gather, ordered sum)
  3. H update on the local rows (row-local)
  4. Ht all-gather; P_g = A[v_lo:v_hi, :] Ht;  Q = ordered sum of Q_g
  5. W update, column by column: the tiled phase 2 for column t gives each
     rank's sum of squares; the world's partials are all-gathered and every
     rank normalises with sqrt(sum in rank order) — bit-identical on all ranks
     (proj/src/tiled.cpp:129-146 is the single-process original)
  6. error: <P,W> summed in rank order, <S,Q>, the Gram identity
     (proj/src/metrics.cpp:94-127), cadence / stop rule as iterate()

Collectives come from torch.distributed (NCCL on GPUs, gloo in the CPU tests);
compute comes from a backend: GpuShardBackend drives the CUDA engine through
the C-ABI (plnmf_gpu_create_shard & co.); the tests plug in a numpy backend
with the same interface.  Deterministic for a fixed world size.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L
from .plnmf import CsrMatrix, SolverConfig, _check, _f64p, _i64p


@dataclass
class ShardPlan:
    """Balanced contiguous split of V rows and D rows over `world` ranks."""
    v: int
    d: int
    world: int

    @staticmethod
    def _range(n, world, g):
        base, extra = divmod(n, world)
        lo = g * base + min(g, extra)
        return lo, lo + base + (1 if g < extra else 0)

    def v_range(self, g):
        return self._range(self.v, self.world, g)

    def d_range(self, g):
        return self._range(self.d, self.world, g)


def shard_blocks(a: CsrMatrix, plan: ShardPlan, rank: int):
    """(A[v_lo:v_hi, :], A^T[d_lo:d_hi, :]) as CSR with global indices; the
    transposed block keeps each row's entries in ascending source-row order
    (the order of transpose(), proj/src/csr_matrix.cpp:30-50)."""
    v_lo, v_hi = plan.v_range(rank)
    d_lo, d_hi = plan.d_range(rank)
    e0, e1 = a.row_ptr[v_lo], a.row_ptr[v_hi]
    rows = CsrMatrix(v_hi - v_lo, a.cols, a.row_ptr[v_lo:v_hi + 1] - e0, a.col_idx[e0:e1], a.values[e0:e1])
    row_of = np.repeat(np.arange(a.rows, dtype=np.int64), np.diff(a.row_ptr))
    sel = (a.col_idx >= d_lo) & (a.col_idx < d_hi)
    cols_sel, rows_sel, vals_sel = a.col_idx[sel], row_of[sel], a.values[sel]
    order = np.argsort(cols_sel, kind="stable")  # stable: rows stay ascending within a column
    counts = np.bincount(cols_sel - d_lo, minlength=d_hi - d_lo)
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    cols = CsrMatrix(d_hi - d_lo, a.rows, rp, rows_sel[order], vals_sel[order])
    return rows, cols


# ------------------------------------------------------------------------- GPU backend
class _DevArray:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class GpuShardBackend:
    """The CUDA engine in shard mode; buffers exposed to torch as CUDA tensors."""

    def __init__(self, device, world, plan: ShardPlan, rank, rows: CsrMatrix, cols: CsrMatrix, a_norm_sq, k):
        import torch
        self.torch, self.device = torch, device
        self._h = C.c_void_p()
        v_lo, v_hi = plan.v_range(rank)
        d_lo, d_hi = plan.d_range(rank)
        _check(L.lib().plnmf_gpu_create_shard(device, world, plan.v, plan.d, v_lo, v_hi, d_lo, d_hi, rows.nnz(),
                                              _i64p(rows.row_ptr), _i64p(rows.col_idx), _f64p(rows.values),
                                              cols.nnz(), _i64p(cols.row_ptr), _i64p(cols.col_idx),
                                              _f64p(cols.values), a_norm_sq, k, C.byref(self._h)))
        self.k = k
        self.W, self.Ht = self._buf(0), self._buf(1)
        self.W_full, self.Ht_full = self._buf(2), self._buf(3)
        self.S, self.Q = self._buf(4), self._buf(5)
        self.col_ss, self.world_ss = self._buf(8).view(-1), self._buf(9).view(-1)

    def _buf(self, which):
        ptr, r, c = C.c_void_p(), C.c_int64(), C.c_int64()
        _check(L.lib().plnmf_gpu_buffer(self._h, which, C.byref(ptr), C.byref(r), C.byref(c)))
        return self.torch.as_tensor(_DevArray(ptr.value, (r.value, c.value)), device=f"cuda:{self.device}")

    def sync(self):
        _check(L.lib().plnmf_gpu_synchronize(self._h))
        self.torch.cuda.synchronize(self.device)

    def set_local_factors(self, w_colmajor, ht_colmajor):
        w = np.asfortranarray(w_colmajor, dtype=np.float64)
        ht = np.asfortranarray(ht_colmajor, dtype=np.float64)
        _check(L.lib().plnmf_gpu_set_factors(self._h, _f64p(w), _f64p(ht)))

    def get_local_factors(self):
        w = np.zeros((self.W.shape[0], self.k), order="F")
        ht = np.zeros((self.Ht.shape[0], self.k), order="F")
        _check(L.lib().plnmf_gpu_get_factors(self._h, _f64p(w), _f64p(ht)))
        return w, ht

    def publish(self):
        _check(L.lib().plnmf_gpu_shard_publish(self._h))

    def products_h(self):
        _check(L.lib().plnmf_gpu_precompute_h_products(self._h))

    def products_w(self):
        _check(L.lib().plnmf_gpu_precompute_w_products(self._h))

    def update_h(self, cfg, algorithm):
        c = cfg.to_c()
        _check(L.lib().plnmf_gpu_update_h(self._h, C.byref(c), int(algorithm)))

    def w_begin(self, cfg):
        c = cfg.to_c()
        _check(L.lib().plnmf_gpu_w_begin(self._h, C.byref(c)))

    def w_column_step(self, cfg, t):
        c = cfg.to_c()
        _check(L.lib().plnmf_gpu_w_column_step(self._h, C.byref(c), t))

    def w_normalize(self, cfg, t):
        c = cfg.to_c()
        _check(L.lib().plnmf_gpu_w_normalize(self._h, C.byref(c), t))

    def w_phase3(self, cfg, b):
        c = cfg.to_c()
        _check(L.lib().plnmf_gpu_w_phase3(self._h, C.byref(c), b))

    def w_end(self):
        _check(L.lib().plnmf_gpu_w_end(self._h))

    def local_pw(self):
        out = C.c_double()
        _check(L.lib().plnmf_gpu_local_pw(self._h, C.byref(out)))
        return out.value

    def close(self):
        if self._h:
            L.lib().plnmf_gpu_destroy(self._h)
            self._h = C.c_void_p()


# ------------------------------------------------------------------------- driver
@dataclass
class ShardTrace:
    initial_error: float = 0.0
    rel_errors: List[float] = field(default_factory=list)


class ShardedNMF:
    """The iteration loop over a sharded backend (tiled W update)."""

    def __init__(self, backend, plan: ShardPlan, rank: int, a_norm_sq: float, group=None):
        import torch.distributed as dist
        self.b, self.plan, self.rank, self.a2, self.group, self.dist = backend, plan, rank, a_norm_sq, group, dist

    # -- collectives (deterministic: rank-ordered)
    def _gather_rows(self, full, ranges):
        for g in range(self.plan.world):
            lo, hi = ranges(g)
            if hi > lo:
                self.dist.broadcast(full[lo:hi], src=g, group=self.group)

    def _ordered_sum_into(self, t):
        parts = [self.b.torch.empty_like(t) for _ in range(self.plan.world)]
        self.dist.all_gather(parts, t.contiguous(), group=self.group)
        total = parts[0].clone()
        for p in parts[1:]:
            total = total + p
        t.copy_(total)

    def _ordered_scalar_sum(self, x: float) -> float:
        t = self.b.torch.tensor([x], dtype=self.b.torch.float64, device=self.b.W.device)
        parts = [self.b.torch.empty_like(t) for _ in range(self.plan.world)]
        self.dist.all_gather(parts, t, group=self.group)
        s = 0.0
        for p in parts:
            s = s + float(p.item())
        return s

    def _sync(self):
        self.b.sync()

    # -- steps
    def gather_w_products_h(self):
        self.b.publish()
        self._sync()
        self._gather_rows(self.b.W_full, self.plan.v_range)
        self._sync()
        self.b.products_h()  # R local, S partial
        self._sync()
        self._ordered_sum_into(self.b.S)
        self._sync()

    def gather_h_products_w(self):
        self.b.publish()
        self._sync()
        self._gather_rows(self.b.Ht_full, self.plan.d_range)
        self._sync()
        self.b.products_w()  # P local, Q partial
        self._sync()
        self._ordered_sum_into(self.b.Q)
        self._sync()

    def update_w(self, cfg: SolverConfig):
        k, T = cfg.rank, cfg.tile_size
        self.b.w_begin(cfg)
        for b0 in range(0, k, T):
            for t in range(b0, min(k, b0 + T)):
                self.b.w_column_step(cfg, t)
                self._sync()
                parts = [self.b.torch.empty_like(self.b.col_ss) for _ in range(self.plan.world)]
                self.dist.all_gather(parts, self.b.col_ss, group=self.group)
                self.b.world_ss.copy_(self.b.torch.cat(parts))
                self._sync()
                self.b.w_normalize(cfg, t)
            self.b.w_phase3(cfg, b0)
        self.b.w_end()

    def error(self):
        """Gram identity with the current products: S must be gram(W), P/Q of the current Ht."""
        pw = self._ordered_scalar_sum(self.b.local_pw())
        sq = float((self.b.S * self.b.Q).sum().item())
        frob = self.a2 - 2.0 * pw + sq
        frob = max(frob, 0.0)
        return math.sqrt(frob / self.a2)

    def iterate(self, cfg: SolverConfig, algorithm) -> ShardTrace:
        """proj/src/solver.cpp:53-115 for the tiled algorithm on the shards."""
        cfg.validate()
        if not (1 <= cfg.tile_size <= cfg.rank):
            raise ValueError("iterate: tiled algorithm needs tile_size in [1, rank]")
        tr = ShardTrace()
        self.gather_h_products_w()
        self.gather_w_products_h()  # S = gram(W) for the initial error (and R for iteration 1)
        tr.initial_error = prev = self.error()
        for it in range(1, cfg.max_iters + 1):
            self.b.update_h(cfg, algorithm)  # R, S of the current W are in place
            self.gather_h_products_w()
            self.update_w(cfg)
            self.gather_w_products_h()  # S = gram(new W), R for the next iteration
            if it % cfg.error_every == 0:
                rel = self.error()
                if not math.isfinite(rel):
                    raise RuntimeError(f"iterate: objective became non-finite at iteration {it}")
                tr.rel_errors.append(rel)
                if prev > 0.0 and abs(prev - rel) / prev < cfg.rel_tol:
                    break
                prev = rel
        return tr
