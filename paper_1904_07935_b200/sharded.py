"""The sharded (multi-GPU) engine: host side.

One engine per GPU.  Rank g of `world` owns the W rows [v_lo, v_hi) and the Ht
rows [d_lo, d_hi) of balanced contiguous splits (ShardPlan), A's CSR row block
and the CSR of A^T's row block (shard_blocks, or generated on the device for the
synthetic workloads).  The iteration itself runs inside the engine
(csrc/shard_engine.cu): the factor and Gram all-gathers are stores into the
peers' windows and the per-column W norm (proj/src/tiled.cpp:129-146) is
exchanged inside the persistent W kernel, so once the ranks are connected the
ordinary Engine calls (iterate, run_iterations, the step API) run the sharded
iteration with no host synchronisation and no NCCL on the data path.

This module only sets the ranks up:
  * connect(engine, group): one process per GPU — the windows' CUDA IPC
    handles are all-gathered over torch.distributed (any backend) and opened;
    ||A||^2 is chained rank 0 -> world-1 (the reference's serial sum,
    proj/src/input_matrix.cpp:15-20, bit for bit) when the engine generated
    its blocks itself;
  * connect_local(engines): several ranks in one process (one GPU shared, or
    several GPUs with peer access).
Every rank must then make the same engine calls in the same order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib as L
from .plnmf import CsrMatrix, Engine, _check, _f64p, _i64p

IPC_HANDLE_BYTES = 64


@dataclass
class ShardPlan:
    """Balanced contiguous split of V rows and D rows over `world` ranks (the
    engine's rule: the first n % world ranks get one row more)."""
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


class ShardEngine(Engine):
    """One rank of the sharded engine; after connecting, the Engine methods
    (set/get/init_factors — local rows —, iterate, run_iterations, the step
    API, evaluate_error) run the sharded iteration."""

    @classmethod
    def from_csr(cls, a: CsrMatrix, world: int, rank: int, k: int, device: int = 0,
                 a_norm_sq: Optional[float] = None) -> "ShardEngine":
        """Rank `rank` holding its blocks of the host matrix `a`."""
        plan = ShardPlan(a.rows, a.cols, world)
        rows, cols = shard_blocks(a, plan, rank)
        if a_norm_sq is None:
            n2 = 0.0  # the reference's serial order (input_matrix.cpp:15-20)
            for x in a.values.tolist():
                n2 += x * x
            a_norm_sq = n2
        h = C.c_void_p()
        _check(L.lib().plnmf_gpu_create_shard(device, world, rank, a.rows, a.cols, rows.nnz(), _i64p(rows.row_ptr),
                                              _i64p(rows.col_idx), _f64p(rows.values), cols.nnz(),
                                              _i64p(cols.row_ptr), _i64p(cols.col_idx), _f64p(cols.values),
                                              float(a_norm_sq), k, C.byref(h)))
        return cls._adopt(h, k)

    @classmethod
    def generate(cls, rows: int, cols: int, density: float, seed: int, k: int, world: int, rank: int,
                 device: int = 0) -> "ShardEngine":
        """Rank `rank` of the synthetic matrix of synth_csr(rows, cols, density,
        seed), its row and column blocks generated on the device.  ||A||^2 is set
        by connect() / connect_local(chain_norm=True) (chained over the ranks)."""
        h = C.c_void_p()
        _check(L.lib().plnmf_gpu_create_shard_synthetic(device, world, rank, rows, cols, float(density), int(seed),
                                                        k, C.byref(h)))
        return cls._adopt(h, k)

    def _info(self, rank):
        super()._info(rank)
        w, g = C.c_int32(), C.c_int32()
        r = [C.c_int64() for _ in range(4)]
        _check(L.lib().plnmf_gpu_shard_info(self._h, C.byref(w), C.byref(g), *[C.byref(x) for x in r]))
        self.world, self.shard_rank = w.value, g.value
        self.v_range = (r[0].value, r[1].value)
        self.d_range = (r[2].value, r[3].value)

    def norm_sq_from(self, start: float) -> float:
        out = C.c_double()
        _check(L.lib().plnmf_gpu_shard_norm_sq(self._h, float(start), C.byref(out)))
        return out.value

    def set_norm_sq(self, value: float) -> None:
        _check(L.lib().plnmf_gpu_shard_set_norm_sq(self._h, float(value)))
        self.norm_sq = float(value)

    def set_timeout(self, seconds: float) -> None:
        _check(L.lib().plnmf_gpu_shard_set_timeout(self._h, float(seconds)))

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(L.lib().plnmf_gpu_shard_ipc_handle(self._h, buf))
        return buf.raw

    def connect_handles(self, handles: Sequence[bytes]) -> None:
        if len(handles) != self.world or any(len(h) != IPC_HANDLE_BYTES for h in handles):
            raise ValueError("connect: one 64-byte IPC handle per rank, in rank order")
        _check(L.lib().plnmf_gpu_shard_connect(self._h, b"".join(handles)))


def connect(engine: ShardEngine, group=None, chain_norm: bool = True) -> None:
    """Connects this process's rank to the others of `group` (torch.distributed,
    one process per GPU): all-gathers the windows' IPC handles and opens them;
    with chain_norm, sets ||A||^2 = the serial sum over all ranks' rows."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world != engine.world or rank != engine.shard_rank:
        raise ValueError("connect: the process group does not match the engine's world / rank")
    handles = [None] * world
    dist.all_gather_object(handles, engine.ipc_handle(), group=group)
    if world > 1:
        engine.connect_handles(handles)
    if chain_norm:
        acc = 0.0
        for g in range(world):
            obj = [engine.norm_sq_from(acc) if g == rank else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, g) if group is not None else g,
                                       group=group)
            acc = obj[0]
        engine.set_norm_sq(acc)
    dist.barrier(group)


def connect_local(engines: Sequence[ShardEngine], chain_norm: bool = False) -> None:
    """Connects the ranks 0..world-1 held by this process (several ranks on one
    GPU share its SMs and need CUDA_MODULE_LOADING=EAGER; several GPUs need peer
    access).  The ranks then use each other's windows: close them together."""
    arr = (C.c_void_p * len(engines))(*[e._h for e in engines])
    _check(L.lib().plnmf_gpu_shard_connect_local(arr, len(engines)))
    if chain_norm:
        acc = 0.0
        for e in engines:
            acc = e.norm_sq_from(acc)
        for e in engines:
            e.set_norm_sq(acc)
