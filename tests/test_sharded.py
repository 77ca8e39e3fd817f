"""The sharded engine's host side on CPU: the row/column
partition, the shard blocks, and the rank bootstrap of
paper_1904_07935_b200.sharded.connect over torch.distributed (gloo,
world_size 2) — the IPC handles all-gathered in rank order and ||A||^2 chained
over the ranks, which must equal the reference's single serial sum bit for bit
(proj/src/input_matrix.cpp:15-20).  The device side runs in
test_sharded_gpu.py.  Plus the arithmetic the sharded iteration promises: with
the K x K Gram partials and the norm partials summed in rank order, one
iteration stays within ~1 ulp of the unsharded reference iteration."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from _helpers import Restated as R, rel_max
from paper_1904_07935_b200 import plnmf as P
from paper_1904_07935_b200.sharded import ShardPlan, connect, shard_blocks

V, D, K, TILE = 60, 45, 7, 3


def test_shard_plan_covers_rows_and_blocks_are_exact():
    plan = ShardPlan(10, 7, 3)
    assert [plan.v_range(g) for g in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert [plan.d_range(g) for g in range(3)] == [(0, 3), (3, 5), (5, 7)]
    m = P.synth_csr(40, 30, 0.2, 1)
    trp, tci, tval = R.transpose(40, 30, m.row_ptr, m.col_idx, m.values)
    dense = m.to_dense()
    for g in range(3):
        plan = ShardPlan(40, 30, 3)
        rows, cols = shard_blocks(m, plan, g)
        (v0, v1), (d0, d1) = plan.v_range(g), plan.d_range(g)
        assert np.array_equal(rows.to_dense(), dense[v0:v1])
        assert np.array_equal(cols.to_dense(), dense[:, d0:d1].T)
        # the transposed block keeps transpose()'s entry order
        e0, e1 = trp[d0], trp[d1]
        assert np.array_equal(cols.col_idx, tci[e0:e1]) and np.array_equal(cols.values, tval[e0:e1])


class HostShard:
    """The bootstrap surface of ShardEngine (ipc_handle, connect_handles,
    norm_sq_from, set_norm_sq) over a host row block: what connect() drives."""

    def __init__(self, m, world, rank):
        self.world, self.shard_rank = world, rank
        self.rows, _ = shard_blocks(m, ShardPlan(m.rows, m.cols, world), rank)
        self.handles = None
        self.norm_sq = None

    def ipc_handle(self):
        return bytes([self.shard_rank + 1]) * 64

    def connect_handles(self, handles):
        self.handles = list(handles)

    def norm_sq_from(self, start):
        acc = start
        for x in self.rows.values.tolist():
            acc += x * x
        return acc

    def set_norm_sq(self, value):
        self.norm_sq = value


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bootstrap_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = P.synth_csr(V, D, 0.15, 5)
        eng = HostShard(m, world, rank)
        connect(eng)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), handles=np.frombuffer(b"".join(eng.handles), np.uint8),
                 norm=eng.norm_sq)
    finally:
        dist.destroy_process_group()


def test_connect_gathers_handles_and_chains_the_norm_over_gloo(tmp_path):
    world = 2
    mp.spawn(_bootstrap_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    m = P.synth_csr(V, D, 0.15, 5)
    want = b"".join(bytes([g + 1]) * 64 for g in range(world))
    for g in range(world):
        out = np.load(tmp_path / f"r{g}.npz")
        assert out["handles"].tobytes() == want  # rank order
        assert float(out["norm"]) == R.norm_sq(m.values)  # the single serial sum, bit for bit


def conditioned_state():
    m = P.synth_csr(V, D, 0.15, 5)
    w, ht = R.init_factors(V, D, K, seed=2)
    trp, tci, tval = R.transpose(V, D, m.row_ptr, m.col_idx, m.values)
    for _ in range(6):
        ht = R.update_h_reference(ht, R.spmm(D, V, trp, tci, tval, w), R.gram(w))
        w, _ = R.update_w_reference(w, R.spmm(V, D, m.row_ptr, m.col_idx, m.values, ht), R.gram(ht))
    return m, w, ht


def sharded_iteration(m, w, ht, world):
    """One tiled iteration with the sharded engine's summation structure: the
    Gram products as rank-ordered sums of the ranks' partials, each W column
    norm as the rank-ordered sum of the ranks' sums of squares
    (csrc/shard_engine.cu, peer.cuh: world_sum); everything else is the
    reference's per-element order."""
    plan = ShardPlan(V, D, world)
    vr = [plan.v_range(g) for g in range(world)]
    dr = [plan.d_range(g) for g in range(world)]
    trp, tci, tval = R.transpose(V, D, m.row_ptr, m.col_idx, m.values)
    s = sum(R.gram(np.ascontiguousarray(w[slice(*x)])) for x in vr)
    ht, _ = R.update_tiled(ht, s, R.spmm(D, V, trp, tci, tval, w), TILE, is_w=False)
    q = sum(R.gram(np.ascontiguousarray(ht[slice(*x)])) for x in dr)
    p = R.spmm(V, D, m.row_ptr, m.col_idx, m.values, ht)
    # the W update with the norm partials per rank: phase 2 column by column
    nb = w * np.diag(q)[None, :]
    for tau in range(1, (K + TILE - 1) // TILE):
        b, e = tau * TILE, min(K, tau * TILE + TILE)
        for j in range(b):
            for kk in range(b, e):
                nb[:, j] = nb[:, j] + (-1.0 * q[kk, j]) * w[:, kk]
    for b in range(0, K, TILE):
        e = min(K, b + TILE)
        for t in range(b, e):
            acc = np.zeros(V)
            for kk in range(b, t):
                acc = acc + nb[:, kk] * q[kk, t]
            for kk in range(t, e):
                acc = acc + w[:, kk] * q[kk, t]
            nb[:, t] = np.maximum(1e-16, (nb[:, t] + p[:, t]) - acc)
            tot = 0.0
            for x in vr:
                tot += float(np.sum(nb[slice(*x), t] ** 2))
            nb[:, t] = np.maximum(1e-16, nb[:, t] / np.sqrt(tot))
        for c in range(e, K):
            for kk in range(b, e):
                nb[:, c] = nb[:, c] + (-1.0 * q[kk, c]) * nb[:, kk]
    return nb, ht


def test_sharded_summation_stays_within_an_ulp_of_the_reference_iteration():
    m, w, ht = conditioned_state()
    trp, tci, tval = R.transpose(V, D, m.row_ptr, m.col_idx, m.values)
    ht_ref, _ = R.update_tiled(ht, R.gram(w), R.spmm(D, V, trp, tci, tval, w), TILE, is_w=False)
    w_ref, _ = R.update_tiled(w, R.gram(ht_ref), R.spmm(V, D, m.row_ptr, m.col_idx, m.values, ht_ref), TILE,
                              is_w=True)
    for world in (1, 2, 3):
        w_sh, ht_sh = sharded_iteration(m, w, ht, world)
        assert rel_max(ht_ref, ht_sh) <= 1e-13 and rel_max(w_ref, w_sh) <= 1e-12
