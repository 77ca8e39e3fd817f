"""The sharded engine's device kernels (plnmf_gpu_create_shard, the products
on gathered factors, the column-stepped W update) through the real driver.
Only one GPU is available here, so the ranks share cuda:0 over gloo (NCCL
refuses two ranks on one device); the multi-GPU launch differs only in the
process-group backend."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _helpers import Restated as R, rel_max
from paper_1904_07935_b200 import plnmf as P
from paper_1904_07935_b200.sharded import GpuShardBackend, ShardedNMF, ShardPlan, shard_blocks

pytestmark = pytest.mark.gpu
K, TILE, V, D = 24, 5, 1500, 900


def conditioned_state():
    m = P.synth_csr(V, D, 0.02, 9)
    w, ht = R.init_factors(V, D, K, seed=1)
    trp, tci, tval = R.transpose(V, D, m.row_ptr, m.col_idx, m.values)
    for _ in range(4):
        ht = R.update_h_reference(ht, R.spmm(D, V, trp, tci, tval, w), R.gram(w))
        w, _ = R.update_w_reference(w, R.spmm(V, D, m.row_ptr, m.col_idx, m.values, ht), R.gram(ht))
    return m, w, ht


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, w0, ht0 = conditioned_state()
        plan = ShardPlan(V, D, world)
        rows, cols = shard_blocks(m, plan, rank)
        be = GpuShardBackend(0, world, plan, rank, rows, cols, R.norm_sq(m.values), K)
        (v0, v1), (d0, d1) = plan.v_range(rank), plan.d_range(rank)
        be.set_local_factors(w0[v0:v1], ht0[d0:d1])
        drv = ShardedNMF(be, plan, rank, R.norm_sq(m.values))
        tr = drv.iterate(P.SolverConfig(rank=K, tile_size=TILE, max_iters=2, rel_tol=0.0), P.Algorithm.tiled)
        w, ht = be.get_local_factors()
        np.savez(os.path.join(out_dir, f"g{world}_r{rank}.npz"), w=w, ht=ht, init=tr.initial_error,
                 rel=np.array(tr.rel_errors))
        be.close()
    finally:
        dist.destroy_process_group()


def _run(world, tmp_path):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"g{world}_r{g}.npz") for g in range(world)]
    return np.concatenate([p["w"] for p in parts]), np.concatenate([p["ht"] for p in parts]), parts


def test_sharded_engine_matches_single_engine_and_oracle(gpu, tmp_path):
    w1, ht1, p1 = _run(1, tmp_path)
    w2, ht2, p2 = _run(2, tmp_path)
    m, w, ht = conditioned_state()
    # the unsharded engine on the same state
    eng = P.Engine(P.InputMatrix(m), K)
    eng.set_factors(P.FactorPair(w, ht))
    tr = eng.iterate(P.SolverConfig(rank=K, tile_size=TILE, max_iters=2, rel_tol=0.0), P.Algorithm.tiled)
    single = eng.get_factors()
    # the oracle's tiled iterations
    trp, tci, tval = R.transpose(V, D, m.row_ptr, m.col_idx, m.values)
    for _ in range(2):
        ht, _ = R.update_tiled(ht, R.gram(w), R.spmm(D, V, trp, tci, tval, w), TILE, is_w=False)
        w, _ = R.update_tiled(w, R.gram(ht), R.spmm(V, D, m.row_ptr, m.col_idx, m.values, ht), TILE, is_w=True)
    for wx, hx in [(w1, ht1), (w2, ht2), (single.w, single.ht)]:
        assert rel_max(w, wx) <= 1e-10 and rel_max(ht, hx) <= 1e-10
    assert rel_max(w1, w2) <= 1e-12 and rel_max(ht1, ht2) <= 1e-12
    assert abs(float(p1[0]["init"]) - tr.initial_error) <= 1e-13 * tr.initial_error
    assert np.allclose(p1[0]["rel"], [r.rel_error for r in tr.records], rtol=1e-10, atol=0)
    assert np.array_equal(p2[0]["rel"], p2[1]["rel"])
