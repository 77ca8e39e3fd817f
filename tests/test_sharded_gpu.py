"""The sharded engine (csrc/shard_engine.cu) on the device: several ranks in
one process share cuda:0 (plnmf_gpu_shard_connect_local gives each rank's
persistent W kernel an equal share of the SMs), each driven from its own host
thread, exactly as one process per GPU would drive them.  The ranks exchange
everything through their peer windows — the factor / Gram all-gathers and the
per-column W norm inside the persistent kernel — so these tests run the same
device code as the multi-GPU launch; only the window mapping differs (the same
device's pointers instead of CUDA IPC over NVLink).  Ranks that share a GPU
wait on one another's kernels, which CUDA's lazy module loading can deadlock,
so every case runs in a fresh process with CUDA_MODULE_LOADING=EAGER.

Checked against the oracle's restatement of the sharded arithmetic (the
reference's per-element order everywhere; the K x K Gram partials and the
error partial summed in rank order), bit for bit where the engine promises it
(R, S, P, Q, Ht), and W to 1e-12 (norm partial order)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))  # also run as a script (the eager subprocess)
from _helpers import Restated as R, bits_equal, rel_max
from paper_1904_07935_b200 import plnmf as P
from paper_1904_07935_b200.sharded import ShardEngine, ShardPlan, connect_local

pytestmark = pytest.mark.gpu
K, TILE, V, D = 24, 5, 1500, 900


def conditioned_state(v=V, d=D, k=K, density=0.02, seed=9):
    """A few fast-hals iterations from the seed: past iteration 1's collapse."""
    m = P.synth_csr(v, d, density, seed)
    w, ht = R.init_factors(v, d, k, seed=1)
    trp, tci, tval = R.transpose(v, d, m.row_ptr, m.col_idx, m.values)
    for _ in range(4):
        ht = R.update_h_reference(ht, R.spmm(d, v, trp, tci, tval, w), R.gram(w))
        w, _ = R.update_w_reference(w, R.spmm(v, d, m.row_ptr, m.col_idx, m.values, ht), R.gram(ht))
    return m, w, ht


def on_ranks(engines, fn):
    """fn(engine, g) on every rank concurrently (one host thread per rank)."""
    with ThreadPoolExecutor(len(engines)) as ex:
        return list(ex.map(lambda g: fn(engines[g], g), range(len(engines))))


def make_ranks(m, world, k=K):
    engines = [ShardEngine.from_csr(m, world, g, k) for g in range(world)]
    connect_local(engines)
    return engines


def ordered_sum(parts):
    s = parts[0].copy()
    for x in parts[1:]:
        s = s + x
    return s


def case_step_products_and_updates(world):
    # uneven splits (padded window rows, remapped indices) and an odd K (8-byte push path)
    V, D, K = 1501, 899, 23
    m, w0, ht0 = conditioned_state(V, D, K)
    plan = ShardPlan(V, D, world)
    vr = [plan.v_range(g) for g in range(world)]
    dr = [plan.d_range(g) for g in range(world)]
    engines = make_ranks(m, world, K)
    if world == 3:  # the column-blocked SpMM on the padded window rows (small blocks, many passes)
        for e in engines:
            e.force_spmm_blocks(97)
    on_ranks(engines, lambda e, g: e.set_factors(P.FactorPair(w0[slice(*vr[g])], ht0[slice(*dr[g])])))
    cfg = P.SolverConfig(rank=K, tile_size=TILE)
    trp, tci, tval = R.transpose(V, D, m.row_ptr, m.col_idx, m.values)

    # R = A^T W (local rows, bitwise) and S = sum_g gram(W_g) in rank order (bitwise)
    on_ranks(engines, lambda e, g: e.precompute_h_products())
    r_full = R.spmm(D, V, trp, tci, tval, w0)
    s_sh = ordered_sum([R.gram(np.ascontiguousarray(w0[slice(*vr[g])])) for g in range(world)])
    for g, e in enumerate(engines):
        assert bits_equal(e.get_product("r"), r_full[slice(*dr[g])])
        assert bits_equal(e.get_product("s"), s_sh)

    # H update (row-local): bitwise
    on_ranks(engines, lambda e, g: e.update_h(cfg, P.Algorithm.tiled))
    ht1, _ = R.update_tiled(ht0, s_sh, r_full, TILE, is_w=False)
    for g, e in enumerate(engines):
        assert bits_equal(e.get_factors().ht, ht1[slice(*dr[g])])

    # P = A Ht on the gathered Ht (bitwise), Q in rank order (bitwise)
    on_ranks(engines, lambda e, g: e.precompute_w_products())
    p_full = R.spmm(V, D, m.row_ptr, m.col_idx, m.values, ht1)
    q_sh = ordered_sum([R.gram(np.ascontiguousarray(ht1[slice(*dr[g])])) for g in range(world)])
    for g, e in enumerate(engines):
        assert bits_equal(e.get_product("p"), p_full[slice(*vr[g])])
        assert bits_equal(e.get_product("q"), q_sh)

    # W update: the norm of every column exchanged across the ranks inside the kernel
    on_ranks(engines, lambda e, g: e.update_w(cfg, P.Algorithm.tiled))
    w1, norms = R.update_tiled(w0, q_sh, p_full, TILE, is_w=True)
    w_got = np.concatenate([e.get_factors().w for e in engines])
    assert rel_max(w1, w_got) <= 1e-12
    got_norms = [e.get_product("column_norms") for e in engines]
    assert all(bits_equal(got_norms[0], x) for x in got_norms[1:])  # every rank used the same norms
    assert np.max(np.abs(got_norms[0] - norms) / norms) <= 1e-13

    # the error: every rank the same bits, the oracle's value to 1e-12
    reps = on_ranks(engines, lambda e, g: e.evaluate_error())
    assert all(r.relative == reps[0].relative for r in reps)
    e_ref = R.relative_error_gram(R.norm_sq(m.values), w1, p_full, q_sh, R.gram(w1))[1]
    assert abs(reps[0].relative - e_ref) <= 1e-12 * e_ref
    for e in engines:
        e.close()


def case_iterate_matches_single_engine(world):
    m, w0, ht0 = conditioned_state()
    plan = ShardPlan(V, D, world)
    cfg = P.SolverConfig(rank=K, tile_size=TILE, max_iters=3, rel_tol=0.0)
    single = P.Engine(P.InputMatrix(m), K)
    single.set_factors(P.FactorPair(w0, ht0))
    tr1 = single.iterate(cfg, P.Algorithm.tiled)
    f1 = single.get_factors()

    engines = make_ranks(m, world)
    if world == 3:  # H on the streaming plan too: the Ht all-gather fused into that kernel
        for e in engines:
            e.force_streaming(True)
    on_ranks(engines, lambda e, g: e.set_factors(P.FactorPair(w0[slice(*plan.v_range(g))],
                                                              ht0[slice(*plan.d_range(g))])))
    trs = on_ranks(engines, lambda e, g: e.iterate(cfg, P.Algorithm.tiled))
    for tr in trs[1:]:  # every rank reports the same trajectory, bit for bit
        assert tr.initial_error == trs[0].initial_error
        assert [r.rel_error for r in tr.records] == [r.rel_error for r in trs[0].records]
    assert abs(trs[0].initial_error - tr1.initial_error) <= 1e-13 * tr1.initial_error
    for a, b in zip(trs[0].records, tr1.records):
        assert abs(a.rel_error - b.rel_error) <= 1e-10 * b.rel_error
    w = np.concatenate([e.get_factors().w for e in engines])
    ht = np.concatenate([e.get_factors().ht for e in engines])
    assert rel_max(f1.w, w) <= 1e-10 and rel_max(f1.ht, ht) <= 1e-10
    # run_iterations: the same sharded iteration without error evaluation or host syncs
    ms = on_ranks(engines, lambda e, g: e.run_iterations(cfg, P.Algorithm.tiled, 2))
    assert all(x > 0 for x in ms)
    for e in engines:
        e.close()


def case_fast_hals_sharded(world):
    """The reference (fast-hals) algorithm on the sharded engine: update_w_reference's column
    norms exchanged between the ranks inside its persistent kernel, H row-local."""
    m, w0, ht0 = conditioned_state()
    plan = ShardPlan(V, D, world)
    cfg = P.SolverConfig(rank=K, max_iters=3, rel_tol=0.0)
    single = P.Engine(P.InputMatrix(m), K)
    single.set_factors(P.FactorPair(w0, ht0))
    tr1 = single.iterate(cfg, P.Algorithm.reference)
    f1 = single.get_factors()
    engines = make_ranks(m, world)
    on_ranks(engines, lambda e, g: e.set_factors(P.FactorPair(w0[slice(*plan.v_range(g))],
                                                              ht0[slice(*plan.d_range(g))])))
    trs = on_ranks(engines, lambda e, g: e.iterate(cfg, P.Algorithm.reference))
    for tr in trs[1:]:
        assert [r.rel_error for r in tr.records] == [r.rel_error for r in trs[0].records]
    for a, b in zip(trs[0].records, tr1.records):
        assert abs(a.rel_error - b.rel_error) <= 1e-10 * b.rel_error
    w = np.concatenate([e.get_factors().w for e in engines])
    ht = np.concatenate([e.get_factors().ht for e in engines])
    assert rel_max(f1.w, w) <= 1e-10 and rel_max(f1.ht, ht) <= 1e-10
    for e in engines:
        e.close()


def case_generated_shards(world):
    """The C5 path: each rank generates its row block and its A^T block on the
    device; products from init_factors equal those of shards built from the
    host generator's CSR, and ||A||^2 chained over the ranks equals the serial sum."""
    v, d, dens, seed, k = 3000, 2200, 0.01, 20, 16
    m = P.synth_csr(v, d, dens, seed)
    gen = [ShardEngine.generate(v, d, dens, seed, k, world, g) for g in range(world)]
    connect_local(gen, chain_norm=True)
    host = make_ranks(m, world, k)
    assert all(e.norm_sq == R.norm_sq(m.values) for e in gen)
    cfg = P.SolverConfig(rank=k, tile_size=4, seed=3)
    full = P.init_factors(v, d, cfg)
    plan = ShardPlan(v, d, world)
    out = {}
    for name, engs in (("gen", gen), ("host", host)):
        on_ranks(engs, lambda e, g: e.init_factors(cfg))
        for g, e in enumerate(engs):
            f = e.get_factors()
            assert bits_equal(f.w, full.w[slice(*plan.v_range(g))])
            assert bits_equal(f.ht, full.ht[slice(*plan.d_range(g))])
        on_ranks(engs, lambda e, g: (e.precompute_h_products(), e.update_h(cfg, P.Algorithm.tiled),
                                     e.precompute_w_products()))
        out[name] = [(e.get_product("r"), e.get_product("p"), e.get_product("s")) for e in engs]
    for a, b in zip(out["gen"], out["host"]):
        assert all(bits_equal(x, y) for x, y in zip(a, b))
    for e in gen + host:
        e.close()


def case_missing_rank_times_out(world):
    m, w0, ht0 = conditioned_state(400, 300, 8, 0.05, 3)
    engines = make_ranks(m, world, 8)
    engines[0].set_timeout(0.5)
    plan = ShardPlan(400, 300, 2)
    engines[0].set_factors(P.FactorPair(w0[slice(*plan.v_range(0))], ht0[slice(*plan.d_range(0))]))
    with pytest.raises(P.DeviceError, match="did not arrive"):
        engines[0].precompute_h_products()  # rank 1 never pushed its W rows
    for e in engines:
        e.close()


def case_ipc_rank(world):
    """One rank of a multi-process run (one process per rank, all on cuda:0):
    torch.distributed (gloo) all-gathers the windows' CUDA IPC handles
    (sharded.connect) — the launch path of one process per GPU.  Without MPS
    the ranks' contexts time-slice the GPU, so the in-kernel waits span
    context switches: slow, but the protocol is the multi-GPU one."""
    import torch.distributed as dist
    from paper_1904_07935_b200.sharded import connect
    rank = int(os.environ["RANK"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, w0, ht0 = conditioned_state(400, 300, 8, 0.05, 3)
        plan = ShardPlan(400, 300, world)
        e = ShardEngine.from_csr(m, world, rank, 8)
        e.set_timeout(120.0)
        connect(e, chain_norm=False)
        e.set_factors(P.FactorPair(w0[slice(*plan.v_range(rank))], ht0[slice(*plan.d_range(rank))]))
        cfg = P.SolverConfig(rank=8, tile_size=3)
        e.precompute_h_products()
        e.update_h(cfg, P.Algorithm.tiled)
        e.precompute_w_products()
        e.update_w(cfg, P.Algorithm.tiled)
        rep = e.evaluate_error()
        f = e.get_factors()
        np.savez(os.environ["OUT"] + f"_r{rank}.npz", w=f.w, ht=f.ht, err=rep.relative, q=e.get_product("q"))
        e.close()
    finally:
        dist.destroy_process_group()


CASES = {f.__name__: f for f in (case_step_products_and_updates, case_iterate_matches_single_engine,
                                  case_fast_hals_sharded, case_generated_shards, case_missing_rank_times_out,
                                  case_ipc_rank)}


def _run_case(name, world):
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    res = subprocess.run([sys.executable, str(Path(__file__).resolve()), name, str(world)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_step_products_and_updates_match_the_restatement(gpu, world):
    _run_case("case_step_products_and_updates", world)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_iterate_matches_single_engine(gpu, world):
    _run_case("case_iterate_matches_single_engine", world)


@pytest.mark.parametrize("world", [2, 3])
def test_fast_hals_on_the_sharded_engine(gpu, world):
    _run_case("case_fast_hals_sharded", world)


@pytest.mark.parametrize("world", [2, 4])
def test_generated_shards_match_host_blocks_and_init(gpu, world):
    _run_case("case_generated_shards", world)


def test_missing_rank_times_out_instead_of_hanging(gpu):
    _run_case("case_missing_rank_times_out", 2)


def test_two_processes_connected_over_cuda_ipc(gpu, tmp_path):
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    world = 2
    procs = []
    for g in range(world):
        env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", RANK=str(g), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), OUT=str(tmp_path / "ipc"))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), "case_ipc_rank", str(world)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(o[-3000:] for o in outs)
    got = [np.load(tmp_path / f"ipc_r{g}.npz") for g in range(world)]
    # the same arithmetic as the in-process ranks: the sharded restatement
    m, w0, ht0 = conditioned_state(400, 300, 8, 0.05, 3)
    plan = ShardPlan(400, 300, world)
    trp, tci, tval = R.transpose(400, 300, m.row_ptr, m.col_idx, m.values)
    s_sh = ordered_sum([R.gram(np.ascontiguousarray(w0[slice(*plan.v_range(g))])) for g in range(world)])
    ht1, _ = R.update_tiled(ht0, s_sh, R.spmm(300, 400, trp, tci, tval, w0), 3, is_w=False)
    q_sh = ordered_sum([R.gram(np.ascontiguousarray(ht1[slice(*plan.d_range(g))])) for g in range(world)])
    w1, _ = R.update_tiled(w0, q_sh, R.spmm(400, 300, m.row_ptr, m.col_idx, m.values, ht1), 3, is_w=True)
    for g in range(world):
        assert bits_equal(got[g]["ht"], ht1[slice(*plan.d_range(g))])
        assert bits_equal(got[g]["q"], q_sh)
    assert rel_max(w1, np.concatenate([x["w"] for x in got])) <= 1e-12
    assert float(got[0]["err"]) == float(got[1]["err"])


def test_ranks_sharing_a_gpu_require_eager_loading(gpu):
    env = dict(os.environ, CUDA_MODULE_LOADING="LAZY")
    code = ("import sys; sys.path.insert(0, %r); from paper_1904_07935_b200 import plnmf as P; "
            "from paper_1904_07935_b200.sharded import ShardEngine, connect_local\n"
            "m = P.synth_csr(200, 100, 0.05, 1); e = [ShardEngine.from_csr(m, 2, g, 4) for g in range(2)]\n"
            "try:\n    connect_local(e)\nexcept P.InvalidArgument as x:\n    print('refused:', x)\n")
    res = subprocess.run([sys.executable, "-c", code % str(Path(__file__).resolve().parents[1])], env=env,
                         capture_output=True, text=True, timeout=300)
    assert "refused:" in res.stdout and "CUDA_MODULE_LOADING=EAGER" in res.stdout, res.stdout + res.stderr


if __name__ == "__main__":
    CASES[sys.argv[1]](int(sys.argv[2]))
    print("ok")
