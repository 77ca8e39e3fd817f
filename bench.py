#!/usr/bin/env python
"""Benchmark: FAST-HALS iterations/sec (BASELINE.json metric), PL-NMF tiled
algorithm, fp64, on the B200 engine.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference] [--workload c2|c5]

N = 1 (default): configs[1] = SURVEY.md C2, the 20News-shaped sparse A at
K=240.  A step is one FAST-HALS iteration (R=A^T W, S=W^T W, H update, P=A Ht,
Q=Ht^T Ht, W update) with everything resident in HBM, timed with CUDA events on
the engine stream; L2 is flushed (a 512 MiB write) between steps, outside the
timed interval.

N > 1 (torchrun, one process per GPU): configs[4] = SURVEY.md C5 (2M x 1M, ~1e9
nonzeros, K=256) on the sharded engine — W rows and Ht rows split over the
ranks, the all-gathers and the per-column norm exchange over NVLink peer
memory (csrc/shard_engine.cu).  One problem of fixed size: strong scaling;
`--workload c5` runs the same engine on one GPU for the 1-GPU point.  The max
over ranks of the device time is reported.  One JSON line, printed by rank 0.

--impl reference times the reference's own CPU implementation (oracle/_ref:
libplnmf compiled from the unmodified sources) on this host's cores, same
workload and metric (C5: a 64x scaled C5-shaped sample, extrapolated); its
input comes from oracle/synth.c, so that arm never loads the engine library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# C2 of SURVEY.md 8(d): 20News shape, nnz ~ 1,018,191, K=240.
V, D, NNZ_TARGET, K = 26214, 11314, 1018191, 240
DENSITY = NNZ_TARGET / (V * D)
GEN_SEED = 20
TILE = 16  # T_auto of the reference's cost model for K=240 (best_integer_tile), BASELINE.md 2
METRIC = "FAST-HALS iters/sec at K=240 (20News-shaped sparse A); SpMM % HBM peak"


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.out = index, None, ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out = self.proc.communicate(timeout=5)[0]
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [[x.strip() for x in ln.split(",")] for ln in self.out.splitlines() if ln.count(",") >= 5]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else None  # noqa: E731
        sm = [v for v in (num(r[0]) for r in rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[2:6]) if v.strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def make_input():
    from paper_1904_07935_b200 import plnmf as P
    return P.synth_csr(V, D, DENSITY, GEN_SEED)


class _RefCsr:
    """The same C2 matrix for the reference arm, built by oracle/synth.c (the
    engine's generator stream restated on the reference side) so that the
    reference arm never loads the engine library."""

    def __init__(self):
        from oracle.oracle import synth_csr
        self.rows, self.cols = V, D
        self.row_ptr, self.col_idx, self.values = synth_csr(V, D, DENSITY, GEN_SEED)

    def nnz(self):
        return int(self.row_ptr[-1])


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# BENCH_DIST_BACKEND=gloo (a test hook): the ranks' bootstrap and host-side reductions over gloo,
# and ranks may share GPUs (LOCAL_RANK modulo the visible devices) — the launch path of N GPUs
# exercised on one (the ranks' contexts then time-slice the GPU: correct but not a measurement).
DIST_BACKEND = os.environ.get("BENCH_DIST_BACKEND", "nccl")


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if DIST_BACKEND == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group(DIST_BACKEND)
        return rank, world, local, dist
    return rank, world, local, None


def _reduce(dist, local, x: float, op) -> float:
    import torch
    dev = f"cuda:{local}" if DIST_BACKEND == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def allmax(dist, local, x: float) -> float:
    if dist is None:
        return x
    return _reduce(dist, local, x, dist.ReduceOp.MAX)


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ----------------------------------------------------------------------------- reference arm
def time_reference_cpu(m, steps, warmup, tiled=True):
    """The reference's own iterate() (oracle/_ref: libplnmf compiled from the
    unmodified sources) on this host's cores, as ONE call of
    max_iters = 1 + warmup + steps with error_every = 1: iteration 1 (which also
    builds the cached transpose, hals.cpp:26) and `warmup` more are discarded;
    each timed iteration is its wall-clock delta minus its error evaluation
    (the reference's convention, (total - error_eval) / iters,
    acceptance.cpp:251, per iteration), so setup never counts."""
    from oracle.oracle import RefInput, ref, ref_init_factors, ref_iterate
    a = RefInput(m.rows, m.cols, m.row_ptr, m.col_idx, m.values)
    w, ht = ref_init_factors(m.rows, m.cols, K, seed=0)
    cores = ref().ref_max_threads()
    n = 1 + warmup + steps
    _, _, tr = ref_iterate(a, w, ht, K, max_iters=n, rel_tol=0.0, error_every=1,
                           tile=TILE if tiled else 0, tiled=tiled)
    rec = tr["records"]  # iteration, rel_error, elapsed_s (cumulative), 9 phase buckets (error_eval last)
    el = rec[:, 2]
    per = [(el[i] - el[i - 1]) - rec[i, 11] for i in range(1 + warmup, n)]
    return per, cores


def reference_sample(steps, warmup, tiled):
    alg = f"PL-NMF (T={TILE})" if tiled else "FAST-HALS (update_w_reference: serial W update)"
    return (f"{steps} {alg} iterations of C2 timed inside one reference iterate(max_iters={1 + warmup + steps}, "
            f"error_every=1) call after {1 + warmup} discarded (setup + warm-up); per iteration = wall delta "
            f"- error_eval (acceptance.cpp:251 convention); oracle/_ref = the reference compiled from its "
            f"unmodified sources, OpenMP on all host cores ({cpu_model()})")


def reference_arm(args, workload="c2"):
    # CPU-only: under torchrun rank 0 alone runs it, the other ranks exit 0 without work
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if workload == "c5":
        try:
            val, cores, sample = time_reference_c5(steps=min(args.steps, 2))
        except ImportError as e:
            print(json.dumps({"impl": "reference", "unavailable": str(e)}))
            return
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": val, "unit": "iters/s", "n_gpus": args.gpus,
            "steps": min(args.steps, 2), "warmup": 1, "ms_per_step": 1e3 / val, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c5_config(args.gpus), "extrapolated": f"x{C5_SAMPLE} from a scaled C5-shaped sample",
            "cpu_baseline": {"value": val, "unit": "iters/s", "cores": cores, "kind": "reference",
                             "cpu": cpu_model(), "sample": sample},
            "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
            flush=True)
        return
    try:
        m = _RefCsr()
        per, cores = time_reference_cpu(m, args.steps, args.warmup, tiled=True)
        fh_steps = 2
        per_fh, _ = time_reference_cpu(m, fh_steps, 0, tiled=False)
    except ImportError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return
    spi = float(np.mean(per))
    val = 1.0 / spi
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": spi * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(m),
        "cpu_baseline": {"value": val, "unit": "iters/s", "cores": cores, "kind": "reference",
                         "cpu": cpu_model(), "sample": reference_sample(args.steps, args.warmup, True)},
        "fast_hals": {"value": 1.0 / float(np.mean(per_fh)), "unit": "iters/s", "cores": cores,
                      "sample": reference_sample(fh_steps, 0, False)},
        "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(m):
    return {"workload": f"C2: 20News-shaped synthetic CSR {V}x{D}, nnz={m.nnz()}, K={K}, PL-NMF tile {TILE}, "
                        "FAST-HALS iteration (H then W update)",
            "V": V, "D": D, "nnz": m.nnz(), "K": K, "tile_size": TILE, "algorithm": "pl-nmf (tiled)",
            "generator": f"splitmix64 geometric-gap Bernoulli rows, seed {GEN_SEED}, values U(0.1,2.0) fp32-rounded",
            "l2": "flushed (512 MiB write) between timed steps"}


# ----------------------------------------------------------------------------- engine arm
def spmm_bytes(rows, other_rows, nnz, k):
    """Algorithmic HBM bytes of one fp64 CSR SpMM launch: values (8 B) + int32
    column indices (4 B) per nonzero, int64 row pointers, the dense operand read
    once and the output written once."""
    return 12 * nnz + 8 * (rows + 1) + 8 * other_rows * k + 8 * rows * k


def engine_arm(args):
    import torch
    from paper_1904_07935_b200 import plnmf as P

    rank, world, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    m = make_input()
    a = P.InputMatrix(m)
    eng = P.Engine(a, K, device=local)
    eng.set_math(P.Math.exact if args.math == "exact" else P.Math.fused)
    cfg = P.SolverConfig(rank=K, tile_size=TILE, max_iters=1, rel_tol=0.0, seed=rank)
    alg = P.Algorithm.tiled
    eng.init_factors(cfg)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    for _ in range(args.warmup):
        eng.run_iterations(cfg, alg, 1)
    launches0 = eng.stats()["kernel_launches"]
    step_ms = []
    barrier(dist)
    torch.cuda.synchronize()
    phase_tot = {}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            step_ms.append(eng.run_iterations(cfg, alg, 1))
            for k2, v2 in eng.phase_ms().items():  # CUDA events on the engine stream, inside the timed steps
                phase_tot[k2] = phase_tot.get(k2, 0.0) + v2
    torch.cuda.synchronize()
    barrier(dist)
    launches = eng.stats()["kernel_launches"] - launches0
    total_ms = allmax(dist, local, float(sum(step_ms)))
    value = world * args.steps / (total_ms * 1e-3)

    # back-to-back (L2 warm) for context
    eng.run_iterations(cfg, alg, 2)
    warm_ms = allmax(dist, local, eng.run_iterations(cfg, alg, args.steps)) / args.steps

    # per-kernel times (CUDA events on the engine stream) for the roofline
    reps = 10
    kt = {"spmm_A_Ht": eng.time_kernel(cfg, 0, reps), "spmm_At_W": eng.time_kernel(cfg, 1, reps),
          "gram_W": eng.time_kernel(cfg, 2, reps), "update_w_tiled": eng.time_kernel(cfg, 3, reps),
          "update_h_tiled": eng.time_kernel(cfg, 4, reps)}
    pk = peaks()
    hbm = float(pk["hbm_gbs"])
    nnz = m.nnz()
    b_p = spmm_bytes(V, D, nnz, K)
    b_r = spmm_bytes(D, V, nnz, K)
    step = total_ms / args.steps
    # dominant kernel by share of the step (two SpMMs per step)
    shares = {"spmm": kt["spmm_A_Ht"] + kt["spmm_At_W"], "update_w_tiled": kt["update_w_tiled"],
              "update_h_tiled": kt["update_h_tiled"], "gram": 2 * kt["gram_W"]}
    # W update (the dominant kernel) compulsory bytes: read W and P, write W_new (V x K each), read Q
    b_w = 3 * 8 * V * K + 8 * K * K
    w_ms = phase_tot["update_w"] / args.steps  # per launch, measured inside the timed steps
    rl_w = b_w / (w_ms * 1e-3) / 1e9
    roofline = {"kernel": "pl_update_kernel (W update, tiled; the step's dominant kernel)", "bound": "hbm",
                "achieved": rl_w, "peak": hbm, "unit": "GB/s", "frac": rl_w / hbm,
                "traffic": ncu_traffic("wupdate"), "algorithmic_bytes": b_w, "launch_ms": w_ms,
                "share_of_step": w_ms / (total_ms / args.steps),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if not pk.get("_fallback") else "fallback",
                # what actually bounds it: K = 240 dependent grid-wide norm reductions (tiled.cpp:92-148)
                "latency": {"us_per_column": w_ms * 1e3 / K, "isolated_chain_plus_exchange_us": 1.73,
                            "frac_of_floor": 1.73 / (w_ms * 1e3 / K),
                            "source": "tools/chain_bench.cu, tools/exchange_bench2.cu (profiles/r1_microbench.txt)"}}
    rl_spmm = b_p / (kt["spmm_A_Ht"] * 1e-3) / 1e9
    l2 = l2_peak()
    # e2e through the reference-facing C-ABI call with host factors
    e2e = e2e_arm(P, a, eng, cfg, alg, args, torch)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            per, cores = time_reference_cpu(m, steps=args.cpu_steps, warmup=1, tiled=True)
            cpu = {"value": 1.0 / float(np.mean(per)), "unit": "iters/s", "cores": cores, "kind": "reference",
                   "cpu": cpu_model(), "sample": reference_sample(args.cpu_steps, 1, True)}
            per_fh, _ = time_reference_cpu(m, steps=2, warmup=0, tiled=False)
            cpu["fast_hals"] = {"value": 1.0 / float(np.mean(per_fh)), "unit": "iters/s",
                                "sample": reference_sample(2, 0, False)}
        except ImportError as e:
            cpu = {"value": None, "unit": "iters/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload_config(m),
            "math": args.math, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "warm_l2_ms_per_iter": warm_ms,
            "kernels_ms": kt, "kernel_share_of_step": {k2: v2 / step for k2, v2 in shares.items()},
            "phase_ms_per_step": {k2: v2 / args.steps for k2, v2 in phase_tot.items()},
            # the SpMMs (BASELINE metric's second half) against HBM and against the
            # measured L2 gather ceiling that actually bounds them (Finding 3)
            "spmm_roofline": {"A_Ht_GBps": rl_spmm, "At_W_GBps": b_r / (kt["spmm_At_W"] * 1e-3) / 1e9,
                              "hbm_frac_A_Ht": rl_spmm / hbm, "bytes_A_Ht": b_p, "bytes_At_W": b_r,
                              "l2_gather_bytes": 8 * nnz * K,
                              "l2_gather_GBps": 8 * nnz * K / (kt["spmm_A_Ht"] * 1e-3) / 1e9,
                              "l2_gather_peak_GBps": l2.get("gather_l2_gbs_16B"),
                              "l2_frac": (8 * nnz * K / (kt["spmm_A_Ht"] * 1e-3) / 1e9 / l2["gather_l2_gbs_16B"])
                              if l2.get("gather_l2_gbs_16B") else None,
                              "l2_peak_source": "profiles/l2_peak.json (tools/l2bw_bench.cu on a B200)",
                              "traffic": ncu_traffic("spmm")},
            "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


E2E_ITERS = 100  # configs[1]: "K=240, 100 iterations on 1 B200"


def e2e_arm(P, a, eng, cfg, alg, args, torch):
    """Each step = one drop-in iterate() call through the C-ABI with HOST
    factors in pinned memory (plnmf_gpu_iterate_host), on BASELINE.json
    configs[1]'s workload: 100 FAST-HALS iterations with the reference's
    defaults (error evaluated every iteration, solver.cpp:75-76,94-95; rel_tol 0
    so all 100 run).  Timed on the host wall clock: H2D of W and Ht, the 101
    error evaluations, 100 iterations, D2H of W, Ht and the trace."""
    import ctypes as C
    from paper_1904_07935_b200 import _lib as L
    f = eng.get_factors()
    # pinned, column-major (Fortran) host factors: a (K, n) row-major pinned tensor viewed transposed
    tw = torch.empty((K, V), dtype=torch.float64, pin_memory=True)
    th = torch.empty((K, D), dtype=torch.float64, pin_memory=True)
    w, ht = tw.numpy().T, th.numpy().T
    w[...] = f.w
    ht[...] = f.ht
    assert w.flags.f_contiguous and ht.flags.f_contiguous
    w0, ht0 = w.copy(order="F"), ht.copy(order="F")
    c = P.SolverConfig(rank=K, tile_size=TILE, max_iters=E2E_ITERS, rel_tol=0.0, error_every=1).to_c()
    buf = P._TraceBuf(E2E_ITERS)
    lib = L.lib()
    ptr = lambda x: x.ctypes.data_as(L.P_f64)  # noqa: E731
    P._check(lib.plnmf_gpu_iterate_host(eng._h, C.byref(c), int(alg), ptr(w), ptr(ht), C.byref(buf.c)))  # warm
    n = max(2, min(5, args.steps // 10))
    dt = 0.0
    for _ in range(n):
        w[...] = w0  # every call restarts from the same host factors (outside the timed region)
        ht[...] = ht0
        t0 = time.perf_counter()
        P._check(lib.plnmf_gpu_iterate_host(eng._h, C.byref(c), int(alg), ptr(w), ptr(ht), C.byref(buf.c)))
        dt += time.perf_counter() - t0
    fb = 8 * (V + D) * K
    tb = 8 * 3 + 8 * 12 * E2E_ITERS  # initial error + one trace record per iteration
    return {"value": n * E2E_ITERS / dt, "unit": "iters/s", "h2d_bytes_per_step": fb, "d2h_bytes_per_step": fb + tb,
            "iters_per_step": E2E_ITERS, "steps": n,
            "what": f"plnmf_gpu_iterate_host(max_iters={E2E_ITERS}, error_every=1, rel_tol=0) on pinned host W,Ht "
                    "(col-major f64): upload, 100 iterations with the reference's per-iteration error evaluation "
                    "and stop-rule check, download; host wall clock"}


def l2_peak():
    try:
        return json.loads((ROOT / "profiles" / "l2_peak.json").read_text())
    except Exception:
        return {}


def ncu_traffic(kernel):
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        d = json.loads(p.read_text())
        return d.get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ----------------------------------------------------------------------------- C5: the sharded engine
# 2M x 1M, density 5e-4 (~1e9 nonzeros, ~500 per row), K=256, T_auto=16;
# W row-sharded over V, H over D (8(e)); every rank generates its blocks on the device.
V5, D5, DENS5, K5, TILE5 = 2_000_000, 1_000_000, 5e-4, 256, 16
C5_SAMPLE = 64  # reference arm: a C5-shaped instance scaled down 64x in rows and columns


def c5_config(world, nnz=None):
    return {"workload": f"C5: synthetic CSR {V5}x{D5}, density {DENS5} (~1e9 nonzeros), K={K5}, PL-NMF tile "
                        f"{TILE5}, FAST-HALS iteration, W rows / Ht rows sharded over {world} GPU(s)",
            "V": V5, "D": D5, "nnz": nnz, "K": K5, "tile_size": TILE5, "algorithm": "pl-nmf (tiled)",
            "generator": f"splitmix64 geometric-gap Bernoulli rows, seed {GEN_SEED}, values U(0.1,2.0) fp32-rounded, "
                         "generated on the device per rank",
            "parallelism": f"row/column-sharded x{world} (peer-memory all-gathers + in-kernel norm exchange)",
            "l2": "inputs larger than L2 (A 12 GB, W 4 GB): no flush"}


def c5_arm(args):
    """The large config through the sharded engine: one process per GPU, the
    ranks connected over torch.distributed (IPC handles), one problem of fixed
    size (strong scaling).  A step is one FAST-HALS iteration of the whole
    problem; every rank times its run_iterations with CUDA events on its engine
    stream and the max over ranks is reported."""
    import torch
    from paper_1904_07935_b200 import plnmf as P
    from paper_1904_07935_b200.sharded import ShardEngine, connect

    rank, world, local, dist = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    t0 = time.perf_counter()
    eng = ShardEngine.generate(V5, D5, DENS5, GEN_SEED, K5, world, rank, device=local)
    if dist is not None:
        connect(eng)  # IPC handles all-gathered, ||A||^2 chained over the ranks
    else:
        eng.set_norm_sq(eng.norm_sq_from(0.0))
    setup_s = time.perf_counter() - t0
    nnz_local = eng.nnz
    nnz = int(allsum(dist, local, float(nnz_local)))
    alg = P.Algorithm.tiled
    cfg = P.SolverConfig(rank=K5, tile_size=TILE5, max_iters=1, rel_tol=0.0)
    rng = np.random.default_rng(1000 + rank)  # synthetic factors: each rank's rows, U(1e-3, 1)
    f0 = P.FactorPair(np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.v, K5))),
                      np.asfortranarray(rng.uniform(1e-3, 1.0, (eng.d, K5))))
    eng.set_factors(f0)
    for _ in range(args.warmup):
        eng.run_iterations(cfg, alg, 1)
    launches0 = eng.stats()["kernel_launches"]
    barrier(dist)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = eng.run_iterations(cfg, alg, args.steps)
    torch.cuda.synchronize()
    barrier(dist)
    launches = eng.stats()["kernel_launches"] - launches0
    phases = {k2: v2 / args.steps for k2, v2 in eng.phase_ms().items()}
    total_ms = allmax(dist, local, ms)
    value = args.steps / (total_ms * 1e-3)

    # e2e through the public API with host factors: upload this rank's rows, iterate()
    # (error evaluated every iteration, reference defaults), download
    e2e_iters = 2
    ecfg = P.SolverConfig(rank=K5, tile_size=TILE5, max_iters=e2e_iters, rel_tol=0.0, error_every=1)
    barrier(dist)
    t1 = time.perf_counter()
    eng.set_factors(f0)
    eng.iterate(ecfg, alg)
    f1 = eng.get_factors()
    e2e_s = allmax(dist, local, time.perf_counter() - t1)
    fb = 8 * (eng.v + eng.d) * K5

    # P = A_g Ht_full (the precompute_w phase, which also holds Q = gram(Ht_g)) against HBM with its
    # compulsory bytes, and its operand-row gathers (one K-wide row per nonzero) against the measured
    # L2 gather peak: the column-blocked SpMM (spmm.cu) keeps each block's operand rows in L2
    pk = peaks()
    hbm = float(pk["hbm_gbs"])
    pw_ms = phases["precompute_w"]
    b_alg = 12.0 * nnz_local + 8.0 * (eng.v + 1) + 8.0 * D5 * K5 + 8.0 * eng.v * K5
    gather = 8.0 * nnz_local * K5
    l2 = l2_peak()
    rate = b_alg / (pw_ms * 1e-3) / 1e9
    roofline = {"kernel": "spmm_blocked_kernel (P = A_g Ht_full, column-blocked; timed as the precompute_w "
                          "phase, which also holds Q = gram(Ht_g))", "bound": "hbm",
                "achieved": rate, "peak": hbm, "unit": "GB/s", "frac": rate / hbm,
                "traffic": ncu_traffic("c5_spmm_per_spmm"), "algorithmic_bytes": b_alg,
                "bytes_definition": "12 B per nonzero + row pointers + the operand read once + P written once",
                "launch_ms": pw_ms, "share_of_step": pw_ms / (total_ms / args.steps),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if not pk.get("_fallback") else "fallback",
                "l2_gather": {"bytes": gather, "GBps": gather / (pw_ms * 1e-3) / 1e9,
                              "peak_GBps": l2.get("gather_l2_gbs_16B"),
                              "frac": (gather / (pw_ms * 1e-3) / 1e9 / l2["gather_l2_gbs_16B"])
                              if l2.get("gather_l2_gbs_16B") else None,
                              "peak_source": "profiles/l2_peak.json (tools/l2bw_bench.cu on a B200)"}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            val, cores, sample = time_reference_c5(steps=2)
            cpu = {"value": val, "unit": "iters/s", "cores": cores, "kind": "reference", "cpu": cpu_model(),
                   "sample": sample}
        except ImportError as e:
            cpu = {"value": None, "unit": "iters/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c5_config(world, nnz), "math": "exact", "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": e2e_iters / e2e_s, "unit": "iters/s", "h2d_bytes_per_step": fb,
                    "d2h_bytes_per_step": fb, "iters_per_step": e2e_iters,
                    "what": "per rank: set_factors (this rank's W, Ht rows from host), iterate(max_iters=2, "
                            "error_every=1, rel_tol=0), get_factors; host wall clock, max over ranks"},
            "gpu_launches": launches, "clocks": clk.summary(), "phase_ms_per_step": phases,
            "setup_s": setup_s, "nnz_per_rank": nnz_local,
            "parallelism": f"sharded x{world}",
            "workload_note": "N = 1 runs configs[1] (C2, the metric's config); N > 1 runs configs[4] (C5, the "
                             "config that shards). The 1-GPU point of THIS workload is `bench.py --workload c5`",
            "one_gpu_same_workload": c5_one_gpu_reference(),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if dist is not None:
        dist.destroy_process_group()


def c5_one_gpu_reference():
    """The committed 1-GPU measurement of the C5 workload (bench.py --workload c5 on a B200)."""
    try:
        d = json.loads((ROOT / "profiles" / "r2_bench_c5_1gpu.json").read_text())
        return {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                "source": "profiles/r2_bench_c5_1gpu.json (bench.py --workload c5, one B200)"}
    except Exception:
        return None


def time_reference_c5(steps):
    """The reference on a C5-shaped instance scaled down C5_SAMPLE x in rows and
    columns with the same nonzeros per row (so nnz, the Grams and the updates
    all scale by 1/C5_SAMPLE), timed like time_reference_cpu; the per-iteration
    time is multiplied by C5_SAMPLE.  The sample's factors fit the host caches
    far better than C5's, so the estimate favours the reference."""
    from oracle.oracle import RefInput, ref, ref_init_factors, ref_iterate, synth_csr
    v, d = V5 // C5_SAMPLE, D5 // C5_SAMPLE
    rp, ci, val = synth_csr(v, d, DENS5 * C5_SAMPLE, GEN_SEED)
    a = RefInput(v, d, rp, ci, val)
    w, ht = ref_init_factors(v, d, K5, seed=0)
    cores = ref().ref_max_threads()
    n = 1 + steps
    _, _, tr = ref_iterate(a, w, ht, K5, max_iters=n, rel_tol=0.0, error_every=1, tile=TILE5, tiled=True)
    rec = tr["records"]
    el = rec[:, 2]
    per = [(el[i] - el[i - 1]) - rec[i, 11] for i in range(1, n)]
    spi = float(np.mean(per)) * C5_SAMPLE
    sample = (f"{steps} PL-NMF (T={TILE5}) iterations of a C5-shaped {v}x{d} instance ({int(rp[-1])} nonzeros, "
              f"~{DENS5 * C5_SAMPLE * d:.0f} per row as in C5), K={K5}, after 1 discarded; per iteration = wall delta "
              f"- error_eval, x{C5_SAMPLE} (every phase is linear in rows at fixed nonzeros per row); oracle/_ref "
              f"on all host cores ({cpu_model()})")
    return 1.0 / spi, cores, sample


def allsum(dist, local, x: float) -> float:
    if dist is None:
        return x
    return _reduce(dist, local, x, dist.ReduceOp.SUM)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--math", default="exact", choices=["exact", "fused"])
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default=None, choices=["c2", "c5"],
                    help="default: C2 on 1 GPU (the metric's config), the sharded C5 on N > 1 GPUs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    workload = args.workload or ("c5" if max(world, args.gpus) > 1 else "c2")
    if args.impl == "reference":
        reference_arm(args, workload)
    elif workload == "c5":
        c5_arm(args)
    else:
        engine_arm(args)


if __name__ == "__main__":
    main()
