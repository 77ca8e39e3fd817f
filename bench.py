#!/usr/bin/env python
"""Benchmark: FAST-HALS iterations/sec on the 20News-shaped sparse A at K=240
(BASELINE.json metric; configs[1] = SURVEY.md C2), PL-NMF tiled algorithm,
fp64, on the B200 engine.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

A step is one FAST-HALS iteration (R=A^T W, S=W^T W, H update, P=A Ht,
Q=Ht^T Ht, W update) with everything resident in HBM.  Each step is timed
with CUDA events on the engine stream; L2 is flushed (a 512 MiB write) between
steps, outside the timed interval.  N>1 runs N independent replicas (one
process per GPU; C2 does not shard) and reports the max over
ranks.  One JSON line is printed by rank 0.

--impl reference times the reference's own CPU implementation (oracle/_ref:
libplnmf compiled from the unmodified sources) on this host's cores, same
workload and metric; its input comes from oracle/synth.c, so that arm never
loads the engine library.
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


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return rank, world, local, dist
    return rank, world, local, None


def allmax(dist, local, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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


def reference_arm(args):
    # CPU-only: under torchrun rank 0 alone runs it, the other ranks exit 0 without work
    if int(os.environ.get("RANK", "0")) != 0:
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--math", default="exact", choices=["exact", "fused"])
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        engine_arm(args)


if __name__ == "__main__":
    main()
