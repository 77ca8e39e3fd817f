// Look-ahead GEMM variants measured in tools/gemm_bench.cu and NOT used by the
// engine ("What was tried"): group-staged RG-rows x 1-column items
// (lookahead_gemm), group-staged row x CG items (lookahead_gemm_rows) and a
// producer-warp mbarrier ring (lookahead_gemm_bulk).  The engine's variant,
// lookahead_gemm_private, lives in paper_1904_07935_b200/csrc/lookahead.cuh.
#pragma once

#include "lookahead.cuh"

namespace plnmf {

// MODE (microbenchmarks only): 0 full, 1 arithmetic without staging, 2 staging without arithmetic
template <class M, int RG, int MODE = 0>
__device__ __forceinline__ void lookahead_gemm(const GemmArgs& g) {
    const int wn = g.en - g.bn, k = g.k;
    const int ngroups = (g.nrows + RG - 1) / RG;
    const int nitems = ngroups * wn;
    const int n1 = k - g.en;
    const int nch1 = (n1 + kGemmKC - 1) / kGemmKC, nch = nch1 + (g.bprev + kGemmKC - 1) / kGemmKC;
    const unsigned xb = smem_u32(g.xbuf), qb = smem_u32(g.q);
    auto chunk = [&](int ch, const double*& src, int& kk0, int& n) {
        if (ch < nch1) { src = g.old_m; kk0 = g.en + ch * kGemmKC; n = min(kGemmKC, k - kk0); }
        else { src = g.out; kk0 = (ch - nch1) * kGemmKC; n = min(kGemmKC, g.bprev - kk0); }
    };
    auto stage = [&](int ch) {
        if (MODE != 1 && ch < nch) {
            const double* src; int kk0, n;
            chunk(ch, src, kk0, n);
            double* xs = g.xbuf + (ch % kGemmStages) * g.buf_doubles;
            const double* gsrc = src + g.r0 * k + kk0;
            if (((k | kk0 | n) & 1) == 0) {
                const int nu = n >> 1;
                for (int idx = g.self; idx < g.nrows * nu; idx += g.count) {
                    const int r = idx / nu, u = idx - r * nu;
                    cp_async16(xs + r * kGemmKCP + 2 * u, gsrc + (int64_t)r * k + 2 * u);
                }
            } else {
                for (int idx = g.self; idx < g.nrows * n; idx += g.count) {
                    const int r = idx / n, u = idx - r * n;
                    cp_async8(xs + r * kGemmKCP + u, gsrc + (int64_t)r * k + u);
                }
            }
        }
        cp_async_commit();  // possibly empty: keeps the group count uniform
    };
    for (int pass = 0; pass < nitems; pass += g.count) {
        const int item = pass + g.self;
        const bool act = item < nitems;
        const int grp = act ? item / wn : 0, c = act ? item - grp * wn : 0;
        const int rb = grp * RG;
        const int rn = act ? min(RG, g.nrows - rb) : 0;
        double a[RG];
#pragma unroll
        for (int i = 0; i < RG; ++i) {
            a[i] = 0.0;
            if (i < rn) {
                const double o = g.old_m[(g.r0 + rb + i) * k + g.bn + c];
                a[i] = g.use_diag ? dmul(o, lds64(qb + 8u * ((g.bn + c) * g.tq + c))) : o;
            }
        }
        stage(0);
        stage(1);
        for (int ch = 0; ch < nch; ++ch) {
            cp_async_wait<1>();
            named_sync(g.bar, g.count);  // chunk ch visible; chunk ch-1's buffer free
            stage(ch + 2);
            const double* src; int kk0, n;
            chunk(ch, src, kk0, n);
            const unsigned xs = xb + 8u * ((ch % kGemmStages) * g.buf_doubles + rb * kGemmKCP);
            const unsigned qc = qb + 8u * (kk0 * g.tq + c);
            if (MODE == 2) {
            } else if (n == kGemmKC && rn == RG) {
#pragma unroll
                for (int j = 0; j < kGemmKC; j += 2) {
                    const double q0 = -1.0 * lds64(qc + 8u * (j * g.tq));
                    const double q1 = -1.0 * lds64(qc + 8u * ((j + 1) * g.tq));
#pragma unroll
                    for (int i = 0; i < RG; ++i) {
                        const double2 xx = lds128(xs + 8u * (i * kGemmKCP + j));
                        a[i] = M::madd(a[i], q0, xx.x);
                        a[i] = M::madd(a[i], q1, xx.y);
                    }
                }
            } else {
                for (int j = 0; j < n; ++j) {
                    const double q0 = -1.0 * lds64(qc + 8u * (j * g.tq));
#pragma unroll
                    for (int i = 0; i < RG; ++i)
                        if (i < rn) a[i] = M::madd(a[i], q0, lds64(xs + 8u * (i * kGemmKCP + j)));
                }
            }
        }
        cp_async_wait<0>();
        named_sync(g.bar, g.count);  // every buffer free before the next pass / caller reuse
#pragma unroll
        for (int i = 0; i < RG; ++i)
            if (i < rn) g.dst[(rb + i) * g.ldt + c] = a[i];
    }
}

}  // namespace plnmf

namespace plnmf {

// Row-major variant: a thread item is ONE row and CG consecutive columns of
// the tile (lanes = consecutive rows).  Per kk pair a thread reads its own
// row's operand pair (one conflict-free 16-byte load: rows are kGemmKCP = 10
// doubles apart) and the CG coefficients of the pair (CG/2 + CG/2 16-byte
// loads, the same address in every lane: broadcast), then issues 4*CG fp64
// instructions — fp64-pipe bound for CG >= 8.  Staging is cooperative and
// coalesced (a warp copies 8 rows x 64 B per instruction, no integer
// division), kGemmStages-deep with one named barrier per chunk.  Per-element
// term order as lookahead_gemm: bit-identical under Math::exact.
template <class M, int CG, int NI = 1, int MODE = 0, int KC = kGemmKC, int ST = kGemmStages>
__device__ __forceinline__ void lookahead_gemm_rows(const GemmArgs& g) {
    static_assert(CG % 2 == 0, "CG must be even");
    const int wn = g.en - g.bn, k = g.k;
    const int ncg = (wn + CG - 1) / CG;
    const int nitems = g.nrows * ncg;
    const int n1 = k - g.en;
    const int nch1 = (n1 + KC - 1) / KC, nch = nch1 + (g.bprev + KC - 1) / KC;
    const unsigned xb = smem_u32(g.xbuf), qb = smem_u32(g.q);
    const bool vec = (k & 1) == 0;  // 16-byte global alignment of even columns
    auto chunk = [&](int ch, const double*& src, int& kk0, int& n) {
        if (ch < nch1) { src = g.old_m; kk0 = g.en + ch * KC; n = min(KC, k - kk0); }
        else { src = g.out; kk0 = (ch - nch1) * KC; n = min(KC, g.bprev - kk0); }
    };
    auto stage = [&](int ch) {
        if (MODE != 1 && ch < nch) {
            const double* src; int kk0, n;
            chunk(ch, src, kk0, n);
            double* xs = g.xbuf + (ch % ST) * g.buf_doubles;
            const double* gsrc = src + g.r0 * k + kk0;
            if (vec && ((kk0 | n) & 1) == 0 && n == KC) {
                constexpr int P = KC / 2;  // 16-byte pieces per row
                for (int idx = g.self; idx < g.nrows * P; idx += g.count) {
                    const int r = idx / P, u = idx % P;
                    cp_async16(xs + r * (KC + 2) + 2 * u, gsrc + (int64_t)r * k + 2 * u);
                }
            } else {
                for (int idx = g.self; idx < g.nrows * n; idx += g.count) {
                    const int r = idx / n, u = idx - r * n;
                    cp_async8(xs + r * (KC + 2) + u, gsrc + (int64_t)r * k + u);
                }
            }
        }
        cp_async_commit();
    };
    for (int pass = 0; pass < nitems; pass += NI * g.count) {
        int rr[NI], c0[NI], cn[NI];
        double a[NI][CG];
#pragma unroll
        for (int it = 0; it < NI; ++it) {
            const int item = pass + it * g.count + g.self;
            const bool act = item < nitems;
            const int cgi = act ? item / g.nrows : 0;
            rr[it] = act ? item - cgi * g.nrows : 0;
            c0[it] = cgi * CG;
            cn[it] = act ? min(CG, wn - c0[it]) : 0;
#pragma unroll
            for (int u = 0; u < CG; ++u) {
                a[it][u] = 0.0;
                if (u < cn[it]) {
                    const int c = c0[it] + u;
                    const double o = g.old_m[(g.r0 + rr[it]) * k + g.bn + c];
                    a[it][u] = g.use_diag ? dmul(o, lds64(qb + 8u * ((g.bn + c) * g.tq + c))) : o;
                }
            }
        }
#pragma unroll
        for (int st = 0; st < ST - 1; ++st) stage(st);
        for (int ch = 0; ch < nch; ++ch) {
            cp_async_wait<ST - 2>();
            named_sync(g.bar, g.count);  // chunk ch visible; chunk ch-1's buffer free
            stage(ch + ST - 1);
            if (MODE == 2) continue;
            const double* src; int kk0, n;
            chunk(ch, src, kk0, n);
#pragma unroll
            for (int it = 0; it < NI; ++it) {
                if (cn[it] <= 0) continue;
                const unsigned xs = xb + 8u * ((ch % ST) * g.buf_doubles + rr[it] * (KC + 2));
                const unsigned qc = qb + 8u * (kk0 * g.tq + c0[it]);
                if (n == KC) {
#pragma unroll
                    for (int j = 0; j < KC; j += 2) {
                        const double2 xx = lds128(xs + 8u * j);
#pragma unroll
                        for (int u = 0; u < CG; u += 2) {
                            // padded coefficient columns (c >= wn) are 0: harmless, never stored
                            const double2 qa = lds128(qc + 8u * (j * g.tq + u));
                            const double2 qn = lds128(qc + 8u * ((j + 1) * g.tq + u));
                            a[it][u] = M::madd(a[it][u], -1.0 * qa.x, xx.x);
                            a[it][u + 1] = M::madd(a[it][u + 1], -1.0 * qa.y, xx.x);
                            a[it][u] = M::madd(a[it][u], -1.0 * qn.x, xx.y);
                            a[it][u + 1] = M::madd(a[it][u + 1], -1.0 * qn.y, xx.y);
                        }
                    }
                } else {
                    for (int j = 0; j < n; ++j) {
                        const double x = lds64(xs + 8u * j);
#pragma unroll
                        for (int u = 0; u < CG; u += 2) {
                            const double2 qa = lds128(qc + 8u * (j * g.tq + u));
                            a[it][u] = M::madd(a[it][u], -1.0 * qa.x, x);
                            a[it][u + 1] = M::madd(a[it][u + 1], -1.0 * qa.y, x);
                        }
                    }
                }
            }
        }
        cp_async_wait<0>();
        named_sync(g.bar, g.count);
#pragma unroll
        for (int it = 0; it < NI; ++it)
#pragma unroll
            for (int u = 0; u < CG; ++u)
                if (u < cn[it]) g.dst[rr[it] * g.ldt + c0[it] + u] = a[it][u];
    }
}

}  // namespace plnmf

namespace plnmf {

// ---------------------------------------------------------------- mbarrier / bulk-copy pipeline
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared, completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Chunked operand ring of the bulk look-ahead GEMM.  `it` counts chunks
// across calls (uniform over the group) so stage/phase carry over tiles.
constexpr int kBulkKC = 16, kBulkKCP = kBulkKC + 2, kBulkStages = 3;
struct BulkPipe {
    unsigned full, empty;  // shared addresses of kBulkStages mbarriers each
    unsigned bufs;         // shared address of kBulkStages x buf_doubles
    int buf_doubles;
    unsigned it;
};

// Pipelined variant of lookahead_gemm_rows for even k / even chunk bounds
// (16-byte aligned rows): the LAST warp of the group is the producer — it
// cp.asyncs each row's kBulkKC-wide slice of a chunk into a kBulkStages ring
// (coalesced), each lane's completion arriving on the stage's `full` mbarrier
// (count 32, cp.async.mbarrier.arrive.noinc); the other
// warps consume (one row x CG columns per thread) and release the slot on its
// `empty` mbarrier (count = group warps - 1).  No group-wide barriers inside.
// Requires nrows * ceil(wn / CG) <= count - 32.
template <class M, int CG>
__device__ __forceinline__ void lookahead_gemm_bulk(const GemmArgs& g, BulkPipe& pp) {
    constexpr int KC = kBulkKC, KCP = kBulkKCP, ST = kBulkStages;
    const int wn = g.en - g.bn, k = g.k;
    const int ncg = (wn + CG - 1) / CG;
    const int nitems = g.nrows * ncg;
    const int nch1 = (k - g.en + KC - 1) / KC, nch = nch1 + (g.bprev + KC - 1) / KC;
    const int warp = g.self >> 5, lane = g.self & 31;
    const int prod = (g.count >> 5) - 1;
    const unsigned qb = smem_u32(g.q);
    auto chunk = [&](int ch, const double*& src, int& kk0, int& n) {
        if (ch < nch1) { src = g.old_m; kk0 = g.en + ch * KC; n = min(KC, k - kk0); }
        else { src = g.out; kk0 = (ch - nch1) * KC; n = min(KC, g.bprev - kk0); }
    };
    if (warp == prod) {
        for (int ch = 0; ch < nch; ++ch) {
            const unsigned it = pp.it + ch, st = it % ST, ph = (it / ST) & 1u;
            const double* src; int kk0, n;
            chunk(ch, src, kk0, n);
            if (lane == 0) mbar_wait(pp.empty + 8u * st, ph ^ 1u);
            __syncwarp();
            double* dst = g.xbuf + st * g.buf_doubles;
            const double* gsrc = src + g.r0 * k + kk0;
            // coalesced 16-byte pieces: a warp instruction covers 4 rows x 128 B
            const int pr = n >> 1, np = g.nrows * pr;
            for (int idx = lane; idx < np; idx += 32) {
                const int rr = idx / pr, u = idx - rr * pr;
                cp_async16(dst + rr * KCP + 2 * u, gsrc + (int64_t)rr * k + 2 * u);
            }
            // each producer lane's copies arrive on `full` when they land (count 32)
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(pp.full + 8u * st) : "memory");
        }
    } else {
        const int item = g.self;
        const bool act = item < nitems;
        const int cgi = act ? item / g.nrows : 0, r = act ? item - cgi * g.nrows : 0;
        const int c0 = cgi * CG;
        const int cn = act ? min(CG, wn - c0) : 0;
        double a[CG];
#pragma unroll
        for (int u = 0; u < CG; ++u) {
            a[u] = 0.0;
            if (u < cn) {
                const int c = c0 + u;
                const double o = g.old_m[(g.r0 + r) * k + g.bn + c];
                a[u] = g.use_diag ? dmul(o, lds64(qb + 8u * ((g.bn + c) * g.tq + c))) : o;
            }
        }
        for (int ch = 0; ch < nch; ++ch) {
            const unsigned it = pp.it + ch, st = it % ST, ph = (it / ST) & 1u;
            mbar_wait(pp.full + 8u * st, ph);
            if (act) {
                const double* src; int kk0, n;
                chunk(ch, src, kk0, n);
                const unsigned xs = pp.bufs + 8u * (st * g.buf_doubles + r * KCP);
                const unsigned qc = qb + 8u * (kk0 * g.tq + c0);
                if (n == KC) {
#pragma unroll
                    for (int j = 0; j < KC; j += 2) {
                        const double2 xx = lds128(xs + 8u * j);
#pragma unroll
                        for (int u = 0; u < CG; u += 2) {
                            // padded coefficient columns (c >= wn) are 0: harmless, never stored
                            const double2 qa = lds128(qc + 8u * (j * g.tq + u));
                            const double2 qn = lds128(qc + 8u * ((j + 1) * g.tq + u));
                            a[u] = M::madd(a[u], -1.0 * qa.x, xx.x);
                            a[u + 1] = M::madd(a[u + 1], -1.0 * qa.y, xx.x);
                            a[u] = M::madd(a[u], -1.0 * qn.x, xx.y);
                            a[u + 1] = M::madd(a[u + 1], -1.0 * qn.y, xx.y);
                        }
                    }
                } else {
                    for (int j = 0; j < n; ++j) {
                        const double x = lds64(xs + 8u * j);
#pragma unroll
                        for (int u = 0; u < CG; u += 2) {
                            const double2 qa = lds128(qc + 8u * (j * g.tq + u));
                            a[u] = M::madd(a[u], -1.0 * qa.x, x);
                            a[u + 1] = M::madd(a[u + 1], -1.0 * qa.y, x);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(pp.empty + 8u * st);
        }
#pragma unroll
        for (int u = 0; u < CG; ++u)
            if (u < cn) g.dst[r * g.ldt + c0 + u] = a[u];
    }
    pp.it += nch;
}

}  // namespace plnmf

