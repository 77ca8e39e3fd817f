// The staged look-ahead GEMM of the tiled updates (update.cu) and its
// shared-memory / cp.async helpers; a header so tools/gemm_bench.cu can time
// it in isolation.
#pragma once

#include "common.cuh"

namespace plnmf {

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


// ---------------------------------------------------------------- staged look-ahead GEMM
// The look-ahead builds the next tile's accumulators of this CTA's rows:
//   dst(r, c) = init(old(r, bn+c))                       init_new_accumulator, tiled.cpp:44
//             + sum_{kk in [en, k)}    -coeff(kk, bn+c) * old(r, kk)    phase 1, tiled.cpp:58-60
//             + sum_{kk in [0, bprev)} -coeff(kk, bn+c) * out(r, kk)    phase 3 of earlier tiles
// every element's terms in the reference's order (kk ascending, phase 1 then
// phase 3), so Math::exact stays bit-identical.  GemmArgs describes one call;
// kGemmKC / kGemmStages are the chunking of the group-staged variants kept in
// tools/gemm_variants.cuh (measured, not used).
constexpr int kGemmKC = 8, kGemmKCP = kGemmKC + 2, kGemmStages = 3;
constexpr int kPrivKC = 16;  // lookahead_gemm_private chunk width in the engine

struct GemmArgs {
    double* dst;
    int ldt;
    const double* q;  // shared: coeff(kk, bn + c) at q[kk * tq + c]
    int tq;
    int bn, en, bprev, use_diag;
    const double* old_m;
    const double* out;
    int64_t r0;
    int nrows, k;
    double* xbuf;  // shared: kGemmStages x buf_doubles
    int buf_doubles;
    int count, self, bar;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double2 lds128(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

}  // namespace plnmf

namespace plnmf {

// Private-staging variant: each thread stages its item's row chunk into ITS
// OWN ring (buffer index = thread; 8-byte aligned rows: cp.async 16 B when k
// is even) and consumes it, so the ring needs only per-thread
// cp.async.wait_group — no group barrier, and no buffer is shared between
// threads (two items of one row live in different threads' rings).  One row x
// CG columns per item; a thread walks items self, self + count, ... .
template <class M, int CG, int KC, int ST, int TQC = 0>
__device__ __forceinline__ void lookahead_gemm_private(const GemmArgs& g) {
    constexpr int KCP = KC + 2;
    const int tq = TQC > 0 ? TQC : g.tq;  // compile-time panel stride lets loads use immediate offsets
    const int wn = g.en - g.bn, k = g.k;
    const int ncg = (wn + CG - 1) / CG;
    const int nitems = g.nrows * ncg;
    const int nch1 = (k - g.en + KC - 1) / KC, nch = nch1 + (g.bprev + KC - 1) / KC;
    const unsigned qb = smem_u32(g.q);
    const bool vec = (k & 1) == 0;
    double* myrow = g.xbuf + g.self * KCP;
    for (int item = g.self; item < nitems; item += g.count) {
    const int cgi = item / g.nrows, r = item - cgi * g.nrows;
    const int c0 = cgi * CG, cn = min(CG, wn - c0);
    auto chunk = [&](int ch, const double*& src, int& kk0, int& n) {
        if (ch < nch1) { src = g.old_m; kk0 = g.en + ch * KC; n = min(KC, k - kk0); }
        else { src = g.out; kk0 = (ch - nch1) * KC; n = min(KC, g.bprev - kk0); }
    };
    auto stage = [&](int ch) {
        if (ch < nch) {
            const double* src; int kk0, n;
            chunk(ch, src, kk0, n);
            double* xs = myrow + (ch % ST) * g.buf_doubles;
            const double* gs = src + (g.r0 + r) * k + kk0;
            if (vec && ((kk0 | n) & 1) == 0) {
                for (int u = 0; u < n; u += 2) cp_async16(xs + u, gs + u);
            } else {
                for (int u = 0; u < n; ++u) cp_async8(xs + u, gs + u);
            }
        }
        cp_async_commit();
    };
    double a[CG];
#pragma unroll
    for (int u = 0; u < CG; ++u) {
        a[u] = 0.0;
        if (u < cn) {
            const int c = c0 + u;
            const double o = g.old_m[(g.r0 + r) * k + g.bn + c];
            a[u] = g.use_diag ? dmul(o, lds64(qb + 8u * ((g.bn + c) * tq + c))) : o;
        }
    }
#pragma unroll
    for (int st = 0; st < ST - 1; ++st) stage(st);
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait<ST - 2>();
        stage(ch + ST - 1);  // refills the slot consumed at ch - 1 (this thread's own)
        const double* src; int kk0, n;
        chunk(ch, src, kk0, n);
        const unsigned xs = smem_u32(myrow + (ch % ST) * g.buf_doubles);
        const unsigned qc = qb + 8u * (kk0 * tq + c0);
        if (n == KC) {
#pragma unroll
            for (int j = 0; j < KC; j += 2) {
                const double2 xx = lds128(xs + 8u * j);
#pragma unroll
                for (int u = 0; u < CG; u += 2) {
                    const double2 qa = lds128(qc + 8u * (j * tq + u));
                    const double2 qn = lds128(qc + 8u * ((j + 1) * tq + u));
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
                    const double2 qa = lds128(qc + 8u * (j * tq + u));
                    a[u] = M::madd(a[u], -1.0 * qa.x, x);
                    a[u + 1] = M::madd(a[u + 1], -1.0 * qa.y, x);
                }
            }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int u = 0; u < CG; ++u)
        if (u < cn) g.dst[r * g.ldt + c0 + u] = a[u];
    }
}

}  // namespace plnmf

namespace plnmf {

// Resident-rows variant (H update: the CTA's whole row block of the old
// factor sits in shared memory, rows ld apart, finished tiles written back in
// place): no staging and no barriers.  A thread item is ONE column c (lanes =
// consecutive columns, so the row operands of a kk are broadcast within each
// 16-lane half and the coefficient load is one conflict-free wavefront) and up
// to RG rows g, g + ng, g + 2 ng, ... (ng = count / 16 row groups).
// Per-element order as lookahead_gemm_private: bit-identical under Math::exact.
template <int OFF>
__device__ __forceinline__ double lds64_at(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
    return v;
}

template <int OFF>
__device__ __forceinline__ double2 lds128_at(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y) : "r"(a), "n"(OFF));
    return v;
}

template <class M, int RG>
__device__ __forceinline__ void lookahead_gemm_resident(const GemmArgs& g, const double* resid, int ld) {
    const int wn = g.en - g.bn, k = g.k;
    const int ng = g.count / 16;  // row groups
    const int c = g.self % 16, grp = g.self / 16;
    if (c >= wn || grp >= ng || grp >= g.nrows) return;
    const unsigned qb = smem_u32(g.q), xb = smem_u32(resid);
    // rows past the block recompute the last row (no predicates in the loop);
    // only the first rn are stored
    int rr[RG];
    int rn = 0;
#pragma unroll
    for (int i = 0; i < RG; ++i) {
        const int r = grp + i * ng;
        if (r < g.nrows) rn = i + 1;
        rr[i] = min(r, g.nrows - 1);
    }
    double a[RG];
#pragma unroll
    for (int i = 0; i < RG; ++i) {
        const double o = resid[rr[i] * ld + g.bn + c];
        a[i] = g.use_diag ? dmul(o, lds64(qb + 8u * ((g.bn + c) * g.tq + c))) : o;
    }
    // addresses advance by increments; the row operands of 4 consecutive kk
    // are immediate offsets from one base
    const unsigned qs = 8u * g.tq, qs2 = 2u * qs, qs3 = 3u * qs, qs4 = 4u * qs;
    auto seg = [&](int k0, int k1) {
        unsigned qa = qb + 8u * (k0 * g.tq + c);
        unsigned xa[RG];
#pragma unroll
        for (int i = 0; i < RG; ++i) xa[i] = xb + 8u * (rr[i] * ld + k0);
        int n = k1 - k0;
        if (((ld | k0) & 1) == 0) {
            // 16-byte aligned rows: the row operands of 4 consecutive kk as two LDS.128
            // (the look-ahead is shared-memory issue bound: ncu short_sb / mio stalls)
            for (; n >= 4; n -= 4) {
                const double q0 = -1.0 * lds64(qa), q1 = -1.0 * lds64(qa + qs), q2 = -1.0 * lds64(qa + qs2),
                             q3 = -1.0 * lds64(qa + qs3);
#pragma unroll
                for (int i = 0; i < RG; ++i) {
                    const double2 x01 = lds128_at<0>(xa[i]), x23 = lds128_at<16>(xa[i]);
                    a[i] = M::madd(a[i], q0, x01.x);
                    a[i] = M::madd(a[i], q1, x01.y);
                    a[i] = M::madd(a[i], q2, x23.x);
                    a[i] = M::madd(a[i], q3, x23.y);
                    xa[i] += 32u;
                }
                qa += qs4;
            }
        }
        for (; n >= 4; n -= 4) {
            const double q0 = -1.0 * lds64(qa), q1 = -1.0 * lds64(qa + qs), q2 = -1.0 * lds64(qa + qs2),
                         q3 = -1.0 * lds64(qa + qs3);
#pragma unroll
            for (int i = 0; i < RG; ++i) {
                a[i] = M::madd(a[i], q0, lds64_at<0>(xa[i]));
                a[i] = M::madd(a[i], q1, lds64_at<8>(xa[i]));
                a[i] = M::madd(a[i], q2, lds64_at<16>(xa[i]));
                a[i] = M::madd(a[i], q3, lds64_at<24>(xa[i]));
                xa[i] += 32u;
            }
            qa += qs4;
        }
        for (; n > 0; --n) {
            const double q = -1.0 * lds64(qa);
#pragma unroll
            for (int i = 0; i < RG; ++i) {
                a[i] = M::madd(a[i], q, lds64(xa[i]));
                xa[i] += 8u;
            }
            qa += qs;
        }
    };
    seg(g.en, k);     // phase 1: old values of the columns right of the tile
    seg(0, g.bprev);  // phase 3 of the tiles before the previous one: finished values
#pragma unroll
    for (int i = 0; i < RG; ++i)
        if (i < rn) g.dst[rr[i] * g.ldt + c] = a[i];
}

}  // namespace plnmf
