// Cross-GPU exchange over peer memory for the sharded engine.
//
// Every rank owns one device allocation, its "window" (layout in
// PeerLayout), which it exports with a CUDA IPC handle; every other rank maps
// it (cudaIpcOpenMemHandle: NVLink P2P on the B200 box) so a kernel on rank g
// can store straight into rank p's window.  Nothing here calls NCCL: the two
// kinds of traffic of the sharded iteration are
//
//   * the per-column norm of the W update (proj/src/tiled.cpp:129-146: column
//     t+1 cannot start before sum_g ||W_g[:,t]||^2 is known) — inside the
//     persistent W kernel: each rank's CTA 0 stores its rank's sum into slot
//     (t, rank) of every rank's window and releases an epoch flag; every CTA
//     of every rank acquires the world's flags in its OWN window and adds the
//     values in rank order (world_sum), so all ranks get the same bits;
//   * the factor / Gram all-gathers — a push kernel stores the rank's slice
//     into every peer's window (16-byte stores over NVLink) and the last CTA
//     releases the channel's epoch flag there; consumers wait for the world's
//     flags in their own window (ag_wait) before reading.
//
// Epochs make the slots reusable without resets: every rank performs the
// same sequence of pushes and W updates, so the k-th use of a channel carries
// epoch k on all ranks; a flag equal to the current epoch means "this use's
// data is in place".  Waits are bounded (kPeerTimeoutNs): a missing peer sets
// the window's error word instead of hanging the GPU, and the host raises it.
#pragma once

#include "common.cuh"

namespace plnmf {

constexpr int kMaxWorld = 8;                 // one NVLink/NVSwitch node
constexpr int kWRep = 4;                     // replicas of each norm slot (spreads the 148-CTA poll)
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;  // default

enum PeerChannel : int { kChanW = 0, kChanHt = 1, kChanS = 2, kChanQ = 3, kChanPW = 4, kChannels = 5 };

struct PeerPtrs {
    void* p[kMaxWorld];
};

// Arguments of the in-kernel norm exchange (by value in the kernel params).
struct WorldXch {
    int world = 1, rank = 0;
    unsigned epoch = 0;
    unsigned long long timeout_ns = kPeerTimeoutNs;
    int* error = nullptr;            // this rank's window error word
    double* vals[kMaxWorld] = {};    // rank p's norm value slots (in p's window)
    unsigned* flags[kMaxWorld] = {}; // rank p's norm flag slots
};

__host__ __device__ inline int64_t xch_slot(int64_t t, int rep, int src) {
    return (t * kWRep + rep) * kMaxWorld + src;
}

__device__ __forceinline__ unsigned long long peer_clock_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void st_release_sys_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys_f64(double* p, double v) {
    asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys_f64(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_volatile_s32(const int* p) { return *(const volatile int*)p; }

// Spin until *flag == epoch or the timeout; true when the flag arrived.
__device__ __forceinline__ bool wait_flag(const unsigned* flag, unsigned epoch, int* error,
                                          unsigned long long timeout_ns) {
    if (ld_acquire_sys_u32(flag) == epoch) return true;
    if (ld_volatile_s32(error)) return false;
    const unsigned long long t0 = peer_clock_ns();
    while (ld_acquire_sys_u32(flag) != epoch) {
        if (peer_clock_ns() - t0 > timeout_ns) {
            atomicExch(error, 1);
            return false;
        }
    }
    return true;
}

// A collective fused into a producing kernel: the kernel stores each finished
// piece of its output into every other rank's window as well (dst: this rank's
// slice there, same layout as the local output), and the last CTA to finish
// releases the channel's epoch flag in every window (flag[p]).
struct FusedPush {
    int world = 1, rank = 0;
    unsigned epoch = 0;
    unsigned* done = nullptr;           // zeroed local CTA counter
    double* dst[kMaxWorld] = {};
    unsigned* flag[kMaxWorld] = {};
};

// the end of a kernel that pushed with f: every CTA calls it (all threads)
__device__ __forceinline__ void fused_push_finish(const FusedPush& f) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();  // this CTA's peer stores before its count
        const unsigned prev = atomicAdd(f.done, 1u);
        if (prev == gridDim.x - 1) {
            *f.done = 0;
            __threadfence_system();
            for (int p = 0; p < f.world; ++p) st_release_sys_u32(f.flag[p], f.epoch);
        }
    }
}

// The world's sum for column t, called by one full warp of every CTA after
// the rank-local grid exchange has given every CTA the same local sum.  The
// world's values are added in rank order by every CTA of every rank.
__device__ __forceinline__ double world_sum(double s_local, int t, const WorldXch& x) {
    const int lane = lane_id();
    if (blockIdx.x == 0) {
        for (int i = lane; i < x.world * kWRep; i += kWarp) {
            const int p = i / kWRep, rep = i % kWRep;
            const int64_t slot = xch_slot(t, rep, x.rank);
            st_relaxed_sys_f64(x.vals[p] + slot, s_local);
            st_release_sys_u32(x.flags[p] + slot, x.epoch);  // orders the value store before it
        }
    }
    const int rep = blockIdx.x % kWRep;
    double v = 0.0;
    if (lane < x.world) {
        const int64_t slot = xch_slot(t, rep, lane);
        wait_flag(x.flags[x.rank] + slot, x.epoch, x.error, x.timeout_ns);
        v = ld_relaxed_sys_f64(x.vals[x.rank] + slot);
    }
    double s = __shfl_sync(0xffffffffu, v, 0);
    for (int q = 1; q < x.world; ++q) s = dadd(s, __shfl_sync(0xffffffffu, v, q));
    return s;
}

}  // namespace plnmf
