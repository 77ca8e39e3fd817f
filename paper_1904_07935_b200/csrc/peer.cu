// The sharded engine's peer-memory collectives (peer.cuh): the window layout,
// the push all-gather, the flag wait, the rank-ordered sum of gathered
// partials, and the index remap of the shard blocks onto the padded window
// layout.
#include "common.cuh"
#include "kernels.cuh"
#include "peer.cuh"

namespace plnmf {
namespace {

constexpr int kPushThreads = 512;

// dst.p[p] already points at this rank's slice in rank p's window; the last
// CTA to finish releases the channel flag in every window (threadfence
// reduction at system scope: every CTA fences its stores before it counts
// itself done, the last one fences again before the release stores).
template <class V>
__global__ void __launch_bounds__(kPushThreads) push_kernel(const V* __restrict__ src, int64_t n, PeerPtrs dst,
                                                            int world, int rank, int skip_self, PeerPtrs flag,
                                                            unsigned epoch, unsigned* done) {
    const int64_t stride = (int64_t)gridDim.x * kPushThreads;
    for (int64_t i = (int64_t)blockIdx.x * kPushThreads + threadIdx.x; i < n; i += stride) {
        const V v = src[i];
#pragma unroll
        for (int p = 0; p < kMaxWorld; ++p)  // constant indices: the peer pointers stay in registers
            if (p < world && !(skip_self && p == rank)) static_cast<V*>(dst.p[p])[i] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned prev = atomicAdd(done, 1u);
        if (prev == gridDim.x - 1) {
            *done = 0;  // ready for the next push (stream order)
            __threadfence_system();
            for (int p = 0; p < world; ++p) st_release_sys_u32(static_cast<unsigned*>(flag.p[p]), epoch);
        }
    }
}

__global__ void wait_kernel(const unsigned* flags, int world, unsigned epoch, int* error,
                            unsigned long long timeout_ns) {
    if ((int)threadIdx.x < world) wait_flag(flags + threadIdx.x, epoch, error, timeout_ns);
}

// out[i] = ((parts[0][i] + parts[1][i]) + parts[2][i]) + ... (rank order)
__global__ void sum_parts_kernel(const double* __restrict__ parts, int world, int64_t n, int64_t stride,
                                 double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = parts[i];
        for (int g = 1; g < world; ++g) s = dadd(s, parts[g * stride + i]);
        out[i] = s;
    }
}

// global index x of a balanced contiguous split (base, extra) -> owner * cap + (x - lo(owner))
__global__ void remap_kernel(int32_t* idx, int64_t nnz, int64_t base, int64_t extra, int64_t cap) {
    const int64_t big = extra * (base + 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = idx[i];
        int64_t owner, lo;
        if (x < big) {
            owner = x / (base + 1);
            lo = owner * (base + 1);
        } else {
            owner = extra + (x - big) / base;
            lo = big + (owner - extra) * base;
        }
        idx[i] = (int32_t)(owner * cap + (x - lo));
    }
}

inline unsigned grid_for(int64_t n, int threads, int cap) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cap, (n + threads - 1) / threads));
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

namespace kern {

PeerLayout peer_layout(int world, int64_t vcap, int64_t dcap, int64_t k) {
    PeerLayout L;
    L.world = world;
    L.vcap = vcap;
    L.dcap = dcap;
    L.k = k;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = align256(o + bytes);
        return at;
    };
    for (int i = 0; i < 2; ++i) L.off_wfull[i] = take(sizeof(double) * (size_t)(world * vcap * k));
    for (int i = 0; i < 2; ++i) L.off_hfull[i] = take(sizeof(double) * (size_t)(world * dcap * k));
    L.off_sparts = take(sizeof(double) * (size_t)(world * k * k));
    L.off_qparts = take(sizeof(double) * (size_t)(world * k * k));
    L.off_pw = take(sizeof(double) * kMaxWorld);
    L.off_xvals = take(sizeof(double) * (size_t)(k * kWRep * kMaxWorld));
    L.off_xflags = take(sizeof(unsigned) * (size_t)(k * kWRep * kMaxWorld));
    L.off_agflags = take(sizeof(unsigned) * kChannels * kMaxWorld);
    L.off_error = take(sizeof(int) * 4);
    L.total = o;
    return L;
}

int peer_push(cudaStream_t s, const void* src, int64_t bytes, const PeerPtrs& dst, int world, int rank,
              bool skip_self, const PeerPtrs& flag, unsigned epoch, unsigned* done, int sms) {
    bool v16 = (bytes % 16) == 0 && (reinterpret_cast<uintptr_t>(src) % 16) == 0;
    for (int p = 0; p < world; ++p) v16 = v16 && (reinterpret_cast<uintptr_t>(dst.p[p]) % 16) == 0;
    if (v16) {
        const int64_t n = bytes / 16;
        push_kernel<double2><<<grid_for(n, kPushThreads, 2 * sms), kPushThreads, 0, s>>>(
            static_cast<const double2*>(src), n, dst, world, rank, skip_self ? 1 : 0, flag, epoch, done);
    } else {
        const int64_t n = bytes / 8;
        push_kernel<double><<<grid_for(n, kPushThreads, 2 * sms), kPushThreads, 0, s>>>(
            static_cast<const double*>(src), n, dst, world, rank, skip_self ? 1 : 0, flag, epoch, done);
    }
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int peer_wait(cudaStream_t s, const unsigned* flags, int world, unsigned epoch, int* error,
              unsigned long long timeout_ns) {
    wait_kernel<<<1, kWarp, 0, s>>>(flags, world, epoch, error, timeout_ns);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int sum_parts(cudaStream_t s, const double* parts, int world, int64_t n, int64_t stride, double* out) {
    sum_parts_kernel<<<grid_for(n, 256, 592), 256, 0, s>>>(parts, world, n, stride, out);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

int remap_split_index(cudaStream_t s, int32_t* idx, int64_t nnz, int64_t n, int world, int64_t cap) {
    if (nnz <= 0 || world <= 1) return 0;
    remap_kernel<<<grid_for(nnz, 256, 4736), 256, 0, s>>>(idx, nnz, n / world, n % world, cap);
    PLNMF_CUDA_CHECK(cudaGetLastError());
    return 1;
}

}  // namespace kern
}  // namespace plnmf
