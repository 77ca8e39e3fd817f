// L2 bandwidth ceilings for the SpMM roofline (bench.py reads the result from
// profiles/l2_peak.json):
//   stream   every CTA re-reads an L2-resident buffer with 16-byte loads
//   gather   the SpMM's access pattern: each warp reads whole 1,920-byte rows
//            (K = 240 doubles) at random row indices of a 21.7 MB operand
//            (the C2 Ht), 8-byte lanes (as spmm_csr) and 16-byte lanes
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2bw_bench.bin tools/l2bw_bench.cu
#include <cstdio>
#include <cstdint>

__global__ void stream_kernel(const double2* __restrict__ x, int64_t n2, int passes, double* out) {
    double s = 0.0;
    for (int p = 0; p < passes; ++p)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
            const double2 v = __ldcg(x + i);
            s += v.x + v.y;
        }
    if (s == 12345.678) *out = s;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

template <int VEC>
__global__ void gather_kernel(const double* __restrict__ x, int rows, int k, int per_warp, double* out) {
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    double s = 0.0;
    for (int i = 0; i < per_warp; i += 4) {
        double v[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = (int)(hash32(warp * 7919u + (uint32_t)(i + u)) % (uint32_t)rows);
            const double* xr = x + (int64_t)r * k;
            if (VEC == 1) {
#pragma unroll
                for (int g = 0; g < 8; ++g) v[u][g] = (lane + 32 * g < k) ? __ldg(xr + lane + 32 * g) : 0.0;
            } else {
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const int c = 2 * lane + 64 * g;
                    double2 t = make_double2(0.0, 0.0);
                    if (c + 1 < k) t = __ldg(reinterpret_cast<const double2*>(xr + c));
                    v[u][2 * g] = t.x;
                    v[u][2 * g + 1] = t.y;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int g = 0; g < 8; ++g) s += v[u][g];
    }
    if (s == 12345.678) *out = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double* out;
    cudaMalloc(&out, 8);
    {
        const int64_t bytes = 32ll << 20;
        double2* x;
        cudaMalloc(&x, bytes);
        cudaMemset(x, 0, bytes);
        const int passes = 50;
        stream_kernel<<<sms * 4, 512>>>(x, bytes / 16, 2, out);
        cudaEventRecord(a);
        stream_kernel<<<sms * 4, 512>>>(x, bytes / 16, passes, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"stream_l2_gbs\": %.1f, ", (double)bytes * passes / (ms * 1e-3) / 1e9);
        cudaFree(x);
    }
    {
        const int rows = 11314, k = 240;
        double* x;
        cudaMalloc(&x, sizeof(double) * rows * k);
        cudaMemset(x, 0, sizeof(double) * rows * k);
        const int per_warp = 256;
        const int blocks = sms * 8, threads = 256;
        const double nbytes = (double)blocks * (threads / 32) * per_warp * k * 8.0;
        float ms1, ms2;
        gather_kernel<1><<<blocks, threads>>>(x, rows, k, per_warp, out);
        cudaEventRecord(a);
        gather_kernel<1><<<blocks, threads>>>(x, rows, k, per_warp, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms1, a, b);
        gather_kernel<2><<<blocks, threads>>>(x, rows, k, per_warp, out);
        cudaEventRecord(a);
        gather_kernel<2><<<blocks, threads>>>(x, rows, k, per_warp, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms2, a, b);
        printf("\"gather_l2_gbs_8B\": %.1f, \"gather_l2_gbs_16B\": %.1f, ", nbytes / (ms1 * 1e-3) / 1e9,
               nbytes / (ms2 * 1e-3) / 1e9);
        printf("\"what\": \"stream: 16-B __ldcg re-reads of a 32 MiB L2-resident buffer (%d CTAs x 512); gather: "
               "random 1920-B rows of an 11314x240 f64 operand (the C2 Ht), one row per warp per step, 4 rows "
               "in flight\"}\n", sms * 4);
        cudaFree(x);
    }
    return 0;
}
