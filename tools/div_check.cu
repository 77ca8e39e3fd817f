// Exhaustive-sampling check that the reciprocal + one-fma correction
//   y = RN(1/b); q0 = RN(a*y); r = fma(-q0, b, a); q = fma(r, y, q0)
// reproduces the correctly rounded quotient RN(a/b) (= __ddiv_rn) bit for bit
// on the W update's domain (positive, normal operands and quotients).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/div_check.bin tools/div_check.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
// random positive double: mantissa uniform, exponent uniform in [emin, emax]
__device__ __forceinline__ double rnd(uint64_t s, int emin, int emax) {
    const uint64_t m = mix(s) & ((1ull << 52) - 1);
    const int e = emin + (int)(mix(s ^ 0x5555) % (uint64_t)(emax - emin + 1));
    return __longlong_as_double((long long)(((uint64_t)(e + 1023) << 52) | m));
}

__global__ void check(uint64_t base, int64_t n, int emin, int emax, unsigned long long* bad, double* ex) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t s = base + 2 * (uint64_t)i;
        double a = rnd(s, emin, emax), b = rnd(s + 1, emin, emax);
        if ((mix(s) & 7) == 0) {  // mantissa-edge cases: powers of two and all-ones mantissas
            const uint64_t t = mix(s ^ 0x1234);
            a = __longlong_as_double((__double_as_longlong(a) & ~((1ll << 52) - 1)) | ((t & 1) ? ((1ll << 52) - 1) : 0));
            b = __longlong_as_double((__double_as_longlong(b) & ~((1ll << 52) - 1)) | ((t & 2) ? ((1ll << 52) - 1) : 1));
        }
        const double want = __ddiv_rn(a, b);
        const double y = __drcp_rn(b);
        const double q0 = __dmul_rn(a, y);
        const double r = __fma_rn(-q0, b, a);
        const double got = __fma_rn(r, y, q0);
        if (__double_as_longlong(got) != __double_as_longlong(want)) {
            const unsigned long long k = atomicAdd(bad, 1ull);
            if (k < 4) {
                ex[4 * k] = a;
                ex[4 * k + 1] = b;
                ex[4 * k + 2] = want;
                ex[4 * k + 3] = got;
            }
        }
    }
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMalloc(&bad, 8);
    cudaMalloc(&ex, 16 * 8);
    struct R { int emin, emax; } ranges[] = {{-60, 60}, {-500, 500}, {-1000, 1000}, {-2, 2}};
    for (auto rg : ranges) {
        cudaMemset(bad, 0, 8);
        const int64_t n = 1ll << 33;
        check<<<148 * 16, 256>>>(0x1234567ull * (rg.emax + 7), n, rg.emin, rg.emax, bad, ex);
        cudaDeviceSynchronize();
        unsigned long long hb;
        double he[16];
        cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(he, ex, sizeof(he), cudaMemcpyDeviceToHost);
        printf("exponents [%5d, %4d]: %lld pairs, %llu mismatches (%s)\n", rg.emin, rg.emax, (long long)n, hb,
               cudaGetErrorString(cudaGetLastError()));
        for (unsigned long long i = 0; i < hb && i < 4; ++i)
            printf("   a=%.17g b=%.17g div=%.17g markstein=%.17g\n", he[4 * i], he[4 * i + 1], he[4 * i + 2],
                   he[4 * i + 3]);
    }
    return 0;
}
