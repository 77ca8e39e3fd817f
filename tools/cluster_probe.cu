// Max co-resident clusters for a 1-CTA-per-SM kernel (512 threads, ~200 KB smem)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_probe.bin tools/cluster_probe.cu
#include <cstdio>
__global__ void __launch_bounds__(512, 1) k(double* o) {
    extern __shared__ double s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) o[blockIdx.x] = s[5];
}
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 8);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
        printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
    }
}
