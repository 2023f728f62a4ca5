// How many thread-block clusters of 2 / 4 / 8 CTAs (one CTA per SM: ~227 KB of shared
// memory each, like the GEMM kernels) can be co-resident on this GPU
// (cudaOccupancyMaxActiveClusters): the grid of a persistent cluster kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_cluster tools/probe_cluster.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dummy(int* x)
{
    extern __shared__ int s[];
    if (threadIdx.x == 0 && x) x[blockIdx.x] = s[0];
}

int main()
{
    const int smem = 227 * 1024;
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int cl : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl * 64);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("{\"cluster\": %d, \"max_active_clusters\": %d, \"sms_used\": %d, \"sms\": %d, \"err\": \"%s\"}\n", cl, n,
               n * cl, sms, cudaGetErrorString(e));
    }
    return 0;
}
