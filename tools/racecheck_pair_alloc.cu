// Minimal repro for compute-sanitizer racecheck's report on the CTA-pair kernels:
// a 2-CTA cluster in which warp 1 of each CTA allocates tensor memory with
// tcgen05.alloc.cta_group::2 (the allocator writes the TMEM address into a shared-
// memory slot), followed by the allocation protocol of the PTX ISA --
// tcgen05.fence::before_thread_sync, a cluster barrier, tcgen05.fence::after_thread_sync --
// and then every thread reads the slot.  The same protocol with cta_group::1 (and a
// CTA barrier) is the control.  Nothing else happens, so a hazard reported here is
// about the allocation write itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/rc tools/racecheck_pair_alloc.cu
//   compute-sanitizer --tool racecheck /tmp/rc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int PAIR>
__device__ __forceinline__ void alloc_body(unsigned* out)
{
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 1) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t = slot;                          // every thread reads the allocated address
    if (threadIdx.x == 0) out[blockIdx.x] = t;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(t) : "memory");
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(t) : "memory");
    }
}

__global__ void __cluster_dims__(2, 1, 1) alloc_pair(unsigned* out) { alloc_body<1>(out); }
__global__ void alloc_single(unsigned* out) { alloc_body<0>(out); }

int main()
{
    unsigned* out;
    unsigned host[64] = {};
    cudaMalloc(&out, 64 * sizeof(unsigned));
    for (int pair = 0; pair < 2; ++pair) {
        if (pair) alloc_pair<<<8, 128>>>(out);
        else alloc_single<<<8, 128>>>(out);
        cudaError_t e = cudaGetLastError();
        cudaError_t e2 = cudaDeviceSynchronize();
        cudaMemcpy(host, out, sizeof(host), cudaMemcpyDeviceToHost);
        printf("cta_group::%d: launch %s, sync %s, tmem addr[0] = 0x%x\n", pair ? 2 : 1, cudaGetErrorString(e),
               cudaGetErrorString(e2), host[0]);
    }
    return 0;
}
