// TMEM read / write throughput probe (tools only, not the product).
// One CTA per SM allocates all 512 TMEM columns; W warps (warp w reads lane
// quadrant w % 4) loop over tcgen05.ld.32x32b.xX (NB loads in flight per
// tcgen05.wait::ld) or tcgen05.st.32x32b.xX.  Prints one JSON line per variant:
// bytes per SM-cycle = W * 32 lanes * X cols * 4 B * iterations / cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_tmem tools/probe_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t (&r)[X]);


template <>
__device__ __forceinline__ void ld<16>(uint32_t t, uint32_t (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(t));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t t, uint32_t (&r)[32])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(t));
}
// 16x256b.x4: 16 lanes x 4 x 256 bits per warp, 16 registers per thread
__device__ __forceinline__ void ld256(uint32_t t, uint32_t (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(t));
}
template <int X>
__device__ __forceinline__ void st(uint32_t taddr, const uint32_t (&r)[X]);
template <>
__device__ __forceinline__ void st<16>(uint32_t t, const uint32_t (&r)[16])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(t), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                   "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
                 : "memory");
}

template <int W, int X, int NB, bool STORE, bool S256 = false>
__global__ void __launch_bounds__(W * 32, 1) tmem_kernel(int iters, unsigned long long* cyc, uint32_t* sink)
{
    __shared__ uint32_t slot;
    const uint32_t warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = slot + (((warp & 3) * 32u) << 16);
    const uint32_t col0 = (warp / 4) * 64;   // warps sharing a quadrant read different columns
    uint32_t acc = 0;
    uint32_t r[NB][X];
#pragma unroll
    for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int i = 0; i < X; ++i) r[b][i] = threadIdx.x * 7 + i + b;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        constexpr uint32_t CW = S256 ? 32 : X;   // columns per load
        const uint32_t c = (col0 + (uint32_t)it * (NB * CW)) & 511u;
        if (STORE) {
#pragma unroll
            for (int b = 0; b < NB; ++b) st<X>(base + ((c + b * CW) & 511u), r[b]);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        } else {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                if constexpr (S256) ld256(base + ((c + b * CW) & 511u), reinterpret_cast<uint32_t(&)[16]>(r[b]));
                else ld<X>(base + ((c + b * CW) & 511u), r[b]);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int b = 0; b < NB; ++b) acc ^= r[b][0] ^ r[b][X - 1];
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

template <int W, int X, int NB, bool STORE, bool S256 = false>
static void run(const char* name)
{
    const int grid = 148, iters = 4096;
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, grid * sizeof(unsigned long long));
    cudaMalloc(&sink, grid * W * 32 * sizeof(uint32_t));
    tmem_kernel<W, X, NB, STORE, S256><<<grid, W * 32>>>(16, cyc, sink);   // warm-up
    tmem_kernel<W, X, NB, STORE, S256><<<grid, W * 32>>>(iters, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < grid; ++i) mean += (double)h[i] / grid;
    // 16x256b.x4 moves 16 regs x 32 threads x 4 B per warp as well (16 lanes x 32 columns)
    const double bytes = (double)W * 32 * X * 4 * NB * iters;
    printf("{\"probe\": \"%s\", \"op\": \"%s\", \"warps\": %d, \"x\": %d, \"in_flight\": %d, \"cycles\": %.0f, "
           "\"bytes_per_cycle_per_sm\": %.1f, \"err\": \"%s\"}\n",
           name, STORE ? "st" : "ld", W, X, NB, mean, bytes / mean, cudaGetErrorString(e));
    cudaFree(cyc);
    cudaFree(sink);
}

int main()
{
    run<4, 16, 1, false>("ld");
    run<4, 16, 2, false>("ld");
    run<4, 32, 1, false>("ld");
    run<4, 32, 2, false>("ld");
    run<8, 16, 1, false>("ld");
    run<8, 16, 2, false>("ld");
    run<8, 32, 2, false>("ld");
    run<16, 16, 1, false>("ld");
    run<16, 16, 2, false>("ld");
    run<16, 32, 1, false>("ld");
    run<4, 16, 2, false, true>("ld16x256b.x4");
    run<16, 16, 2, false, true>("ld16x256b.x4");
    run<4, 16, 1, true>("st");
    run<4, 16, 4, true>("st");
    run<16, 16, 2, true>("st");
    return 0;
}
