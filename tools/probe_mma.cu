// Microbenchmark of raw tcgen05.mma throughput on B200 for the instruction
// shapes the emulated-SGEMM kernels use (no splitting, no epilogue):
//   pair (cta_group::2) M=256 x N in {64, 128, 256}, A from SMEM (SS) or TMEM (TS)
//   single (cta_group::1) M=128 x N in {64, 128, 256}, SS
// One elected thread per CTA (leader for pairs) issues ITERS x 3 MMAs (K=16 f16),
// commits, waits.  Prints dense FP16 TFLOP/s per configuration as JSON lines.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2308_15152_b200/csrc/sm100_ptx.cuh"

using namespace emu;

template <bool PAIR, bool TS, int N>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const uint32_t warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 0) {
        if (PAIR) ptx::tmem_alloc_pair<512>(&slot);
        else ptx::tmem_alloc<512>(&slot);
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    if (PAIR) ptx::cluster_sync(); else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tbase = slot;
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0;
    long long t0 = clock64();
    if (warp == 0 && rank == 0 && ptx::elect_one()) {
        const uint32_t M = PAIR ? 256 : 128;
        const uint32_t idesc = ptx::instr_desc(0u, TS ? 0u : 1u, 0u, M, N);
        const uint32_t sb = ptx::smem_u32(smem);
        const uint64_t dA = ptx::smem_desc(sb, 1024, 2048, 2);
        const uint64_t dB = ptx::smem_desc(sb + 16384, 16, 512, 4);
        const uint32_t d0 = tbase, d1 = tbase + (N <= 128 ? 128 : N);   // D_hi, D_corr (N <= 128 for TS)
        const uint32_t a_t = tbase + 384;                          // A in TMEM (TS)
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const uint32_t d = j == 0 ? d0 : d1;
                if (PAIR) {
                    if (TS) ptx::mma_f16_pair_ts(d, a_t, dB, idesc, 1u);
                    else ptx::mma_f16_pair(d, dA, dB, idesc, 1u);
                } else {
                    ptx::mma_f16(d, dA, dB, idesc, 1u);
                }
            }
        }
        if (PAIR) ptx::tc_commit_pair(&bar, 0x3); else ptx::tc_commit(&bar);
    }
    if (warp == 0 && (rank == 0 || PAIR)) {
        // both CTAs of a pair receive the multicast commit
        if (!PAIR && rank != 0) {}
        ptx::mbar_wait(&bar, 0);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
    ptx::tc_fence_before();
    if (PAIR) ptx::cluster_sync(); else __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        if (PAIR) ptx::tmem_dealloc_pair<512>(tbase);
        else ptx::tmem_dealloc<512>(tbase);
    }
}

template <bool PAIR, bool TS, int N>
void run(const char* name)
{
    auto k = mma_loop<PAIR, TS, N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    unsigned long long* cyc;
    cudaMallocManaged(&cyc, 8);
    const int iters = 4096;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 66 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PAIR ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
        *cyc = 0;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t err = cudaLaunchKernelEx(&cfg, k, iters, cyc);
        cudaEventRecord(e1);
        cudaError_t err2 = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double M = PAIR ? 256 : 128;
        const double ctas_issuing = PAIR ? 74 : 148;
        const double flops = 2.0 * M * N * 16 * 3 * iters * ctas_issuing;
        const double cyc_per_mma = (double)*cyc / (PAIR ? 74 : 148) / (3.0 * iters);
        if (rep == 1)
            printf("{\"probe\": \"%s\", \"err\": \"%s/%s\", \"ms\": %.3f, \"tflops\": %.1f, \"clk_per_mma\": %.1f}\n",
                   name, cudaGetErrorString(err), cudaGetErrorString(err2), ms, flops / ms / 1e9, cyc_per_mma);
    }
}

int main()
{
    run<true, true, 96>("pair_ts_m256_n96");
    run<true, true, 112>("pair_ts_m256_n112");
    run<true, false, 96>("pair_ss_m256_n96");
    run<true, false, 112>("pair_ss_m256_n112");
    run<true, true, 80>("pair_ts_m256_n80");
    run<true, false, 64>("pair_ss_m256_n64");
    run<true, false, 128>("pair_ss_m256_n128");
    run<true, false, 256>("pair_ss_m256_n256");
    run<true, true, 64>("pair_ts_m256_n64");
    run<true, true, 128>("pair_ts_m256_n128");
    run<false, false, 64>("single_ss_m128_n64");
    run<false, false, 128>("single_ss_m128_n128");
    run<false, false, 256>("single_ss_m128_n256");
    return 0;
}
