// HBM streaming probe for the c2 traffic pattern (tools only, not the product).
// Each CTA plays one half of a CTA pair of the A-stationary TS kernel with all
// compute removed: per (item, 128-row half) it TMA-loads A [128 m x 32 k] x 8 stages
// and, per n-tile (2), B [32 k x 64 n] x 8 stages through an S-deep ring, a
// consumer warp releases each stage on arrival, and each tile's 64 KB C block is
// TMA-stored from shared memory.  Variants change only the load boxes:
//   0: the kernel's boxes (A 128x32 no swizzle, B 32x64 SWIZZLE_128B)
//   1: B as [256 k x 8 n] boxes (whole 1 KB columns, 8 KB contiguous)
//   2: 1-D bulk copies of contiguous 16 KB / 8 KB chunks (upper bound)
// Prints one JSON line per variant and ring depth: GB/s = (A + B + C bytes) / time.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2308_15152_b200/csrc/sm100_ptx.cuh"

using namespace emu;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn enc()
{
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    return (EncodeFn)f;
}

static CUtensorMap map3(float* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
                        CUtensorMapSwizzle sw)
{
    CUtensorMap m;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {d0 * 4, d0 * d1 * 4};
    cuuint32_t box[3] = {b0, b1, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return m;
}

constexpr int ITEMS = 1024, M = 256, N = 256, K = 256;
constexpr uint32_t ASTG = 128 * 32 * 4, BSTG = 32 * 64 * 4, STG = ASTG + BSTG;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(ptx::smem_u32(dst)), "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar)) : "memory");
}

template <int VAR, int S>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tA,
                                                       const __grid_constant__ CUtensorMap tB,
                                                       const __grid_constant__ CUtensorMap tC,
                                                       const float* A, const float* B)
{
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* ring = smem;
    float* cst = reinterpret_cast<float*>(smem + S * STG);
    __shared__ uint64_t full[S], empty[S];
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    const int units = ITEMS * 2;   // (item, 128-row half)
    if (warp == 0) {
        if (ptx::elect_one()) {
            uint32_t s = 0, ph = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int b = u >> 1, r = u & 1;
                for (int j = 0; j < 2; ++j) {
                    for (int ks = 0; ks < K / 32; ++ks) {
                        ptx::mbar_wait(&empty[s], ph ^ 1);
                        uint8_t* dst = ring + s * STG;
                        const bool la = j == 0;
                        ptx::mbar_arrive_expect_tx(&full[s], (la ? ASTG : 0) + BSTG);
                        if (VAR == 2) {
                            if (la) bulk_g2s(dst, A + (size_t)b * M * K + (size_t)(r * 8 + ks) * 4096, ASTG, &full[s]);
                            bulk_g2s(dst + ASTG, B + (size_t)b * N * K + (size_t)((j * 2 + r) * 8 + ks) * 2048, BSTG,
                                     &full[s]);
                        } else {
                            if (la) ptx::tma_load_3d_nohint(dst, &tA, &full[s], r * 128, ks * 32, b);
                            if (VAR == 0)
                                ptx::tma_load_3d_nohint(dst + ASTG, &tB, &full[s], ks * 32, j * 128 + r * 64, b);
                            else   // whole columns: 8 columns per stage (8 KB)
                                ptx::tma_load_3d_nohint(dst + ASTG, &tB, &full[s], 0, j * 128 + r * 64 + ks * 8, b);
                        }
                        if (++s == S) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else {
        uint32_t s = 0, ph = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int b = u >> 1, r = u & 1;
            for (int j = 0; j < 2; ++j) {
                for (int ks = 0; ks < K / 32; ++ks) {
                    ptx::mbar_wait(&full[s], ph);
                    if (threadIdx.x == 32) ptx::mbar_arrive(&empty[s]);
                    if (++s == S) { s = 0; ph ^= 1; }
                }
                if (threadIdx.x == 32) {
                    ptx::bulk_wait_group_read0();
                    for (int c = 0; c < 4; ++c) ptx::tma_store_3d(&tC, cst + c * 32 * 128, r * 128, j * 128 + c * 32, b);
                    ptx::bulk_commit_group();
                }
                __syncwarp();
            }
        }
        if (threadIdx.x == 32) ptx::bulk_wait_group0();
    }
}

template <int VAR, int S>
void run(const char* name, float* A, float* B, float* C)
{
    CUtensorMap tA = map3(A, M, K, ITEMS, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    CUtensorMap tB = VAR == 1 ? map3(B, K, N, ITEMS, 256, 8, CU_TENSOR_MAP_SWIZZLE_NONE)
                              : map3(B, K, N, ITEMS, 32, 64, CU_TENSOR_MAP_SWIZZLE_128B);
    CUtensorMap tC = map3(C, M, N, ITEMS, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
    const int smem = S * STG + 128 * 128 * 4 + 2048;
    auto k = stream_kernel<VAR, S>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<148, 64, smem>>>(tA, tB, tC, A, B);
    const int reps = 20;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) k<<<148, 64, smem>>>(tA, tB, tC, A, B);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double bytes = 3.0 * ITEMS * M * N * 4;
    printf("{\"probe\": \"%s\", \"stages\": %d, \"err\": \"%s\", \"ms\": %.4f, \"GBs\": %.1f}\n", name, S,
           cudaGetErrorString(err), ms, bytes / ms / 1e6);
}

int main()
{
    float *A, *B, *C;
    const size_t n = (size_t)ITEMS * M * K;
    cudaMalloc(&A, n * 4);
    cudaMalloc(&B, n * 4);
    cudaMalloc(&C, n * 4);
    cudaMemset(A, 0, n * 4);
    cudaMemset(B, 0, n * 4);
    run<0, 5>("kernel_boxes", A, B, C);
    run<0, 6>("kernel_boxes", A, B, C);
    run<0, 3>("kernel_boxes", A, B, C);
    run<1, 5>("b_whole_columns", A, B, C);
    run<2, 5>("bulk_1d", A, B, C);
    run<2, 6>("bulk_1d", A, B, C);
    return 0;
}
