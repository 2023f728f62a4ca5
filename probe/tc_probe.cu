// tc_probe.cu -- standalone tcgen05 accumulator probe (HARDWARE MEASUREMENT,
// test infrastructure).
//
// What it measures: the FP32 accumulation of ONE tcgen05.mma instruction (and
// of short chains of them accumulating in tensor memory) on chosen operand
// vectors.  The paper says only that the Tensor Core's own accumulation is
// "RZ" (§4.4 WMMAe-TCEC); SPEC.md S:213 gives the probe
// vector (1 + 3*2^-24 -> RZ 1 + 2^-23, RN 1 + 2^-22).  The samples this probe
// produces are the ONLY data tools/tc_fit.py fits the oracle's "sm100"
// tensor-core model to (R#9).
//
// Independence: this file shares no code, header or helper with the product
// library (paper_2308_15152_b200/csrc, libemusgemm.so) nor with oracle/.  Every
// PTX wrapper, descriptor encoder and layout rule below is written out here
// from the PTX ISA.  The operands arrive as raw binary16 / TF32 bit patterns
// (no conversion or split happens on the GPU side).
//
// Layout:
//   * one CTA (cta_group::1, M = 128) or one CTA pair (cta_group::2, M = 256,
//     each CTA holding 128 rows of A and N/2 rows of B) per "problem";
//     `grid` independent problems per launch;
//   * A (and B) in shared memory, K-major, SWIZZLE_128B: rows of 128 bytes
//     (4 instructions' K), 8-row atoms of 1024 bytes, 16-byte chunk c of row r
//     stored at chunk c ^ (r & 7); instruction i uses the 32-byte K slice
//     (i & 3) of K-tile (i >> 2), descriptor start address + 32*(i & 3);
//   * A from tensor memory (a_tmem = 1): lane = row, 32-bit columns along K
//     (two binary16 or one TF32 per column), 8 columns per instruction;
//   * D (FP32) in tensor memory columns [0, N), initialised from D0 by
//     tcgen05.st when given, then n_instr MMAs (accumulate from the first one
//     when D0 is given), one commit, tcgen05.ld back.
//
// C ABI (device pointers, caller-owned; stream is a cudaStream_t):
//   int tcp_run(int kind, int pair, int a_tmem, int n_instr, int N, int grid,
//               const void* A, const void* B, const float* D0, float* D,
//               void* stream)
//     kind    0 = kind::f16 (binary16 operands, K_inst = 16),
//             1 = kind::tf32 (TF32 operands as 32-bit patterns, K_inst = 8)
//     pair    0 = cta_group::1 (M = 128), 1 = cta_group::2 (M = 256)
//     n_instr 1..8 chained instructions (K = n_instr * K_inst per output)
//     N       16..128, multiple of 16 (pair: of 32); D in TMEM columns [0, N),
//             A (TS form) in columns [128, 192)
//     A       [grid][n_instr][M][K_inst] elements (2 or 4 bytes)
//     B       [grid][n_instr][N][K_inst] elements
//     D0      [grid][M][N] float, or NULL (accumulator starts at zero)
//     D       [grid][M][N] float (out)
//   returns 0, or a cudaError_t value / -1 for invalid arguments.
#include <cstdint>
#include <cuda_runtime.h>

namespace tcp {

__device__ __forceinline__ uint32_t saddr(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t ctarank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_barrier()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bar_wait0(uint64_t* b)
{
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "W:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 q, [%0], 0;\n\t"
        "@!q bra W;\n\t}"
        ::"r"(saddr(b)) : "memory");
}

// 128-byte swizzle inside a 1024-byte aligned atom: XOR address bits [4,7) with [7,10)
__device__ __forceinline__ uint32_t sw128(uint32_t off) { return off ^ (((off >> 7) & 7u) << 4); }

// shared-memory matrix descriptor, PTX ISA "tcgen05 shared memory descriptor":
// start >> 4 in [0,14), leading byte offset >> 4 in [16,30), stride byte offset
// >> 4 in [32,46), fixed 0b001 in [46,49), base offset 0 in [49,52), layout in
// [61,64) (2 = SWIZZLE_128B).  K-major swizzled: LBO unused (1), SBO = 1024.
__device__ __forceinline__ uint64_t desc_sw128_kmajor(uint32_t start)
{
    return (uint64_t)((start >> 4) & 0x3fff) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// instruction descriptor for kind::f16 / kind::tf32, FP32 D, both K-major:
// D format [4,6) = 1 (F32); A format [7,10), B format [10,13): 0 = F16 (kind::f16),
// 2 = TF32 (kind::tf32); N >> 3 in [17,23); M >> 4 in [24,29)
__device__ __forceinline__ uint32_t idesc(int kind, uint32_t M, uint32_t N)
{
    const uint32_t f = kind == 0 ? 0u : 2u;
    return (1u << 4) | (f << 7) | (f << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

template <int KIND, int PAIR, int ATMEM>
__device__ __forceinline__ void mma(uint32_t d, uint64_t adesc, uint32_t atm, uint64_t bdesc, uint32_t id,
                                    uint32_t acc)
{
    if (KIND == 0 && PAIR == 0 && ATMEM == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 1 && PAIR == 0 && ATMEM == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 0 && PAIR == 1 && ATMEM == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 1 && PAIR == 1 && ATMEM == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 0 && PAIR == 0 && ATMEM == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(atm), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 1 && PAIR == 0 && ATMEM == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(atm), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 0 && PAIR == 1 && ATMEM == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(atm), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    if (KIND == 1 && PAIR == 1 && ATMEM == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(atm), "l"(bdesc), "r"(id), "r"(acc) : "memory");
}

__device__ __forceinline__ void tst8(uint32_t ta, const uint32_t (&v)[8])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                   "r"(v[7]) : "memory");
}

__device__ __forceinline__ void tld8(uint32_t ta, uint32_t (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr int kMaxInstr = 8;
constexpr int kTileA = 128 * 128;   // bytes of one A K-tile (128 rows x 128 B)
constexpr int kTileB = 128 * 128;   // up to 128 B rows per CTA
constexpr int kSmem = 1024 + 2 * kTileA + 2 * kTileB;   // 2 K-tiles (8 instructions) of each

template <int KIND, int PAIR, int ATMEM>
__global__ void __launch_bounds__(128, 1)
probe_kernel(int n_instr, int N, const uint8_t* __restrict__ A, const uint8_t* __restrict__ B,
             const float* __restrict__ D0, float* __restrict__ D)
{
    extern __shared__ uint8_t raw[];
    __shared__ uint64_t done;
    __shared__ uint32_t tbase_slot;
    uint8_t* sm = raw + ((1024u - (saddr(raw) & 1023u)) & 1023u);
    uint8_t* sA = sm;
    uint8_t* sB = sm + 2 * kTileA;

    const uint32_t rank = PAIR ? ctarank() : 0u;
    const int prob = PAIR ? (blockIdx.x >> 1) : blockIdx.x;
    const int M = PAIR ? 256 : 128;
    const int Nloc = PAIR ? N / 2 : N;
    const int rowbytes = 32;              // one instruction's K slice: 16 x 2 B or 8 x 4 B
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // ---- operands: global -> shared (swizzled K-major), 16-byte chunks
    const uint8_t* Ag = A + ((size_t)prob * n_instr * M + (size_t)rank * 128) * rowbytes;
    const uint8_t* Bg = B + ((size_t)prob * n_instr * N + (size_t)rank * Nloc) * rowbytes;
    for (int t = tid; t < n_instr * 128 * 2; t += 128) {
        const int i = t / 256, r = (t >> 1) & 127, c = t & 1;
        const uint4 v = *reinterpret_cast<const uint4*>(Ag + ((size_t)i * M + r) * rowbytes + c * 16);
        const uint32_t off = sw128((uint32_t)r * 128u + (uint32_t)(i & 3) * 32u + (uint32_t)c * 16u);
        *reinterpret_cast<uint4*>(sA + (i >> 2) * kTileA + off) = v;
    }
    for (int t = tid; t < n_instr * Nloc * 2; t += 128) {
        const int i = t / (Nloc * 2), r = (t >> 1) % Nloc, c = t & 1;
        const uint4 v = *reinterpret_cast<const uint4*>(Bg + ((size_t)i * N + r) * rowbytes + c * 16);
        const uint32_t off = sw128((uint32_t)r * 128u + (uint32_t)(i & 3) * 32u + (uint32_t)c * 16u);
        *reinterpret_cast<uint4*>(sB + (i >> 2) * kTileB + off) = v;
    }

    if (tid == 0) bar_init(&done, 1);
    if (warp == 0) {
        if (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;"
                         ::"r"(saddr(&tbase_slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;"
                         ::"r"(saddr(&tbase_slot)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tbase_slot;
    const uint32_t lane_addr = (warp * 32u) << 16;   // this warp's TMEM lane quadrant
    const int row = warp * 32 + lane;                 // row of this CTA's 128

    // ---- A into tensor memory (TS form): columns [128 + 8 i, +8) for instruction i
    if (ATMEM) {
        for (int i = 0; i < n_instr; ++i) {
            const uint32_t* src = reinterpret_cast<const uint32_t*>(Ag + ((size_t)i * M + row) * rowbytes);
            uint32_t v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = src[c];
            tst8(tb + lane_addr + 128u + 8u * i, v);
        }
    }
    // ---- accumulator initial value
    const bool has_d0 = D0 != nullptr;
    if (has_d0) {
        const float* d0 = D0 + ((size_t)prob * M + rank * 128 + row) * N;
        for (int c0 = 0; c0 < N; c0 += 8) {
            uint32_t v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) v[c] = __float_as_uint(d0[c0 + c]);
            tst8(tb + lane_addr + c0, v);
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) cluster_barrier(); else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- the MMAs: one thread of the (leader) CTA
    if (tid == 0 && rank == 0) {
        const uint32_t id = idesc(KIND, (uint32_t)M, (uint32_t)N);
        for (int i = 0; i < n_instr; ++i) {
            const uint64_t ad = desc_sw128_kmajor(saddr(sA + (i >> 2) * kTileA) + 32u * (i & 3));
            const uint64_t bd = desc_sw128_kmajor(saddr(sB + (i >> 2) * kTileB) + 32u * (i & 3));
            mma<KIND, PAIR, ATMEM>(tb, ad, tb + 128u + 8u * i, bd, id, (i > 0 || has_d0) ? 1u : 0u);
        }
        if (PAIR)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(saddr(&done)), "h"((uint16_t)3) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(saddr(&done)) : "memory");
    }
    bar_wait0(&done);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- read D back: this thread's lane = row, columns [0, N)
    float* dout = D + ((size_t)prob * M + rank * 128 + row) * N;
    for (int c0 = 0; c0 < N; c0 += 8) {
        uint32_t v[8];
        tld8(tb + lane_addr + c0, v);
#pragma unroll
        for (int c = 0; c < 8; ++c) dout[c0 + c] = __uint_as_float(v[c]);
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (PAIR) cluster_barrier(); else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) {
        if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tb) : "memory");
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tb) : "memory");
    }
}

template <int KIND, int PAIR, int ATMEM>
static int launch(int n_instr, int N, int grid, const void* A, const void* B, const float* D0, float* D,
                  cudaStream_t st)
{
    auto k = probe_kernel<KIND, PAIR, ATMEM>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid * (PAIR ? 2 : 1));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = PAIR ? 2 : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k, n_instr, N, static_cast<const uint8_t*>(A), static_cast<const uint8_t*>(B),
                           D0, D);
    return (int)e;
}

}  // namespace tcp

extern "C" __attribute__((visibility("default")))
int tcp_run(int kind, int pair, int a_tmem, int n_instr, int N, int grid, const void* A, const void* B,
            const float* D0, float* D, void* stream)
{
    using namespace tcp;
    if (kind < 0 || kind > 1 || pair < 0 || pair > 1 || a_tmem < 0 || a_tmem > 1) return -1;
    if (n_instr < 1 || n_instr > kMaxInstr || grid < 1 || !A || !B || !D) return -1;
    if (N < 16 || N > 128 || N % 16 != 0 || (pair && N % 32 != 0)) return -1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
#define TCP_CASE(K, P, T) \
    if (kind == K && pair == P && a_tmem == T) return launch<K, P, T>(n_instr, N, grid, A, B, D0, D, st);
    TCP_CASE(0, 0, 0) TCP_CASE(1, 0, 0) TCP_CASE(0, 1, 0) TCP_CASE(1, 1, 0)
    TCP_CASE(0, 0, 1) TCP_CASE(1, 0, 1) TCP_CASE(0, 1, 1) TCP_CASE(1, 1, 1)
#undef TCP_CASE
    return -1;
}
