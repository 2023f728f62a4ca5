// gemm_sm100.cuh -- the emulated-SGEMM kernel for B200 (sm_100a).
//
// One persistent CTA per SM walks output tiles (batch, m-tile, n-tile) of
// BM x BN = 128 x BN.  Warp roles (18 warps, 576 threads):
//   warp 0       TMA producer: FP32 tiles of A (128 m x 32 k) and B (32 k x BN n)
//                HBM -> shared memory ring `f32` (S32 stages), mbarrier complete_tx.
//   warp 1       MMA issuer (one elected thread) + TMEM owner: per 16-k (FP16) or
//                8-k (TF32) step three tcgen05.mma, P1 = A_hi B_hi -> D_hi,
//                P2 = A_lo B_hi and P3 = A_hi B_lo -> D_corr (Eq. corr-5).
//   warps 2-9    splitters: FP32 stage -> hi/lo operand tiles (Eqs. corr-1..4,
//                P:479-488) written straight into the UMMA canonical layouts of
//                the operand ring `op` (SOP stages).  This is the B200 form of the
//                paper's split-on-load: the FP32 tile is read once
//                from shared memory and each part is written once, in the layout
//                the tensor core reads -- no separate FP16 staging copy and no
//                re-layout pass.  Two splitter warps per SM sub-partition.
//   warps 10-17  combine/epilogue: every k-block of KB elements, tcgen05.ld of
//                D_hi and D_corr, t = RN(D_hi + D_corr * 2^-11), C += t in FP32 RN
//                on CUDA cores (the outside-of-TC accumulation of P:495, R#7/R#8);
//                at the tile's end C = RN(alpha*C + RN(beta*C_old)), coalesced
//                column-major stores.
// TMEM: two accumulator buffers x (D_hi, D_corr) x BN columns = 512 columns, so
// the MMA warp fills one buffer while the combine warps drain the other.
//
// Shared-memory layouts (all buffers 1024-byte aligned):
//   f32 A  [32 k][128 m] fp32, plain (TMA box {128, 32}); 512-byte rows
//   f32 B  [BN n][32 k]  fp32, TMA SWIZZLE_128B (box {32, BN}); 128-byte rows
//   op A_hi/A_lo  FP16: MN-major SWIZZLE_128B [k/8][m/64][k%8][128 B], LBO 1024
//                 (next 64-m block), SBO 2048 (next 8-k group).
//                 TF32: K-major SWIZZLE_128B [m][32 k] (SBO 1024), or the 32-bit
//                 MN-major SWIZZLE_128B_BASE32B [k/4][m/32][k%4][128 B] (variant).
//   op B_hi/B_lo  K-major, one row of 32 k per n: FP16 64-byte rows SWIZZLE_64B
//                 (SBO 512), TF32 128-byte rows SWIZZLE_128B (SBO 1024).
// Swizzles are XORs on absolute shared addresses: 16-byte chunk bits [4,7)
// (SW128) or [4,6) (SW64) ^= bits [7,10) / [7,9); BASE32B: 32-byte bits [5,7)
// ^= bits [7,9) -- what both TMA and the UMMA descriptor apply.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "sm100_ptx.cuh"
#include "split.cuh"

namespace emu {

// Optional role timing (build with -DEMU_PROF; tools/ only, never the product
// library): lane 0 of each role warp accumulates clock64() cycles per event.
#ifdef EMU_PROF
enum ProfSlot { P_PROD_WAIT_EMPTY, P_MMA_WAIT_ACC, P_MMA_WAIT_OP, P_SPL_WAIT_F32, P_SPL_WAIT_OP, P_SPL_WORK,
                P_EPI_WAIT_ACC, P_EPI_DRAIN, P_EPI_STORE, P_CTA_TOTAL, P_MMA_ISSUE, P_NSLOTS };
__device__ unsigned long long g_prof[16];
#define PROF_DECL unsigned long long prof_acc[P_NSLOTS] = {}; long long prof_t0 = 0;
#define PROF_T0() (prof_t0 = clock64())
#define PROF_ADD(slot) (prof_acc[slot] += (unsigned long long)(clock64() - prof_t0))
#define PROF_FLUSH()                                                            \
    do {                                                                        \
        if ((threadIdx.x & 31) == 0)                                            \
            for (int i_ = 0; i_ < P_NSLOTS; ++i_)                               \
                if (prof_acc[i_]) atomicAdd(&g_prof[i_], prof_acc[i_]);         \
    } while (0)
// event trace of CTA 0 (the leader of cluster 0): per recording warp a region of
// TRACE_R entries (clock64, event << 32 | arg), written without atomics
constexpr int TRACE_ROLES = 20, TRACE_R = 1 << 12, TRACE_N = TRACE_ROLES * TRACE_R;
__device__ long long g_trace[TRACE_N][2];
__device__ unsigned int g_trace_cnt[TRACE_ROLES];
#ifdef EMU_TRACE
#define TRACE_DECL unsigned trace_i = 0;
#define TRACE_AT(role, ev, arg)                                                                \
    do {                                                                                      \
        if (blockIdx.x == 0 && trace_i < (unsigned)TRACE_R) {                                 \
            long long* e_ = g_trace[(role) * TRACE_R + trace_i++];                            \
            e_[0] = clock64();                                                                \
            e_[1] = ((long long)(ev) << 32) | (unsigned)(arg);                                \
        }                                                                                     \
    } while (0)
#define TRACE_END(role)                                                                       \
    do {                                                                                      \
        if (blockIdx.x == 0) g_trace_cnt[role] = trace_i;                                     \
    } while (0)
#else
#define TRACE_DECL
#define TRACE_AT(role, ev, arg) ((void)0)
#define TRACE_END(role) ((void)0)
#endif
#else
#define TRACE_DECL
#define TRACE_AT(role, ev, arg) ((void)0)
#define TRACE_END(role) ((void)0)
#define PROF_DECL
#define PROF_T0() ((void)0)
#define PROF_ADD(slot) ((void)0)
#define PROF_FLUSH() ((void)0)
#endif

struct GemmParams {
    int m, n, k;
    int a_batched, b_batched;     // 0: batch coordinate 0 for every problem (stride 0)
    float alpha, beta;
    float* C;
    long long ldc, strideC;
    int tiles_m, tiles_n;
    long long num_tiles;
    long long num_units;          // TS kernel: work units (A-stationary: one (batch, m-pair) row block each)
    int unit_tiles;               // TS kernel: tiles per unit (A-stationary: tiles_n, else 1)
    int clc;                      // TS kernel (long-k rings): dynamic tile order by cluster launch
                                  // control -- the grid has one cluster per unit
    int num_k_stages;             // ceil(k / 32)
    int kb_stages;                // KB / 32
    int corr;                     // 1 = the paper's method; 0 = "correction off" control
    int tma_store;                // 1: epilogue stages C in shared memory and TMA-stores it (beta == 0)
    int prefetch;                 // L2 prefetch distance in k-stages (0 = off)
    int group_m;                  // raster: m-tiles per group walking the n-tiles together
    int l2_policy;                // 0 default; bit 1: A evict_last; bit 0: B evict_last
                                  // (TS kernel: B evict_first)
    unsigned int* range_flag;     // nullable (FP16 mode only)
    // range-safe mode (TS kernel): max |x| bit patterns of the rows of A / columns of
    // B, [batch][m] and [batch][n]; nullptr = unscaled (the paper's method)
    const unsigned int* row_max;
    const unsigned int* col_max;
    // direct-load (LDG) variant only: operands read by the splitter warps
    const float* A;
    const float* B;
    long long lda, ldb, strideA, strideB;   // elements; stride 0 = shared operand
    // TS kernel, single problem (emu_sgemm_multicast): the result is also stored to
    // dst[1 .. num_dst-1] (same ldc; peers' buffers for a fused all-gather); 0/1 = C only
    int num_dst;
    float* dst[8];
};

// range-safe mode: exponent e = clamp(ilogb(max) - 14, -125, 125) of a row / column from
// the bit pattern of its max finite |x| (0 for none), and 2^t for |t| <= 125
__device__ __forceinline__ int range_exp_of(unsigned int maxbits)
{
    if (maxbits == 0u) return 0;
    const int be = (int)(maxbits >> 23);
    const int lg = be ? be - 127 : -118 - __clz(maxbits & 0x7fffffu);   // ilogb, subnormals too
    const int e = lg - 14;
    return e < -125 ? -125 : (e > 125 ? 125 : e);
}
__device__ __forceinline__ float pow2i(int t) { return __int_as_float((127 + t) << 23); }

// c * 2^t correctly rounded (one rounding, like ldexpf) for |t| <= 252: two
// power-of-two factors of which only the second can round -- for t > 127 the
// first (2^127) is exact unless it overflows (then so does the result); for
// t < -126 the first (2^(t+126)) is exact unless the result is below 2^-252,
// where both the two-step product and the exact result round to zero
__device__ __forceinline__ float ldexp_rn(float c, int t)
{
    const int t2 = t > 127 ? t - 127 : (t < -126 ? -126 : 0);
    return __fmul_rn(__fmul_rn(c, pow2i(t - t2)), pow2i(t2));
}

// A operand layouts in the operand ring
enum : int {
    A_MN_SW128 = 0,      // MN-major, SWIZZLE_128B (16-bit elements; FP16 mode)
    A_K_SW128 = 1,       // K-major, one row of 32 k per m (TF32: 128-byte rows, SWIZZLE_128B)
    A_MN_SW128_32B = 2,  // MN-major, SWIZZLE_128B_BASE32B (the MN-major layout for 32-bit elements)
};

template <int MODE, int BN, int ALAY = (MODE == 0 ? A_MN_SW128 : A_K_SW128)>
struct GemmCfg {
    static constexpr int BM = 128;
    static constexpr int BK = 32;                       // k per FP32 stage
    static constexpr int ESZ = MODE == 0 ? 2 : 4;       // operand bytes per element
    static constexpr int KSTEP = MODE == 0 ? 16 : 8;    // UMMA K per instruction
    static constexpr int NSTEPS = BK / KSTEP;           // MMAs per product per stage
    static constexpr uint32_t A32_BYTES = BK * BM * 4;
    static constexpr uint32_t B32_BYTES = BK * BN * 4;
    static constexpr uint32_t F32_STAGE = A32_BYTES + B32_BYTES;
    static constexpr uint32_t AOP_BYTES = BM * BK * ESZ;
    static constexpr uint32_t BOP_BYTES = BN * BK * ESZ;
    static constexpr uint32_t OP_STAGE = 2 * AOP_BYTES + 2 * BOP_BYTES;
    static constexpr int S32 = MODE == 0 ? 3 : 2;
    static constexpr int SOP = 2;
    // C staging tile for the TMA-store epilogue (FP16 mode; TF32's operand ring
    // leaves no room, it stores with STG)
    static constexpr uint32_t CSTAGE_BYTES = MODE == 0 ? BM * BN * 4 : 0;
    static constexpr uint32_t B_ROW = BK * ESZ;         // 64 (FP16) or 128 (TF32)
    static constexpr uint32_t B_SBO = 8 * B_ROW;
    static constexpr uint32_t B_LAYOUT = MODE == 0 ? 4 : 2;  // SW64 / SW128
    static_assert(ALAY != A_MN_SW128 || ESZ == 2, "MN-major SW128 here is the 16-bit layout");
    static_assert(ALAY != A_MN_SW128_32B || ESZ == 4, "BASE32B is the 32-bit MN-major layout");
    // A descriptor: leading / stride byte offsets, layout type, bytes per K step, major
    static constexpr uint32_t A_LBO = ALAY == A_MN_SW128 ? 1024 : ALAY == A_K_SW128 ? 16 : 512;
    static constexpr uint32_t A_SBO = ALAY == A_MN_SW128 ? (BM / 64) * 1024
                                    : ALAY == A_K_SW128 ? 8 * B_ROW : (BM / 32) * 512;
    static constexpr uint32_t A_LAYOUT = ALAY == A_MN_SW128 ? 2 : ALAY == A_K_SW128 ? B_LAYOUT : 1;
    static constexpr uint32_t A_STEP = ALAY == A_MN_SW128 ? (KSTEP / 8) * A_SBO
                                     : ALAY == A_K_SW128 ? 32 : (KSTEP / 4) * A_SBO;
    static constexpr uint32_t A_MAJOR = ALAY == A_K_SW128 ? 0 : 1;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t BAR_BYTES = 8 * (2 * S32 + 2 * SOP + 4) + 16;
    static constexpr uint32_t SMEM_BYTES = 1024 + S32 * F32_STAGE + SOP * OP_STAGE + CSTAGE_BYTES + BAR_BYTES;
    static constexpr int SPLIT_WARP0 = 2, NUM_SPLIT_WARPS = 8;
    static constexpr int EPI_WARP0 = 10, NUM_EPI_WARPS = 8;
    static constexpr int NUM_THREADS = 32 * (EPI_WARP0 + NUM_EPI_WARPS);
    static constexpr int SPLIT_THREADS = 32 * NUM_SPLIT_WARPS;
    static_assert(2 * 2 * BN <= 512, "two (D_hi, D_corr) buffers must fit TMEM");
    static_assert(SMEM_BYTES <= 232448, "shared memory");
    static_assert(BN == 128, "this kernel's splitter work division assumes BN = 128");
};

// tile index -> (batch, m-tile, n-tile); groups of up to group_m m-tiles walk the
// n-tiles together so that concurrently running CTAs share A and B in L2.
__device__ __forceinline__ void tile_coords(const GemmParams& p, long long t, int& b, int& mt, int& nt)
{
    const long long per_batch = (long long)p.tiles_m * p.tiles_n;
    b = (int)(t / per_batch);
    int r = (int)(t - (long long)b * per_batch);
    const int GM = p.tiles_m < p.group_m ? p.tiles_m : p.group_m;
    const int group = r / (GM * p.tiles_n);
    const int first_m = group * GM;
    const int gm = (p.tiles_m - first_m) < GM ? (p.tiles_m - first_m) : GM;
    const int rr = r - group * GM * p.tiles_n;
    mt = first_m + rr % gm;
    nt = rr / gm;
}

// ------------------------------------------------------------ split helpers
// Four FP32 values (consecutive along the 16-byte unit the layout stores) ->
// FP16 hi/lo pairs: packed so element 0 is the low half.
__device__ __forceinline__ void split4_fp16(const float4 v, uint2& h, uint2& l)
{
    split_fp16x2x2(v.x, v.y, v.z, v.w, h.x, h.y, l.x, l.y);
}

// LDG = false: TMA stages FP32 tiles in shared memory (the fast path; needs
// 16-byte aligned bases and leading dimensions / strides in 16-byte units).
// LDG = true: the splitter warps read FP32 operands straight from global memory
// with bounds checks (any alignment, any lda/ldb); the TMA warp idles.
template <int MODE, int BN, int ALAY, bool RANGE, bool LDG>
__global__ void __launch_bounds__(GemmCfg<MODE, BN, ALAY>::NUM_THREADS, 1)
emu_sgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const GemmParams p)
{
    using Cfg = GemmCfg<MODE, BN, ALAY>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // keep the pointer derived from the __shared__ array (so loads/stores stay
    // LDS/STS) while aligning to 1024 bytes for the swizzled layouts
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* f32buf = smem;
    uint8_t* opbuf = smem + Cfg::S32 * Cfg::F32_STAGE;
    float* cstage = reinterpret_cast<float*>(opbuf + Cfg::SOP * Cfg::OP_STAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(opbuf + Cfg::SOP * Cfg::OP_STAGE + Cfg::CSTAGE_BYTES);
    uint64_t* f32_full = bars;
    uint64_t* f32_empty = f32_full + Cfg::S32;
    uint64_t* op_full = f32_empty + Cfg::S32;
    uint64_t* op_empty = op_full + Cfg::SOP;
    uint64_t* acc_full = op_empty + Cfg::SOP;
    uint64_t* acc_empty = acc_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    PROF_DECL
#ifdef EMU_PROF
    const long long prof_start = clock64();
#endif

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < Cfg::S32; ++i) {
            ptx::mbar_init(&f32_full[i], 1);
            ptx::mbar_init(&f32_empty[i], Cfg::SPLIT_THREADS);
        }
        for (int i = 0; i < Cfg::SOP; ++i) {
            ptx::mbar_init(&op_full[i], Cfg::SPLIT_THREADS);
            ptx::mbar_init(&op_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&acc_full[i], 1);
            ptx::mbar_init(&acc_empty[i], Cfg::NUM_EPI_WARPS * 32);
        }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_wait_then_allow_next();   // prologue done: wait for the previous kernel on the stream

    const int nks = p.num_k_stages;
    const int nkb = (nks + p.kb_stages - 1) / p.kb_stages;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (!LDG && ptx::elect_one()) {
            // L2 prefetch cursor PF stages ahead of the loads: deepens the memory
            // pipeline beyond the S32 shared-memory stages (the loads then hit L2)
            const int PF = p.prefetch;
            long long pt = blockIdx.x;
            int pks = 0;
            auto prefetch_next = [&]() {
                if (pt >= p.num_tiles) return;
                int b, mt, nt;
                tile_coords(p, pt, b, mt, nt);
                ptx::tma_prefetch_3d(&tmA, mt * Cfg::BM, pks * Cfg::BK, p.a_batched ? b : 0);
                ptx::tma_prefetch_3d(&tmB, pks * Cfg::BK, nt * BN, p.b_batched ? b : 0);
                if (++pks == nks) { pks = 0; pt += gridDim.x; }
            };
            for (int i = 0; i < PF; ++i) prefetch_next();
            const bool do_pf = PF > 0;
            uint32_t s = 0, ph = 0;
            for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                int b, mt, nt;
                tile_coords(p, t, b, mt, nt);
                const int ab = p.a_batched ? b : 0, bb = p.b_batched ? b : 0;
                for (int ks = 0; ks < nks; ++ks) {
                    PROF_T0();
                    ptx::mbar_wait_sleep(&f32_empty[s], ph ^ 1);
                    PROF_ADD(P_PROD_WAIT_EMPTY);
                    uint8_t* dst = f32buf + s * Cfg::F32_STAGE;
                    ptx::mbar_arrive_expect_tx(&f32_full[s], Cfg::F32_STAGE);
                    ptx::tma_load_3d_nohint(dst, &tmA, &f32_full[s], mt * Cfg::BM, ks * Cfg::BK, ab);
                    ptx::tma_load_3d_nohint(dst + Cfg::A32_BYTES, &tmB, &f32_full[s], ks * Cfg::BK, nt * BN, bb);
                    if (do_pf) prefetch_next();
                    if (++s == Cfg::S32) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (ptx::elect_one()) {
            constexpr uint32_t idesc = ptx::instr_desc(MODE == 0 ? 0u : 2u, Cfg::A_MAJOR, 0u, Cfg::BM, BN);
            uint32_t s = 0, ph = 0, acc_it = 0;
            for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
                for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                    const uint32_t buf = acc_it & 1u, aph = (acc_it >> 1) & 1u;
                    PROF_T0();
                    ptx::mbar_wait(&acc_empty[buf], aph ^ 1);
                    PROF_ADD(P_MMA_WAIT_ACC);
                    ptx::tc_fence_after();
                    const uint32_t d_hi = tmem_base + buf * 2 * BN;
                    const uint32_t d_corr = d_hi + BN;
                    const int ks0 = kb * p.kb_stages;
                    const int ks1 = min(ks0 + p.kb_stages, nks);
                    for (int ks = ks0; ks < ks1; ++ks) {
                        PROF_T0();
                        ptx::mbar_wait(&op_full[s], ph);
                        PROF_ADD(P_MMA_WAIT_OP);
                        PROF_T0();
                        ptx::tc_fence_after();
                        const uint32_t base = ptx::smem_u32(opbuf + s * Cfg::OP_STAGE);
                        const uint32_t a_hi = base, a_lo = base + Cfg::AOP_BYTES;
                        const uint32_t b_hi = base + 2 * Cfg::AOP_BYTES;
                        const uint32_t b_lo = b_hi + Cfg::BOP_BYTES;
#pragma unroll
                        for (int st = 0; st < Cfg::NSTEPS; ++st) {
                            const uint32_t aoff = st * Cfg::A_STEP;
                            const uint32_t boff = st * 32;   // K-major: 32 bytes along the swizzled row
                            const uint64_t dA_hi = ptx::smem_desc(a_hi + aoff, Cfg::A_LBO, Cfg::A_SBO, Cfg::A_LAYOUT);
                            const uint64_t dA_lo = ptx::smem_desc(a_lo + aoff, Cfg::A_LBO, Cfg::A_SBO, Cfg::A_LAYOUT);
                            const uint64_t dB_hi = ptx::smem_desc(b_hi + boff, 16, Cfg::B_SBO, Cfg::B_LAYOUT);
                            const uint64_t dB_lo = ptx::smem_desc(b_lo + boff, 16, Cfg::B_SBO, Cfg::B_LAYOUT);
                            const uint32_t acc = (ks > ks0 || st > 0) ? 1u : 0u;
                            if (MODE == 0) {
                                ptx::mma_f16(d_hi, dA_hi, dB_hi, idesc, acc);            // P1
                                if (p.corr) {
                                    ptx::mma_f16(d_corr, dA_lo, dB_hi, idesc, acc);      // P2
                                    ptx::mma_f16(d_corr, dA_hi, dB_lo, idesc, 1u);       // P3
                                }
                            } else {
                                ptx::mma_tf32(d_hi, dA_hi, dB_hi, idesc, acc);
                                if (p.corr) {
                                    ptx::mma_tf32(d_corr, dA_lo, dB_hi, idesc, acc);
                                    ptx::mma_tf32(d_corr, dA_hi, dB_lo, idesc, 1u);
                                }
                            }
                        }
                        ptx::tc_commit(&op_empty[s]);   // operand stage free when these MMAs finish
                        PROF_ADD(P_MMA_ISSUE);
                        if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                    }
                    ptx::tc_commit(&acc_full[buf]);     // k-block accumulators ready
                }
            }
        }
    } else if (warp >= Cfg::SPLIT_WARP0 && warp < Cfg::SPLIT_WARP0 + Cfg::NUM_SPLIT_WARPS) {
        // ------------------------------------------------ splitters (256 threads)
        const uint32_t tid = threadIdx.x - Cfg::SPLIT_WARP0 * 32;   // 0..255
        const uint32_t sw = tid >> 5;                                 // 0..7
        const uint32_t row = tid & 127, half = tid >> 7;              // K-major rows: half of the 32 k each
        uint32_t s32 = 0, ph32 = 0, sop = 0, phop = 0;
        uint32_t nonfinite = 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            int tb = 0, tmt = 0, tnt = 0;
            if (LDG) tile_coords(p, t, tb, tmt, tnt);
            const float* gA = LDG ? p.A + (long long)tb * p.strideA : nullptr;
            const float* gB = LDG ? p.B + (long long)tb * p.strideB : nullptr;
            for (int ks = 0; ks < nks; ++ks) {
                PROF_T0();
                if (!LDG) ptx::mbar_wait(&f32_full[s32], ph32);
                PROF_ADD(P_SPL_WAIT_F32);
                PROF_T0();
                ptx::mbar_wait(&op_empty[sop], phop ^ 1);
                PROF_ADD(P_SPL_WAIT_OP);
                PROF_T0();
                const uint8_t* fa = f32buf + s32 * Cfg::F32_STAGE;
                const uint8_t* fb = fa + Cfg::A32_BYTES;
                const int m0 = tmt * Cfg::BM, n0 = tnt * BN, k0 = ks * Cfg::BK;
                // FP32 A(m0 + m, k0 + k) and B(k0 + k, n0 + n): shared-memory stage or global
                auto a1 = [&](uint32_t m, uint32_t k) -> float {
                    if (LDG) {
                        const int gm = m0 + (int)m, gk = k0 + (int)k;
                        return (gm < p.m && gk < p.k) ? __ldg(gA + gm + (long long)gk * p.lda) : 0.0f;
                    }
                    return reinterpret_cast<const float*>(fa)[k * Cfg::BM + m];
                };
                auto a4 = [&](uint32_t m, uint32_t k) -> float4 {   // A(m..m+3, k)
                    if (LDG) return make_float4(a1(m, k), a1(m + 1, k), a1(m + 2, k), a1(m + 3, k));
                    return *reinterpret_cast<const float4*>(fa + k * 512 + m * 4);
                };
                auto b4 = [&](uint32_t n, uint32_t c) -> float4 {   // B(4c..4c+3, n)
                    if (LDG) {
                        const int gn = n0 + (int)n, gk = k0 + 4 * (int)c;
                        const float* col = gB + (long long)gn * p.ldb + gk;
                        const bool okn = gn < p.n;
                        return make_float4(okn && gk < p.k ? __ldg(col) : 0.0f, okn && gk + 1 < p.k ? __ldg(col + 1) : 0.0f,
                                           okn && gk + 2 < p.k ? __ldg(col + 2) : 0.0f,
                                           okn && gk + 3 < p.k ? __ldg(col + 3) : 0.0f);
                    }
                    return *reinterpret_cast<const float4*>(fb + n * 128 + ((c ^ (n & 7)) << 4));
                };
                uint8_t* o = opbuf + sop * Cfg::OP_STAGE;
                uint8_t* oa_hi = o;
                uint8_t* oa_lo = o + Cfg::AOP_BYTES;
                uint8_t* ob_hi = o + 2 * Cfg::AOP_BYTES;
                uint8_t* ob_lo = ob_hi + Cfg::BOP_BYTES;
                // ---- load phase: every FP32 value this thread splits in this stage is
                // read before the first store (the stores cannot alias the loads, but
                // the compiler cannot prove it and would serialise load -> store)
                float4 va[4], vb[4];
                const uint32_t n = row;
                if (ALAY == A_K_SW128) {
                    // A K-major (TF32): thread = (m row, 16-k half); 4 k per 16-byte chunk
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const uint32_t k4 = 4 * (half * 4 + jj);
                        va[jj] = make_float4(a1(row, k4), a1(row, k4 + 1), a1(row, k4 + 2), a1(row, k4 + 3));
                    }
                } else {
                    // A MN-major: warp sw handles k rows sw, sw+8, ...; lane handles m = 4*lane .. +3
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) va[kk] = a4(lane * 4, sw + 8 * kk);
                }
                // B: thread = (n row, 16-k half): 4 chunks of 4 k
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) vb[jj] = b4(n, half * 4 + jj);

                // ---- split + store phase
                if (ALAY == A_K_SW128) {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const uint32_t j = half * 4 + jj;
                        uint4 hv, lv;
                        split_tf32(va[jj].x, hv.x, lv.x);
                        split_tf32(va[jj].y, hv.y, lv.y);
                        split_tf32(va[jj].z, hv.z, lv.z);
                        split_tf32(va[jj].w, hv.w, lv.w);
                        const uint32_t off = row * Cfg::B_ROW + ((j ^ (row & 7)) << 4);
                        *reinterpret_cast<uint4*>(oa_hi + off) = hv;
                        *reinterpret_cast<uint4*>(oa_lo + off) = lv;
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t k = sw + 8 * kk;
                        const float4 v = va[kk];
                        if (MODE == 0) {
                            const uint32_t g = k >> 3, kr = k & 7;
                            uint2 h, l;
                            split4_fp16(v, h, l);
                            if (RANGE) nonfinite |= f16x2_nonfinite(h.x) | f16x2_nonfinite(h.y);
                            const uint32_t mblk = lane >> 4, chunk = (lane & 15) >> 1;
                            const uint32_t off = g * Cfg::A_SBO + mblk * Cfg::A_LBO + kr * 128 +
                                                 ((chunk ^ kr) << 4) + (lane & 1) * 8;
                            *reinterpret_cast<uint2*>(oa_hi + off) = h;
                            *reinterpret_cast<uint2*>(oa_lo + off) = l;
                        } else {
                            // SWIZZLE_128B_BASE32B: 32 m x 4 k atoms of 512 B, 32-byte units
                            // (address bits [5,7)) XORed with the k row in the atom (bits [7,9))
                            const uint32_t g = k >> 2, kr = k & 3;
                            uint4 h, l;
                            split_tf32(v.x, h.x, l.x);
                            split_tf32(v.y, h.y, l.y);
                            split_tf32(v.z, h.z, l.z);
                            split_tf32(v.w, h.w, l.w);
                            const uint32_t mblk = lane >> 3;
                            const uint32_t inrow = (lane & 7) * 16;
                            const uint32_t off = g * Cfg::A_SBO + mblk * Cfg::A_LBO + kr * 128 + (inrow ^ (kr << 5));
                            *reinterpret_cast<uint4*>(oa_hi + off) = h;
                            *reinterpret_cast<uint4*>(oa_lo + off) = l;
                        }
                    }
                }
                if (MODE == 0) {
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {   // 8 k per 16-byte FP16 chunk
                        const uint32_t j = half * 2 + jj;
                        uint2 h0, l0, h1, l1;
                        split4_fp16(vb[2 * jj], h0, l0);
                        split4_fp16(vb[2 * jj + 1], h1, l1);
                        if (RANGE)
                            nonfinite |= f16x2_nonfinite(h0.x) | f16x2_nonfinite(h0.y) |
                                         f16x2_nonfinite(h1.x) | f16x2_nonfinite(h1.y);
                        const uint32_t off = n * 64 + ((j ^ ((n >> 1) & 3)) << 4);
                        *reinterpret_cast<uint4*>(ob_hi + off) = make_uint4(h0.x, h0.y, h1.x, h1.y);
                        *reinterpret_cast<uint4*>(ob_lo + off) = make_uint4(l0.x, l0.y, l1.x, l1.y);
                    }
                } else {
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {   // 4 k per 16-byte TF32 chunk
                        const uint32_t j = half * 4 + jj;
                        const float4 v = vb[jj];
                        uint4 h, l;
                        split_tf32(v.x, h.x, l.x);
                        split_tf32(v.y, h.y, l.y);
                        split_tf32(v.z, h.z, l.z);
                        split_tf32(v.w, h.w, l.w);
                        const uint32_t off = n * 128 + ((j ^ (n & 7)) << 4);
                        *reinterpret_cast<uint4*>(ob_hi + off) = h;
                        *reinterpret_cast<uint4*>(ob_lo + off) = l;
                    }
                }
                ptx::fence_proxy_async_smem();        // our st.shared -> visible to UMMA
                PROF_ADD(P_SPL_WORK);
                ptx::mbar_arrive(&op_full[sop]);
                if (!LDG) ptx::mbar_arrive(&f32_empty[s32]);
                if (++s32 == Cfg::S32) { s32 = 0; ph32 ^= 1; }
                if (++sop == Cfg::SOP) { sop = 0; phop ^= 1; }
            }
        }
        if (RANGE) {
            nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
            if (nonfinite && lane == 0) atomicOr(p.range_flag, 1u);
        }
    } else if (warp >= Cfg::EPI_WARP0) {
        // ------------------------------------------------ combine + epilogue
        constexpr int HALF = BN / 2;
        const uint32_t e = warp - Cfg::EPI_WARP0;
        const uint32_t q = warp & 3;            // TMEM lane quadrant this warp may access
        const uint32_t h = e >> 2;              // column half
        const float scale = MODE == 0 ? (1.0f / 2048.0f) : 1.0f;
        uint32_t acc_it = 0;
        for (long long t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
            int b, mt, nt;
            tile_coords(p, t, b, mt, nt);
            float creg[HALF];
#pragma unroll
            for (int j = 0; j < HALF; ++j) creg[j] = 0.0f;
            for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                const uint32_t buf = acc_it & 1u, aph = (acc_it >> 1) & 1u;
                PROF_T0();
                ptx::mbar_wait_sleep(&acc_full[buf], aph);
                PROF_ADD(P_EPI_WAIT_ACC);
                PROF_T0();
                ptx::tc_fence_after();
                const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * 2 * BN + h * HALF;
#pragma unroll
                for (int c = 0; c < HALF / 8; ++c) {
                    float vh[8], vc[8];
                    ptx::tmem_ld8(taddr + c * 8, vh);
                    ptx::tmem_ld8(taddr + BN + c * 8, vc);
                    ptx::tmem_wait_ld();
                    if (p.corr) {
#pragma unroll
                        for (int j = 0; j < 8; j += 2)
                            combine2(creg[c * 8 + j], creg[c * 8 + j + 1], vh[j], vh[j + 1], vc[j], vc[j + 1], scale);
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) creg[c * 8 + j] = __fadd_rn(creg[c * 8 + j], vh[j]);
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&acc_empty[buf]);
                PROF_ADD(P_EPI_DRAIN);
            }
            PROF_T0();
            // epilogue: C = RN(alpha*C + RN(beta*C_old)), column-major
            if (Cfg::CSTAGE_BYTES != 0 && p.tma_store) {
                // beta == 0: stage the tile in shared memory ([n][m], 512-byte
                // columns; a warp writes 32 consecutive m -> conflict-free) and let
                // one thread TMA-store it, so these warps go straight back to
                // draining the next tile while the stores stream out.
                const bool leader = (e == 0 && lane == 0);
                if (leader) ptx::bulk_wait_group_read0();       // previous tile's store has read the stage
                ptx::named_bar_sync(1, Cfg::NUM_EPI_WARPS * 32);
                const uint32_t r = q * 32 + lane;
#pragma unroll
                for (int j = 0; j < HALF; ++j)
                    cstage[(h * HALF + j) * Cfg::BM + r] = fmaf(p.alpha, creg[j], 0.0f);
                ptx::fence_proxy_async_smem();
                ptx::named_bar_sync(1, Cfg::NUM_EPI_WARPS * 32);
                if (leader) {
#pragma unroll
                    for (int c = 0; c < BN / 32; ++c)
                        ptx::tma_store_3d(&tmC, cstage + c * 32 * Cfg::BM, mt * Cfg::BM, nt * BN + c * 32, b);
                    ptx::bulk_commit_group();
                }
            } else {
                const int r = mt * Cfg::BM + (int)(q * 32 + lane);
                const int col0 = nt * BN + (int)(h * HALF);
                if (r < p.m) {
                    float* cp = p.C + (long long)b * p.strideC + r + (long long)col0 * p.ldc;
                    if (p.beta != 0.0f) {
#pragma unroll
                        for (int j = 0; j < HALF; ++j)
                            if (col0 + j < p.n) {
                                float* dst = cp + (long long)j * p.ldc;
                                *dst = fmaf(p.alpha, creg[j], __fmul_rn(p.beta, *dst));
                            }
                    } else {
#pragma unroll
                        for (int j = 0; j < HALF; ++j)
                            if (col0 + j < p.n) cp[(long long)j * p.ldc] = fmaf(p.alpha, creg[j], 0.0f);
                    }
                }
            }
            PROF_ADD(P_EPI_STORE);
        }
        if (Cfg::CSTAGE_BYTES != 0 && p.tma_store && warp == Cfg::EPI_WARP0 && lane == 0)
            ptx::bulk_wait_group0();   // global writes complete before the CTA retires
    }
#ifdef EMU_PROF
    if (warp >= 2 || lane == 0) {   // role warps (and the elected lanes of warps 0, 1)
        prof_acc[P_CTA_TOTAL] = (warp == 2 && lane == 0) ? (unsigned long long)(clock64() - prof_start) : 0;
        PROF_FLUSH();
    }
#endif

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
    }
}

}  // namespace emu
