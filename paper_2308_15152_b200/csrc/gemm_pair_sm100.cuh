// gemm_pair_sm100.cuh -- the CTA-pair (cta_group::2) emulated-SGEMM kernel.
//
// A cluster of two CTAs on the two SMs of a TPC computes a 256 (m) x 128 (n)
// output tile with tcgen05.mma.cta_group::2 (M = 256, N = 128):
//   * CTA r holds A rows [256 mt + 128 r, +128) and B columns [128 nt + 64 r, +64);
//     the MMA reads A from both CTAs (128 rows each) and B from both (64 columns
//     each), and writes D rows [128 r, +128) into CTA r's tensor memory.
//   * So each SM splits 128 x 32 + 64 x 32 FP32 elements per 32-k stage instead
//     of 128 x 32 + 128 x 32 for the same tensor work as the single-CTA kernel:
//     the B operand (split, staged and read by the tensor core) is halved --
//     the paper's "reduce the shared-memory footprint per MMA" on
//     B200.
// Roles per CTA (18 warps) as in gemm_sm100.cuh; the MMA issuer exists only in
// the even CTA (cluster rank 0).  Cross-CTA synchronisation:
//   op_full[s]  (leader): 16 arrivals, one per splitter warp of either CTA
//               (release.cluster remote arrives); the leader's MMA thread waits.
//   op_empty[s] (both):   tcgen05.commit multicast from the leader.
//   acc_full[b] (both):   tcgen05.commit multicast at the end of each k-block.
//   acc_empty[b](leader): 16 arrivals, one per combine warp of either CTA.
//   f32 ring:             local (each CTA's own TMA producer and splitters).
#pragma once

#include <cstdint>
#include <cuda.h>

#include "gemm_sm100.cuh"
#include "sm100_ptx.cuh"
#include "split.cuh"

namespace emu {

template <int MODE, int ALAY = (MODE == 0 ? A_MN_SW128 : A_K_SW128)>
struct PairCfg {
    static constexpr int BM = 128;                      // A rows per CTA (pair M = 256)
    static constexpr int BN = 128;                      // pair tile N (D columns per CTA)
    static constexpr int BNC = 64;                      // B columns staged per CTA
    static constexpr int BK = 32;
    static constexpr int ESZ = MODE == 0 ? 2 : 4;
    static constexpr int KSTEP = MODE == 0 ? 16 : 8;
    static constexpr int NSTEPS = BK / KSTEP;
    static constexpr uint32_t A32_BYTES = BK * BM * 4;     // 16 KB
    static constexpr uint32_t B32_BYTES = BK * BNC * 4;    //  8 KB
    static constexpr uint32_t F32_STAGE = A32_BYTES + B32_BYTES;
    static constexpr uint32_t AOP_BYTES = BM * BK * ESZ;
    static constexpr uint32_t BOP_BYTES = BNC * BK * ESZ;
    static constexpr uint32_t OP_STAGE = 2 * AOP_BYTES + 2 * BOP_BYTES;
    static constexpr int S32 = MODE == 0 ? 4 : 3;
    static constexpr int SOP = 2;
    // TMA-store staging: the whole C tile (FP16 mode, 64 KB) or half of it (TF32,
    // 32 KB; the two column halves are staged and stored one after the other)
    static constexpr int CSTAGE_PARTS = MODE == 0 ? 1 : 2;
    static constexpr uint32_t CSTAGE_BYTES = BM * (BN / CSTAGE_PARTS) * 4;
    static constexpr uint32_t B_ROW = BK * ESZ;
    static constexpr uint32_t B_SBO = 8 * B_ROW;
    static constexpr uint32_t B_LAYOUT = MODE == 0 ? 4 : 2;
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
    // warpgroup 0: TMA producer (warp 0), MMA issuer + TMEM owner (warp 1), 2 idle;
    // warpgroups 1-4: 16 splitter warps; warpgroups 5-6: 8 combine/epilogue warps.
    // Registers are re-balanced per warpgroup with setmaxnreg (launch: 72/thread).
    static constexpr int SPLIT_WARP0 = 4, NUM_SPLIT_WARPS = 16;
    static constexpr int EPI_WARP0 = 20, NUM_EPI_WARPS = 8;
    static constexpr int NUM_THREADS = 32 * (EPI_WARP0 + NUM_EPI_WARPS);
    static constexpr uint32_t REGS_CTRL = 40, REGS_SPLIT = 56, REGS_EPI = 120;
    static_assert(128 * REGS_CTRL + 32 * NUM_SPLIT_WARPS * REGS_SPLIT + 32 * NUM_EPI_WARPS * REGS_EPI <= 65536,
                  "register budget");
    static_assert(SMEM_BYTES <= 232448, "shared memory");
    static_assert(ALAY != A_MN_SW128 || ESZ == 2, "MN-major SW128 here is the 16-bit layout");
};

// pair-tile index -> (batch, m-tile of 256, n-tile of 128), grouped raster as in tile_coords
__device__ __forceinline__ void pair_tile_coords(const GemmParams& p, long long t, int& b, int& mt, int& nt)
{
    tile_coords(p, t, b, mt, nt);
}

template <int MODE, int ALAY, bool RANGE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<MODE, ALAY>::NUM_THREADS, 1)
emu_sgemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const GemmParams p)
{
    using Cfg = PairCfg<MODE, ALAY>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
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
    const uint32_t rank = ptx::cluster_ctarank();
    const long long cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    PROF_DECL
#ifdef EMU_PROF
    const long long prof_start = clock64();
#endif

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < Cfg::S32; ++i) {
            ptx::mbar_init(&f32_full[i], 1);
            ptx::mbar_init(&f32_empty[i], Cfg::NUM_SPLIT_WARPS);
        }
        for (int i = 0; i < Cfg::SOP; ++i) {
            ptx::mbar_init(&op_full[i], 2 * Cfg::NUM_SPLIT_WARPS);
            ptx::mbar_init(&op_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&acc_full[i], 1);
            ptx::mbar_init(&acc_empty[i], 2 * Cfg::NUM_EPI_WARPS);
        }
        ptx::fence_mbar_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();   // barriers initialised and TMEM allocated in both CTAs
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_wait_then_allow_next();   // prologue done: wait for the previous kernel on the stream

    const int nks = p.num_k_stages;
    const int nkb = (nks + p.kb_stages - 1) / p.kb_stages;

    if (warp < 4) {
      ptx::setmaxnreg_dec<Cfg::REGS_CTRL>();
      if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (ptx::elect_one()) {
            const int PF = p.prefetch;
            long long pt = cid;
            int pks = 0;
            auto prefetch_next = [&]() {
                if (pt >= p.num_tiles) return;
                int b, mt, nt;
                pair_tile_coords(p, pt, b, mt, nt);
                ptx::tma_prefetch_3d(&tmA, mt * 256 + rank * Cfg::BM, pks * Cfg::BK, p.a_batched ? b : 0);
                ptx::tma_prefetch_3d(&tmB, pks * Cfg::BK, nt * Cfg::BN + rank * Cfg::BNC, p.b_batched ? b : 0);
                if (++pks == nks) { pks = 0; pt += ncl; }
            };
            for (int i = 0; i < PF; ++i) prefetch_next();
            const bool do_pf = PF > 0;
            const uint64_t pol_keep = ptx::l2_policy_evict_last();
            uint32_t s = 0, ph = 0;
            for (long long t = cid; t < p.num_tiles; t += ncl) {
                int b, mt, nt;
                pair_tile_coords(p, t, b, mt, nt);
                const int ab = p.a_batched ? b : 0, bb = p.b_batched ? b : 0;
                for (int ks = 0; ks < nks; ++ks) {
                    PROF_T0();
                    ptx::mbar_wait_sleep(&f32_empty[s], ph ^ 1);
                    PROF_ADD(P_PROD_WAIT_EMPTY);
                    uint8_t* dst = f32buf + s * Cfg::F32_STAGE;
                    ptx::mbar_arrive_expect_tx(&f32_full[s], Cfg::F32_STAGE);
                    if (p.l2_policy & 2)
                        ptx::tma_load_3d(dst, &tmA, &f32_full[s], mt * 256 + rank * Cfg::BM, ks * Cfg::BK, ab, pol_keep);
                    else
                        ptx::tma_load_3d_nohint(dst, &tmA, &f32_full[s], mt * 256 + rank * Cfg::BM, ks * Cfg::BK, ab);
                    if (p.l2_policy & 1)
                        ptx::tma_load_3d(dst + Cfg::A32_BYTES, &tmB, &f32_full[s], ks * Cfg::BK,
                                         nt * Cfg::BN + rank * Cfg::BNC, bb, pol_keep);
                    else
                        ptx::tma_load_3d_nohint(dst + Cfg::A32_BYTES, &tmB, &f32_full[s], ks * Cfg::BK,
                                                nt * Cfg::BN + rank * Cfg::BNC, bb);
                    if (do_pf) prefetch_next();
                    if (++s == Cfg::S32) { s = 0; ph ^= 1; }
                }
            }
        }
      } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA only)
        if (rank == 0 && ptx::elect_one()) {
            constexpr uint32_t idesc = ptx::instr_desc(MODE == 0 ? 0u : 2u, Cfg::A_MAJOR, 0u, 256, Cfg::BN);
            uint32_t s = 0, ph = 0, acc_it = 0;
            for (long long t = cid; t < p.num_tiles; t += ncl) {
                for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                    const uint32_t buf = acc_it & 1u, aph = (acc_it >> 1) & 1u;
                    PROF_T0();
                    ptx::mbar_wait(&acc_empty[buf], aph ^ 1);
                    PROF_ADD(P_MMA_WAIT_ACC);
                    ptx::tc_fence_after();
                    const uint32_t d_hi = tmem_base + buf * 2 * Cfg::BN;
                    const uint32_t d_corr = d_hi + Cfg::BN;
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
                            const uint32_t boff = st * 32;
                            const uint64_t dA_hi = ptx::smem_desc(a_hi + aoff, Cfg::A_LBO, Cfg::A_SBO, Cfg::A_LAYOUT);
                            const uint64_t dA_lo = ptx::smem_desc(a_lo + aoff, Cfg::A_LBO, Cfg::A_SBO, Cfg::A_LAYOUT);
                            const uint64_t dB_hi = ptx::smem_desc(b_hi + boff, 16, Cfg::B_SBO, Cfg::B_LAYOUT);
                            const uint64_t dB_lo = ptx::smem_desc(b_lo + boff, 16, Cfg::B_SBO, Cfg::B_LAYOUT);
                            const uint32_t acc = (ks > ks0 || st > 0) ? 1u : 0u;
                            if (MODE == 0) {
                                ptx::mma_f16_pair(d_hi, dA_hi, dB_hi, idesc, acc);            // P1
                                if (p.corr) {
                                    ptx::mma_f16_pair(d_corr, dA_lo, dB_hi, idesc, acc);      // P2
                                    ptx::mma_f16_pair(d_corr, dA_hi, dB_lo, idesc, 1u);       // P3
                                }
                            } else {
                                ptx::mma_tf32_pair(d_hi, dA_hi, dB_hi, idesc, acc);
                                if (p.corr) {
                                    ptx::mma_tf32_pair(d_corr, dA_lo, dB_hi, idesc, acc);
                                    ptx::mma_tf32_pair(d_corr, dA_hi, dB_lo, idesc, 1u);
                                }
                            }
                        }
                        ptx::tc_commit_pair(&op_empty[s], 0x3);   // both CTAs' operand stage free
                        PROF_ADD(P_MMA_ISSUE);
                        if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                    }
                    ptx::tc_commit_pair(&acc_full[buf], 0x3);     // both CTAs' accumulators ready
                }
            }
        }
      }
    } else if (warp >= Cfg::SPLIT_WARP0 && warp < Cfg::SPLIT_WARP0 + Cfg::NUM_SPLIT_WARPS) {
        // ------------------------------------------------ splitters (512 threads)
        ptx::setmaxnreg_dec<Cfg::REGS_SPLIT>();
        const uint32_t tid = threadIdx.x - Cfg::SPLIT_WARP0 * 32;   // 0..511
        const uint32_t sw = tid >> 5;                                 // 0..15
        const uint32_t row = tid & 127, quarter = tid >> 7;          // A K-major (TF32): 8 k per thread
        const uint32_t n = tid & 63, eighth = tid >> 6;              // B: 4 k per thread
        uint32_t s32 = 0, ph32 = 0, sop = 0, phop = 0;
        uint32_t nonfinite = 0;
        for (long long t = cid; t < p.num_tiles; t += ncl) {
            for (int ks = 0; ks < nks; ++ks) {
                PROF_T0();
                ptx::mbar_wait(&f32_full[s32], ph32);
                PROF_ADD(P_SPL_WAIT_F32);
                PROF_T0();
                ptx::mbar_wait(&op_empty[sop], phop ^ 1);
                PROF_ADD(P_SPL_WAIT_OP);
                PROF_T0();
                const uint8_t* fa = f32buf + s32 * Cfg::F32_STAGE;
                const uint8_t* fb = fa + Cfg::A32_BYTES;
                uint8_t* o = opbuf + sop * Cfg::OP_STAGE;
                uint8_t* oa_hi = o;
                uint8_t* oa_lo = o + Cfg::AOP_BYTES;
                uint8_t* ob_hi = o + 2 * Cfg::AOP_BYTES;
                uint8_t* ob_lo = ob_hi + Cfg::BOP_BYTES;
                // ---- load phase (all loads of the stage before the first store)
                float4 va[2], vb;
                if (ALAY == A_K_SW128) {
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const float* col = reinterpret_cast<const float*>(fa) + 4 * (quarter * 2 + jj) * Cfg::BM + row;
                        va[jj] = make_float4(col[0], col[Cfg::BM], col[2 * Cfg::BM], col[3 * Cfg::BM]);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk)
                        va[kk] = *reinterpret_cast<const float4*>(fa + (sw + 16 * kk) * 512 + lane * 16);
                }
                // B(k = 4 eighth .. +3, n): FP32 16-byte chunk `eighth` of row n
                vb = *reinterpret_cast<const float4*>(fb + n * 128 + ((eighth ^ (n & 7)) << 4));
                // ---- split + store phase
                if (ALAY == A_K_SW128) {
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const uint32_t j = quarter * 2 + jj;
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
                    for (int kk = 0; kk < 2; ++kk) {
                        const uint32_t k = sw + 16 * kk;
                        const uint32_t g = k >> 3, kr = k & 7;
                        uint2 h, l;
                        split4_fp16(va[kk], h, l);
                        if (RANGE) nonfinite |= f16x2_nonfinite(h.x) | f16x2_nonfinite(h.y);
                        const uint32_t mblk = lane >> 4, chunk = (lane & 15) >> 1;
                        const uint32_t off = g * Cfg::A_SBO + mblk * Cfg::A_LBO + kr * 128 + ((chunk ^ kr) << 4) +
                                             (lane & 1) * 8;
                        *reinterpret_cast<uint2*>(oa_hi + off) = h;
                        *reinterpret_cast<uint2*>(oa_lo + off) = l;
                    }
                }
                if (MODE == 0) {
                    // half of a 16-byte FP16 chunk (4 k), K-major SWIZZLE_64B rows
                    uint2 h, l;
                    split4_fp16(vb, h, l);
                    if (RANGE) nonfinite |= f16x2_nonfinite(h.x) | f16x2_nonfinite(h.y);
                    const uint32_t j = eighth >> 1;
                    const uint32_t off = n * 64 + ((j ^ ((n >> 1) & 3)) << 4) + (eighth & 1) * 8;
                    *reinterpret_cast<uint2*>(ob_hi + off) = h;
                    *reinterpret_cast<uint2*>(ob_lo + off) = l;
                } else {
                    // one 16-byte TF32 chunk (4 k), K-major SWIZZLE_128B rows
                    uint4 h, l;
                    split_tf32(vb.x, h.x, l.x);
                    split_tf32(vb.y, h.y, l.y);
                    split_tf32(vb.z, h.z, l.z);
                    split_tf32(vb.w, h.w, l.w);
                    const uint32_t off = n * 128 + ((eighth ^ (n & 7)) << 4);
                    *reinterpret_cast<uint4*>(ob_hi + off) = h;
                    *reinterpret_cast<uint4*>(ob_lo + off) = l;
                }
                ptx::fence_proxy_async_smem();        // our st.shared -> visible to UMMA
                __syncwarp();
                PROF_ADD(P_SPL_WORK);
                if (lane == 0) {
                    ptx::mbar_arrive_cluster(ptx::mapa_shared(&op_full[sop], 0));   // leader's barrier
                    ptx::mbar_arrive(&f32_empty[s32]);
                }
                if (++s32 == Cfg::S32) { s32 = 0; ph32 ^= 1; }
                if (++sop == Cfg::SOP) { sop = 0; phop ^= 1; }
            }
        }
        if (RANGE) {
            nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
            if (nonfinite && lane == 0) atomicOr(p.range_flag, 1u);
        }
    } else if (warp >= Cfg::EPI_WARP0) {
        // ------------------------------------------------ combine + epilogue (both CTAs)
        ptx::setmaxnreg_inc<Cfg::REGS_EPI>();
        constexpr int HALF = Cfg::BN / 2;
        const uint32_t e = warp - Cfg::EPI_WARP0;
        const uint32_t q = warp & 3;
        const uint32_t h = e >> 2;
        const float scale = MODE == 0 ? (1.0f / 2048.0f) : 1.0f;
        const uint32_t acc_empty_leader = ptx::mapa_shared(&acc_empty[0], 0);
        uint32_t acc_it = 0;
        for (long long t = cid; t < p.num_tiles; t += ncl) {
            int b, mt, nt;
            pair_tile_coords(p, t, b, mt, nt);
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
                const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * 2 * Cfg::BN + h * HALF;
#pragma unroll
                for (int c = 0; c < HALF / 16; ++c) {
                    float vh[16], vc[16];
                    ptx::tmem_ld16(taddr + c * 16, vh);
                    ptx::tmem_ld16(taddr + Cfg::BN + c * 16, vc);
                    ptx::tmem_wait_ld();
                    if (p.corr) {
#pragma unroll
                        for (int j = 0; j < 16; j += 2)
                            combine2(creg[c * 16 + j], creg[c * 16 + j + 1], vh[j], vh[j + 1], vc[j], vc[j + 1], scale);
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) creg[c * 16 + j] = __fadd_rn(creg[c * 16 + j], vh[j]);
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(acc_empty_leader + buf * 8);
                PROF_ADD(P_EPI_DRAIN);
            }
            PROF_T0();
            const int mrow0 = mt * 256 + (int)rank * Cfg::BM;
            if (p.tma_store) {
                // stage the C tile (in CSTAGE_PARTS column parts) and TMA-store it
                const bool leader = (e == 0 && lane == 0);
                const uint32_t r = q * 32 + lane;
                constexpr int PART = Cfg::BN / Cfg::CSTAGE_PARTS;
#pragma unroll
                for (int part = 0; part < Cfg::CSTAGE_PARTS; ++part) {
                    if (leader) ptx::bulk_wait_group_read0();   // staging buffer free
                    ptx::named_bar_sync(1, Cfg::NUM_EPI_WARPS * 32);
                    if (Cfg::CSTAGE_PARTS == 1 || h == (uint32_t)part) {
                        float* dst = cstage + (Cfg::CSTAGE_PARTS == 1 ? h * HALF * Cfg::BM : 0);
#pragma unroll
                        for (int j = 0; j < HALF; ++j) dst[j * Cfg::BM + r] = fmaf(p.alpha, creg[j], 0.0f);
                        ptx::fence_proxy_async_smem();
                    }
                    ptx::named_bar_sync(1, Cfg::NUM_EPI_WARPS * 32);
                    if (leader) {
#pragma unroll
                        for (int c = 0; c < PART / 32; ++c)
                            ptx::tma_store_3d(&tmC, cstage + c * 32 * Cfg::BM, mrow0, nt * Cfg::BN + part * PART + c * 32, b);
                        ptx::bulk_commit_group();
                    }
                }
            } else {
                const int r = mrow0 + (int)(q * 32 + lane);
                const int col0 = nt * Cfg::BN + (int)(h * HALF);
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
        if (p.tma_store && warp == Cfg::EPI_WARP0 && lane == 0) ptx::bulk_wait_group0();
    }
#ifdef EMU_PROF
    if (warp == 0 || warp == 1 || warp >= 4 || lane == 0) {
        prof_acc[P_CTA_TOTAL] = (warp == 4 && lane == 0) ? (unsigned long long)(clock64() - prof_start) : 0;
        if (warp != 2 && warp != 3) PROF_FLUSH();
    }
#endif

    ptx::tc_fence_before();
    ptx::cluster_sync();   // all MMAs into both CTAs' TMEM are complete and drained
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
    }
}

}  // namespace emu
