// gemm_pair_ts_sm100.cuh -- CTA-pair kernel with the A operand in TENSOR memory.
//
// The paper's point is that the split operands should not
// make an extra round trip through shared memory.  On B200 the tensor core can
// take A from TMEM: here the splitter warps write A_hi / A_lo with tcgen05.st
// straight into TMEM (each warp its own 32-lane quadrant, lane = row m, K along
// 32-bit columns, two FP16 values per column), so per 32-k stage and CTA the
// shared-memory traffic drops from 108 KB (A and B both staged and read by the
// MMA) to 68 KB (TMA writes and splitter reads of the FP32 tiles, B_hi/B_lo
// writes, tensor-core reads of B only).
//
// Tile (per cluster of two CTAs): 256 (m) x BN (n); MMA cta_group::2, M = 256,
// N = BN per instruction (tools/probe_mma: A-from-TMEM MMAs run at the full
// tensor rate for any N multiple of 16).  TMEM per CTA: DBUF accumulator buffers
// of (D_hi, D_corr) x BN columns, then the A stages:
//   BN = 128 (default): 1 buffer (256 columns).  With SPLITC the correction
//             products (P2, P3 -> D_corr) and P1 (-> D_hi) of a k-block have their
//             own full/empty barriers, so the drain of D_corr overlaps P1 and the
//             drain of D_hi overlaps the next k-block's P2/P3;
//   BN =  64: 2 buffers (256 columns) -- for problems with fewer 256 x 128 tiles
//             than clusters (twice the clusters at work; c4);
//   BN =  96: 2 buffers (384 columns) -- the MMA of k-block j+1 overlaps the
//             drain of k-block j (kept for comparison, EMU_TS_N=96).
// (In this kernel, splitting a 128-wide tile's accumulators into two N = 64 groups was
// much slower -- profiles/r02_summary.md.)
// Streaming tiles load A with L2 evict_last and B with evict_first (p.l2_policy).
// Long-k streaming tiles (LONGK) may take their tiles in a dynamic order (p.clc): the grid
// has one cluster per tile, the resident clusters take over the others with cluster launch
// control (a scheduler thread in the leader CTA claims the next tile p.clc k-stages before
// the current tile's loads end and multicasts the response to both CTAs; every role reads
// it from a 2-slot ring), so the row blocks of a raster group that read the same B panel
// start it together and the panel is reused in L2 (c3 DRAM reads 70 -> ~35 GB per launch).
// A-stationary (ASTAT, short k): the split A of a whole (batch item, 256-row block)
// -- all k, hi and lo -- stays in TMEM (k <= 256 FP16, k <= 128 TF32) while the
// cluster walks every n-tile of that row block, so A is loaded and split once per
// row block instead of once per n-tile (c2: a third less splitter work).
// CTA r stages A rows [256 mt + 128 r, +128) and B columns [BN nt + BN/2 r, +BN/2).
#pragma once

#include <cstdint>
#include <cuda.h>

#include "gemm_sm100.cuh"
#include "sm100_ptx.cuh"
#include "split.cuh"

#ifndef EMU_TS_SOP16
#define EMU_TS_SOP16 5   // FP16 operand slots (short k; tuning: -DEMU_TS_SOP16=n)
#endif
#ifndef EMU_TS_S32
#define EMU_TS_S32 5     // FP32 stages at most (short k; tuning: -DEMU_TS_S32=n)
#endif
#ifndef EMU_TS_REGS_CTRL
#define EMU_TS_REGS_CTRL 40    // setmaxnreg of the control / splitter warps (tuning)
#endif
#ifndef EMU_TS_REGS_SPLIT
#define EMU_TS_REGS_SPLIT 56
#endif

namespace emu {

// LONGK_ (long-k streaming tiles, c3): no C staging area (the epilogue stores with
// st.global -- once per tile, negligible at long k), its 64 KB spent on deeper rings:
// FP16 8 operand slots (a whole KB = 128 k-block plus half of the next) and 6 FP32 stages
template <int MODE, int BN_ = 128, bool SPLITC_ = true, bool ASTAT_ = false, bool LONGK_ = false>
struct PairTsCfg {
    static constexpr bool LONGK = LONGK_ && !ASTAT_;
    static constexpr int BM = 128;                      // A rows per CTA (pair M = 256)
    static constexpr int BN = BN_;                      // pair tile N = D columns per CTA
    static constexpr int BNC = BN / 2;                  // B columns staged per CTA
    static constexpr int DBUF = BN <= 96 ? 2 : 1;       // accumulator buffers in TMEM
    static constexpr bool SPLITC = SPLITC_ && DBUF == 1;
    static constexpr bool ASTAT = ASTAT_ && SPLITC;
    static constexpr int BK = 32;
    static constexpr int ESZ = MODE == 0 ? 2 : 4;
    static constexpr int KSTEP = MODE == 0 ? 16 : 8;
    static constexpr int NSTEPS = BK / KSTEP;
    static constexpr uint32_t A32_BYTES = BK * BM * 4;     // 16 KB
    static constexpr uint32_t B32_BYTES = BK * BNC * 4;    //  8 KB
    static constexpr uint32_t F32_STAGE = A32_BYTES + B32_BYTES;
    static constexpr uint32_t BOP_BYTES = BNC * BK * ESZ;  // one of B_hi / B_lo
    static constexpr uint32_t OP_STAGE = 2 * BOP_BYTES;
    static constexpr uint32_t CSTAGE_BYTES = LONGK ? 0 : BM * BN * 4;  // TMA-store staging (48 / 64 KB)
    static constexpr uint32_t B_ROW = BK * ESZ;            // 64 (FP16) / 128 (TF32) bytes
    static constexpr uint32_t B_SBO = 8 * B_ROW;
    static constexpr uint32_t B_LAYOUT = MODE == 0 ? 4 : 2;
    // TMEM columns: buffer u: D_hi [2 BN u, +BN), D_corr [2 BN u + BN, +BN); A stages
    // from A_COL0: per slot A_hi (ACOLS/2 columns) then A_lo
    static constexpr uint32_t ACOLS = MODE == 0 ? 32 : 64;     // 32 k of hi + lo
    static constexpr uint32_t A_COL0 = DBUF * 2 * BN;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int ASLOTS = (TMEM_COLS - A_COL0) / ACOLS;   // A stages TMEM holds
    // operand ring: B_hi/B_lo in shared memory (and the A stage in TMEM unless ASTAT);
    // FP16: 5 slots still leave room for 5 FP32 stages
    static constexpr int SOP_MAX = MODE == 0 ? (LONGK ? 8 : EMU_TS_SOP16) : 4;
    static constexpr int SOP = ASLOTS < SOP_MAX ? ASLOTS : SOP_MAX;
    // FP32 stages: as many as fit next to the operand ring and C staging (<= 5)
    static constexpr int S32_FIT = (232448 - 2048 - SOP * OP_STAGE - CSTAGE_BYTES) / F32_STAGE;
    static constexpr int S32_MAX = LONGK ? 6 : EMU_TS_S32;
    static constexpr int S32 = S32_FIT < S32_MAX ? S32_FIT : S32_MAX;
    static constexpr uint32_t KCOLS = 8;                       // TMEM columns per MMA K step
    static_assert(A_COL0 + SOP * ACOLS <= TMEM_COLS, "TMEM budget");
    // CLC (long-k streaming tiles, p.clc): two 16-byte cluster-launch-control responses
    // and their full / empty barriers precede the other barriers
    static constexpr bool DYN = LONGK || ASTAT;   // may take its units in the dynamic order
    static constexpr uint32_t CLC_BYTES = DYN ? 32 + 8 * 6 : 0;
    static constexpr int CLC_CONSUMERS = 2 * 1 + 1 + 2 * 8 + 2 * 16;   // producer x2, MMA, splitter, combine warps
    static constexpr uint32_t BAR_BYTES = CLC_BYTES + 8 * (2 * S32 + 2 * SOP + 4 + ASLOTS) + 16;
    static constexpr uint32_t SMEM_BYTES = 1024 + S32 * F32_STAGE + SOP * OP_STAGE + CSTAGE_BYTES + BAR_BYTES;
    // warpgroup 0: producer, MMA issuer, 2 idle; warpgroups 1-2: 8 splitter warps
    // (2 per TMEM lane quadrant, 16 k each); warpgroups 3-6: 16 combine warps (4 per
    // lane quadrant, BN/4 accumulator columns each -- a short drain matters because
    // the MMA waits for it)
    static constexpr int SPLIT_WARP0 = 4, NUM_SPLIT_WARPS = 8;
    static constexpr int EPI_WARP0 = 12, NUM_EPI_WARPS = 16;
    static constexpr int B_THREADS = BNC * 4;                // splitter threads with B work (2 chunks each)
    static_assert(B_THREADS <= 32 * 8, "B split work");
    static constexpr int NUM_THREADS = 32 * (EPI_WARP0 + NUM_EPI_WARPS);
    static constexpr int KS = BK / (NUM_SPLIT_WARPS / 4);   // k per splitter warp (A)
    static constexpr int ECOLS = BN / (NUM_EPI_WARPS / 4);  // accumulator columns per combine warp
    // SPLITC: the combine holds one part (D_corr) in registers while P1 runs
    static constexpr uint32_t REGS_CTRL = EMU_TS_REGS_CTRL, REGS_SPLIT = SPLITC ? EMU_TS_REGS_SPLIT : 64,
                              REGS_EPI = SPLITC ? 88 : 80;
    static_assert(128 * REGS_CTRL + 32 * NUM_SPLIT_WARPS * REGS_SPLIT + 32 * NUM_EPI_WARPS * REGS_EPI <= 65536,
                  "register budget");
    static_assert(SMEM_BYTES <= 232448, "shared memory");
    static_assert(SOP >= 2, "TMEM budget for A stages");
    static_assert(ECOLS % 8 == 0, "combine columns");
    static_assert(!SPLITC || ECOLS % 16 == 0, "split-commit combine drains 16-column chunks");
};

// tile j of work unit u: A-stationary -> n-tile j of (batch, m-pair) row block u;
// otherwise unit u is tile u of the grouped raster
template <bool ASTAT>
__device__ __forceinline__ void ts_unit_tile(const GemmParams& p, long long u, int j, int& b, int& mt, int& nt)
{
    if (ASTAT) {
        b = (int)(u / p.tiles_m);
        mt = (int)(u - (long long)b * p.tiles_m);
        nt = j;
    } else {
        tile_coords(p, u, b, mt, nt);
    }
}

// Operand and epilogue hooks of the kernel (the pipelined form of the device API,
// include/emu_tcec_pipeline.cuh).  The library's own GEMMs use these defaults: both
// FP32 operands come from global memory through TMA, the epilogue is the library's
// C = alpha * C_acc + beta * C_old store.  A user type replaces either operand by a
// rule evaluated by the splitter warps (foreach_ij; the operand never
// exists in memory) and / or the store:
//   gen_a:  __device__ float a(int batch, int i, int p) const   A_b(i, p), i < m, p < k
//   gen_b:  __device__ float b(int batch, int p, int j) const   B_b(p, j), p < k, j < n
//   custom_store: __device__ void store(int batch, int i, int j0, const float* c, int cols) const
//           C_b(i, j0 + jj) from the FP32 accumulator c[jj], jj < cols (i < m, j0 + jj < n)
struct lib_operands {
    static constexpr bool gen_a = false, gen_b = false, custom_store = false;
    __device__ float a(int, int, int) const { return 0.0f; }
    __device__ float b(int, int, int) const { return 0.0f; }
    __device__ void store(int, int, int, const float*, int) const {}
};

// TA / TB: op(A) = A^T (A stored k x m, k contiguous) / op(B) = B^T (B stored n x k):
// only the TMA boxes and the splitters' shared-memory reads change (NEXT row 2)
// RANGE (bit mask): 1 compiles in the FP16 overflow flag (p.range_flag), 2 the range-safe
// mode's power-of-two scaling (p.row_max / p.col_max, R#22); each still enabled by its pointer.
// MC: epilogue stores every tile to p.dst[0 .. num_dst-1] (fused all-gather, NEXT row 3)
template <int MODE, int RANGE, int BN, bool SPLITC_, bool ASTAT_, bool TA = false, bool TB = false, bool MC = false,
          bool LONGK_ = false, class Ops = lib_operands>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairTsCfg<MODE, BN, SPLITC_, ASTAT_, LONGK_>::NUM_THREADS, 1)
emu_sgemm_pair_ts_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmC, const GemmParams p, const Ops ops = Ops())
{
    using Cfg = PairTsCfg<MODE, BN, SPLITC_, ASTAT_, LONGK_>;
    constexpr bool ASTAT = Cfg::ASTAT;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* f32buf = smem;
    uint8_t* opbuf = smem + Cfg::S32 * Cfg::F32_STAGE;
    float* cstage = reinterpret_cast<float*>(opbuf + Cfg::SOP * Cfg::OP_STAGE);
    uint8_t* barbase = opbuf + Cfg::SOP * Cfg::OP_STAGE + Cfg::CSTAGE_BYTES;   // 1024-byte aligned
    uint4* clc_resp = reinterpret_cast<uint4*>(barbase);                       // [2] (CLC_BYTES)
    uint64_t* clc_full = reinterpret_cast<uint64_t*>(barbase + 32);           // [2]
    uint64_t* clc_empty = clc_full + 2;                                        // [2] (leader's used)
    uint64_t* clc_req = clc_empty + 2;                                         // [1] (leader): claim now
    uint64_t* bars = reinterpret_cast<uint64_t*>(barbase + Cfg::CLC_BYTES);
    uint64_t* f32_full = bars;
    uint64_t* f32_empty = f32_full + Cfg::S32;
    uint64_t* op_full = f32_empty + Cfg::S32;
    uint64_t* op_empty = op_full + Cfg::SOP;
    uint64_t* acc_full = op_empty + Cfg::SOP;   // [DBUF] (SPLITC: [0] D_hi, [1] D_corr)
    uint64_t* acc_empty = acc_full + 2;
    uint64_t* aslot_empty = acc_empty + 2;      // [ASLOTS] (ASTAT)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aslot_empty + Cfg::ASLOTS);

    const uint32_t warp = ptx::warp_id();
    const uint32_t lane = ptx::lane_id();
    const uint32_t rank = ptx::cluster_ctarank();
    const long long cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const long long num_units = p.num_units;
    const int R = ASTAT ? p.unit_tiles : 1;
    // tile order: static (cluster c takes units c, c + ncl, ...) or, with CLC, the unit of
    // each cluster launch this cluster cancels (in launch order: the clusters that share an
    // operand panel start it close together, so it is reused in L2)
    const bool clc = Cfg::DYN && p.clc != 0;
    auto clc_next = [&](uint32_t& ci, bool arrive) -> long long {
        const uint32_t slot = ci & 1u, ph = (ci >> 1) & 1u;
        ++ci;
        ptx::mbar_wait(&clc_full[slot], ph);
        const int x = ptx::clc_first_ctaid_x(&clc_resp[slot]);
        ptx::fence_proxy_async_smem();   // our read before the next async-proxy write of the slot
        __syncwarp(__activemask());
        if (arrive) ptx::mbar_arrive_cluster(ptx::mapa_shared(&clc_empty[slot], 0));
        return x < 0 ? -1 : (long long)(x >> 1);
    };
    PROF_DECL
    TRACE_DECL
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
        for (int i = 0; i < Cfg::ASLOTS; ++i) ptx::mbar_init(&aslot_empty[i], 1);
        if (Cfg::DYN) {
            for (int i = 0; i < 2; ++i) {
                ptx::mbar_init(&clc_full[i], 1);
                ptx::mbar_init(&clc_empty[i], Cfg::CLC_CONSUMERS);
            }
            ptx::mbar_init(clc_req, 1);
        }
        ptx::fence_mbar_init();
        if (!Ops::gen_a) ptx::prefetch_tmap(&tmA);
        if (!Ops::gen_b) ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_wait_then_allow_next();   // prologue done: wait for the previous kernel on the stream

    const int nks = p.num_k_stages;
    const int nkb = (nks + p.kb_stages - 1) / p.kb_stages;

    if (warp < 4) {
        ptx::setmaxnreg_dec<Cfg::REGS_CTRL>();
        if (warp == 0) {
            // -------------------------------------------- TMA producer (both CTAs)
            if (ptx::elect_one()) {
                uint32_t s = 0, ph = 0;
                // L2 hints (tuning, EMU_L2_POLICY): bit 0 -> B evict_first, bit 1 -> A evict_last
                // bit 4 (tuning): B evict_last instead of evict_first
                const uint64_t pol_a = ptx::l2_policy_evict_last(),
                               pol_b = (p.l2_policy & 16) ? ptx::l2_policy_evict_last() : ptx::l2_policy_evict_first();
                auto load = [&](uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2, bool hint,
                                uint64_t pol) {
                    if (hint) ptx::tma_load_3d(dst, map, bar, c0, c1, c2, pol);
                    else ptx::tma_load_3d_nohint(dst, map, bar, c0, c1, c2);
                };
                const bool hint_a = (p.l2_policy & 2) != 0, hint_b = (p.l2_policy & 17) != 0;
                uint32_t ci = 0;
                for (long long u = cid; u >= 0 && u < num_units; u = clc ? clc_next(ci, true) : u + ncl) {
                    for (int j = 0; j < R; ++j) {
                        int b, mt, nt;
                        ts_unit_tile<ASTAT>(p, u, j, b, mt, nt);
                        const int ab = p.a_batched ? b : 0, bb = p.b_batched ? b : 0;
                        const bool loadA = !ASTAT || j == 0;
                        for (int ks = 0; ks < nks; ++ks) {
                            PROF_T0();
                            ptx::mbar_wait_sleep(&f32_empty[s], ph ^ 1);
                            PROF_ADD(P_PROD_WAIT_EMPTY);
                            // CLC: the next unit is claimed p.clc stages before this one's loads end,
                            // so the clusters that share an operand panel start it close together
                            if (clc && rank == 0 && j == R - 1 && ks == max(nks - p.clc, 0)) ptx::mbar_arrive(clc_req);
                            uint8_t* dst = f32buf + s * Cfg::F32_STAGE;
                            TRACE_AT(0, 1, ks);
                            // generated operands (Ops::gen_a / gen_b) are not loaded: the splitter
                            // warps evaluate them
                            const uint32_t bytes = (loadA && !Ops::gen_a ? Cfg::A32_BYTES : 0u) +
                                                   (Ops::gen_b ? 0u : Cfg::B32_BYTES);
                            if (bytes) ptx::mbar_arrive_expect_tx(&f32_full[s], bytes);
                            else ptx::mbar_arrive(&f32_full[s]);
                            if (loadA && !Ops::gen_a) {
                                if (TA)   // [128 m][32 k], SWIZZLE_128B rows
                                    load(dst, &tmA, &f32_full[s], ks * Cfg::BK, mt * 256 + rank * Cfg::BM, ab,
                                         hint_a, pol_a);
                                else      // [32 k][128 m]
                                    load(dst, &tmA, &f32_full[s], mt * 256 + rank * Cfg::BM, ks * Cfg::BK, ab,
                                         hint_a, pol_a);
                            }
                            if (Ops::gen_b) {
                            } else if (TB)   // [32 k][BN/2 n]
                                load(dst + Cfg::A32_BYTES, &tmB, &f32_full[s], nt * Cfg::BN + rank * Cfg::BNC,
                                     ks * Cfg::BK, bb, hint_b, pol_b);
                            else          // [BN/2 n][32 k], SWIZZLE_128B rows
                                load(dst + Cfg::A32_BYTES, &tmB, &f32_full[s], ks * Cfg::BK,
                                     nt * Cfg::BN + rank * Cfg::BNC, bb, hint_b, pol_b);
                            if (++s == Cfg::S32) { s = 0; ph ^= 1; }
                        }
                    }
                }
            }
        } else if (warp == 1) {
            // -------------------------------------------- MMA issuer (leader CTA only)
            if (rank == 0 && ptx::elect_one()) {
                constexpr uint32_t idesc = ptx::instr_desc(MODE == 0 ? 0u : 2u, 0u, 0u, 256, Cfg::BN);
                // B operand descriptor of slot 0, K step 0; slot s / step st / the lo part add their
                // byte offsets >> 4 to the start-address field (shared memory < 256 KB: no carry)
                const uint64_t dB0 = ptx::smem_desc(ptx::smem_u32(opbuf), 16, Cfg::B_SBO, Cfg::B_LAYOUT);
                uint32_t s0 = 0, ph0 = 0, acc_it = 0;
                if constexpr (Cfg::SPLITC) {
                    // per k-block: P2 + P3 into D_corr (barrier pair 1), then P1 into D_hi (pair 0)
                    const uint32_t d_hi = tmem_base, d_corr = tmem_base + Cfg::BN;
                    uint32_t ci = 0;
                    for (long long u = cid; u >= 0 && u < num_units; u = clc ? clc_next(ci, true) : u + ncl) {
                        for (int j = 0; j < R; ++j) {
                            const bool lastA = ASTAT && j == R - 1;   // release the A slots after this tile
                            for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                                const int ks0 = kb * p.kb_stages;
                                const int ks1 = min(ks0 + p.kb_stages, nks);
                                const uint32_t aph = acc_it & 1u;
                                PROF_T0();
                                ptx::mbar_wait(&acc_empty[1], aph ^ 1u);
                                PROF_ADD(P_MMA_WAIT_ACC);
                                TRACE_AT(1, 5, kb);
                                ptx::tc_fence_after();
                                // P2 + P3 of stage ks (operand slot s) into D_corr; P1 into D_hi
                                auto issue_corr = [&](int ks, uint32_t s) {
                                    if (!p.corr) return;
                                    const uint32_t a_hi = tmem_base + Cfg::A_COL0 + (ASTAT ? ks : s) * Cfg::ACOLS;
                                    const uint32_t a_lo = a_hi + Cfg::ACOLS / 2;
                                    const uint64_t dB_s = dB0 + (uint64_t)((s * Cfg::OP_STAGE) >> 4);
#pragma unroll
                                    for (int st = 0; st < Cfg::NSTEPS; ++st) {
                                        const uint64_t dB_hi = dB_s + (uint64_t)(st * 2);   // +32 bytes per K step
                                        const uint64_t dB_lo = dB_s + (uint64_t)((Cfg::BOP_BYTES >> 4) + st * 2);
                                        const uint32_t ka = st * Cfg::KCOLS;
                                        const uint32_t acc = (ks > ks0 || st > 0) ? 1u : 0u;
                                        if (MODE == 0) {
                                            ptx::mma_f16_pair_ts(d_corr, a_lo + ka, dB_hi, idesc, acc);   // P2
                                            ptx::mma_f16_pair_ts(d_corr, a_hi + ka, dB_lo, idesc, 1u);    // P3
                                        } else {
                                            ptx::mma_tf32_pair_ts(d_corr, a_lo + ka, dB_hi, idesc, acc);
                                            ptx::mma_tf32_pair_ts(d_corr, a_hi + ka, dB_lo, idesc, 1u);
                                        }
                                    }
                                };
                                auto issue_hi = [&](int ks, uint32_t s) {
                                    const uint32_t a_hi = tmem_base + Cfg::A_COL0 + (ASTAT ? ks : s) * Cfg::ACOLS;
                                    const uint64_t dB_s = dB0 + (uint64_t)((s * Cfg::OP_STAGE) >> 4);
#pragma unroll
                                    for (int st = 0; st < Cfg::NSTEPS; ++st) {
                                        const uint64_t dB_hi = dB_s + (uint64_t)(st * 2);
                                        const uint32_t acc = (ks > ks0 || st > 0) ? 1u : 0u;
                                        if (MODE == 0)
                                            ptx::mma_f16_pair_ts(d_hi, a_hi + st * Cfg::KCOLS, dB_hi, idesc, acc);   // P1
                                        else
                                            ptx::mma_tf32_pair_ts(d_hi, a_hi + st * Cfg::KCOLS, dB_hi, idesc, acc);
                                    }
                                    ptx::tc_commit_pair(&op_empty[s], 0x3);   // B (and non-stationary A) slot free
                                    if (lastA) ptx::tc_commit_pair(&aslot_empty[ks], 0x3);
                                };
                                if (ks1 - ks0 <= Cfg::SOP) {
                                    // the whole k-block fits the operand ring: P2 + P3 of every
                                    // stage, commit D_corr (its drain overlaps P1), then P1
                                    uint32_t s = s0, ph = ph0;
                                    for (int ks = ks0; ks < ks1; ++ks) {
                                        PROF_T0();
                                        ptx::mbar_wait(&op_full[s], ph);
                                        PROF_ADD(P_MMA_WAIT_OP);
                                        TRACE_AT(1, 9, ks);
                                        ptx::tc_fence_after();
                                        PROF_T0();
                                        issue_corr(ks, s);
                                        PROF_ADD(P_MMA_ISSUE);
                                        if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                                    }
                                    ptx::tc_commit_pair(&acc_full[1], 0x3);
                                    TRACE_AT(1, 6, kb);
                                    PROF_T0();
                                    ptx::mbar_wait(&acc_empty[0], aph ^ 1u);
                                    PROF_ADD(P_MMA_WAIT_ACC);
                                    TRACE_AT(1, 7, kb);
                                    ptx::tc_fence_after();
                                    PROF_T0();
                                    s = s0; ph = ph0;
                                    for (int ks = ks0; ks < ks1; ++ks) {
                                        issue_hi(ks, s);
                                        if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                                    }
                                    s0 = s; ph0 = ph;
                                } else {
                                    // a k-block longer than the operand ring is issued in chunks of
                                    // <= SOP stages: P2 + P3 of a chunk, then its P1 (which frees the
                                    // chunk's slots); D_corr is committed before the last chunk's P1,
                                    // so its drain still overlaps P1.  Each accumulator sees its
                                    // stages in ascending order either way.
                                    for (int c0 = ks0; c0 < ks1; c0 += Cfg::SOP) {
                                        const int c1 = min(c0 + Cfg::SOP, ks1);
                                        uint32_t s = s0, ph = ph0;
                                        for (int ks = c0; ks < c1; ++ks) {
                                            ptx::mbar_wait(&op_full[s], ph);
                                            ptx::tc_fence_after();
                                            issue_corr(ks, s);
                                            if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                                        }
                                        if (c1 == ks1) ptx::tc_commit_pair(&acc_full[1], 0x3);
                                        if (c0 == ks0) {
                                            ptx::mbar_wait(&acc_empty[0], aph ^ 1u);
                                            ptx::tc_fence_after();
                                        }
                                        s = s0; ph = ph0;
                                        for (int ks = c0; ks < c1; ++ks) {
                                            issue_hi(ks, s);
                                            if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                                        }
                                        s0 = s; ph0 = ph;
                                    }
                                }
                                ptx::tc_commit_pair(&acc_full[0], 0x3);
                                PROF_ADD(P_MMA_ISSUE);
                                TRACE_AT(1, 8, kb);
                            }
                        }
                    }
                } else {
                    uint32_t ci = 0;
                    for (long long u = cid; u >= 0 && u < num_units; u = clc ? clc_next(ci, true) : u + ncl) {
                        for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                            const int ks0 = kb * p.kb_stages;
                            const int ks1 = min(ks0 + p.kb_stages, nks);
                            const uint32_t buf = Cfg::DBUF == 2 ? (acc_it & 1u) : 0u;
                            const uint32_t aph = (Cfg::DBUF == 2) ? ((acc_it >> 1) & 1u) : (acc_it & 1u);
                            const uint32_t d_hi = tmem_base + buf * 2 * Cfg::BN, d_corr = d_hi + Cfg::BN;
                            PROF_T0();
                            ptx::mbar_wait(&acc_empty[buf], aph ^ 1u);
                            PROF_ADD(P_MMA_WAIT_ACC);
                            ptx::tc_fence_after();
                            uint32_t s = s0, ph = ph0;
                            for (int ks = ks0; ks < ks1; ++ks) {
                                PROF_T0();
                                ptx::mbar_wait(&op_full[s], ph);
                                PROF_ADD(P_MMA_WAIT_OP);
                                ptx::tc_fence_after();
                                PROF_T0();
                                const uint32_t a_hi = tmem_base + Cfg::A_COL0 + s * Cfg::ACOLS;
                                const uint32_t a_lo = a_hi + Cfg::ACOLS / 2;
                                const uint64_t dB_s = dB0 + (uint64_t)((s * Cfg::OP_STAGE) >> 4);
#pragma unroll
                                for (int st = 0; st < Cfg::NSTEPS; ++st) {
                                    const uint64_t dB_hi = dB_s + (uint64_t)(st * 2);
                                    const uint64_t dB_lo = dB_s + (uint64_t)((Cfg::BOP_BYTES >> 4) + st * 2);
                                    const uint32_t ka = st * Cfg::KCOLS;
                                    const uint32_t acc = (ks > ks0 || st > 0) ? 1u : 0u;
                                    if (MODE == 0) {
                                        ptx::mma_f16_pair_ts(d_hi, a_hi + ka, dB_hi, idesc, acc);        // P1
                                        if (p.corr) {
                                            ptx::mma_f16_pair_ts(d_corr, a_lo + ka, dB_hi, idesc, acc);  // P2
                                            ptx::mma_f16_pair_ts(d_corr, a_hi + ka, dB_lo, idesc, 1u);   // P3
                                        }
                                    } else {
                                        ptx::mma_tf32_pair_ts(d_hi, a_hi + ka, dB_hi, idesc, acc);
                                        if (p.corr) {
                                            ptx::mma_tf32_pair_ts(d_corr, a_lo + ka, dB_hi, idesc, acc);
                                            ptx::mma_tf32_pair_ts(d_corr, a_hi + ka, dB_lo, idesc, 1u);
                                        }
                                    }
                                }
                                ptx::tc_commit_pair(&op_empty[s], 0x3);   // slot free
                                PROF_ADD(P_MMA_ISSUE);
                                if (++s == Cfg::SOP) { s = 0; ph ^= 1; }
                            }
                            ptx::tc_commit_pair(&acc_full[buf], 0x3);
                            s0 = s; ph0 = ph;
                        }
                    }
                }
            }
        } else if (warp == 3) {
            // -------------------------------------------- CLC scheduler (leader CTA): keeps the
            // next unit's response one ahead of the roles that consume it
            if (clc && rank == 0 && ptx::elect_one()) {
                const uint32_t peer_full = ptx::mapa_shared(&clc_full[0], 1);
                for (uint32_t i = 0;; ++i) {
                    const uint32_t slot = i & 1u, ph = (i >> 1) & 1u;
                    ptx::mbar_wait_sleep(clc_req, i & 1u);   // the producer nears the end of its unit
                    ptx::mbar_wait(&clc_empty[slot], ph ^ 1u);
                    ptx::mbar_arrive_expect_tx(&clc_full[slot], 16);
                    ptx::mbar_arrive_expect_tx_cluster(peer_full + 8 * slot, 16);
                    ptx::clc_try_cancel(&clc_resp[slot], &clc_full[slot]);
                    ptx::mbar_wait(&clc_full[slot], ph);
                    if (ptx::clc_first_ctaid_x(&clc_resp[slot]) < 0) break;
                }
            }
        }
    } else if (warp < Cfg::EPI_WARP0) {
        // ------------------------------------------------ splitters (256 threads)
        ptx::setmaxnreg_dec<Cfg::REGS_SPLIT>();
        const uint32_t tid = threadIdx.x - Cfg::SPLIT_WARP0 * 32;    // 0..255
        const uint32_t q = warp & 3;                                  // TMEM lane quadrant
        const uint32_t kq = (warp - Cfg::SPLIT_WARP0) >> 2;          // KS-k slice of the stage
        const uint32_t m = q * 32 + lane;                             // A row (TMEM lane)
        const uint32_t n = tid % Cfg::BNC, quarter = tid / Cfg::BNC;  // B: 8 k per thread (tid < B_THREADS)
        const bool has_b = tid < Cfg::B_THREADS;
        const uint32_t tq = tmem_base + ((q * 32u) << 16);
        const uint32_t op_full_leader = ptx::mapa_shared(&op_full[0], 0);   // + 8 * slot
        uint32_t s32 = 0, ph32 = 0, sop = 0, phop = 0, unit_it = 0;
        uint32_t nonfinite = 0;
        const bool chk = (RANGE & 1) && p.range_flag != nullptr;   // the FP16 overflow flag was asked for
        uint32_t ci = 0;
        for (long long u = cid; u >= 0 && u < num_units; u = clc ? clc_next(ci, lane == 0) : u + ncl, ++unit_it) {
            for (int j = 0; j < R; ++j) {
                const bool doA = !ASTAT || j == 0;
                // generated operands: this thread's problem, row of A and column of B
                int gb = 0, grow = 0, gcol = 0;
                if (Ops::gen_a || Ops::gen_b) {
                    int mt_, nt_;
                    ts_unit_tile<ASTAT>(p, u, j, gb, mt_, nt_);
                    grow = mt_ * 256 + (int)rank * Cfg::BM + (int)m;
                    gcol = nt_ * Cfg::BN + (int)rank * Cfg::BNC + (int)n;
                }
                // range-safe mode: this thread's row of A and column of B scale by 2^-e
                float sa = 1.0f, sb = 1.0f;
                if ((RANGE & 2) && p.row_max) {
                    int b, mt, nt;
                    ts_unit_tile<ASTAT>(p, u, j, b, mt, nt);
                    const int r = mt * 256 + (int)rank * Cfg::BM + (int)m;
                    const int c = nt * Cfg::BN + (int)rank * Cfg::BNC + (int)n;
                    if (r < p.m) sa = pow2i(-range_exp_of(p.row_max[(long long)b * p.m + r]));
                    if (has_b && c < p.n) sb = pow2i(-range_exp_of(p.col_max[(long long)b * p.n + c]));
                }
                for (int ks = 0; ks < nks; ++ks) {
                    // operand slot first, then the FP32 stage: a stage is held only while it
                    // is split, so the producer keeps the whole FP32 ring in flight
                    PROF_T0();
                    ptx::mbar_wait(&op_empty[sop], phop ^ 1);
                    if (ASTAT && j == 0) ptx::mbar_wait(&aslot_empty[ks], (unit_it & 1u) ^ 1u);
                    PROF_ADD(P_SPL_WAIT_OP);
                    if (warp == Cfg::SPLIT_WARP0 && lane == 0) TRACE_AT(2, 3, ks);
                    PROF_T0();
                    ptx::mbar_wait(&f32_full[s32], ph32);
                    PROF_ADD(P_SPL_WAIT_F32);
                    if (warp == Cfg::SPLIT_WARP0 && lane == 0) TRACE_AT(2, 2, ks);
                    PROF_T0();
                    ptx::tc_fence_after();
                    const float* fa = reinterpret_cast<const float*>(f32buf + s32 * Cfg::F32_STAGE);
                    const uint8_t* fb = f32buf + s32 * Cfg::F32_STAGE + Cfg::A32_BYTES;
                    uint8_t* ob_hi = opbuf + sop * Cfg::OP_STAGE;
                    uint8_t* ob_lo = ob_hi + Cfg::BOP_BYTES;
                    // ---- load phase: A(m, KS kq .. +KS-1) (a warp reads 32 consecutive m per k),
                    //      B(8 quarter .. +7, n): FP32 16-byte chunks 2 quarter, 2 quarter + 1 of row n
                    float av[Cfg::KS];
                    if (doA && Ops::gen_a) {
                        const int k0 = ks * Cfg::BK + (int)kq * Cfg::KS;
#pragma unroll
                        for (int jj = 0; jj < Cfg::KS; ++jj)
                            av[jj] = (grow < p.m && k0 + jj < p.k) ? ops.a(gb, grow, k0 + jj) : 0.0f;
                    } else if (doA && TA) {
                        // row m holds 32 k (128 bytes, 16-byte chunks XOR-swizzled by m & 7)
                        const uint8_t* ra = reinterpret_cast<const uint8_t*>(fa) + m * 128;
#pragma unroll
                        for (int cc = 0; cc < Cfg::KS / 4; ++cc) {
                            const float4 v = *reinterpret_cast<const float4*>(
                                ra + (((kq * (Cfg::KS / 4) + cc) ^ (m & 7)) << 4));
                            av[4 * cc] = v.x; av[4 * cc + 1] = v.y; av[4 * cc + 2] = v.z; av[4 * cc + 3] = v.w;
                        }
                    } else if (doA) {
#pragma unroll
                        for (int jj = 0; jj < Cfg::KS; ++jj) av[jj] = fa[(kq * Cfg::KS + jj) * Cfg::BM + m];
                    }
                    float4 vb[2];
                    if (has_b && Ops::gen_b) {
                        const int k0 = ks * Cfg::BK + (int)quarter * 8;
                        float x[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) x[i] = (gcol < p.n && k0 + i < p.k) ? ops.b(gb, k0 + i, gcol) : 0.0f;
                        vb[0] = make_float4(x[0], x[1], x[2], x[3]);
                        vb[1] = make_float4(x[4], x[5], x[6], x[7]);
                    } else if (has_b && TB) {
                        // k-row of BN/2 columns: a warp reads 32 consecutive n per k
                        const float* fbt = reinterpret_cast<const float*>(fb);
                        float x[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) x[i] = fbt[(quarter * 8 + i) * Cfg::BNC + n];
                        vb[0] = make_float4(x[0], x[1], x[2], x[3]);
                        vb[1] = make_float4(x[4], x[5], x[6], x[7]);
                    } else if (has_b) {
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            vb[c] = *reinterpret_cast<const float4*>(fb + n * 128 + (((2 * quarter + c) ^ (n & 7)) << 4));
                    }
                    if ((RANGE & 2) && p.row_max) {   // exact power-of-two scaling (RN where the result is subnormal)
                        if (doA) {
#pragma unroll
                            for (int jj = 0; jj < Cfg::KS; jj += 2) scale_f32x2(av[jj], av[jj + 1], sa);
                        }
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            scale_f32x2(vb[c].x, vb[c].y, sb);
                            scale_f32x2(vb[c].z, vb[c].w, sb);
                        }
                    }
                    // ---- A: split into TMEM columns (lane = m)
                    if (doA) {
                        const uint32_t a_hi = tq + Cfg::A_COL0 + (ASTAT ? (uint32_t)ks : sop) * Cfg::ACOLS;
                        const uint32_t a_lo = a_hi + Cfg::ACOLS / 2;
                        if (MODE == 0) {
                            uint32_t h[Cfg::KS / 2], l[Cfg::KS / 2];
#pragma unroll
                            for (int jj = 0; jj < Cfg::KS / 2; ++jj) {
                                split_fp16x2(av[2 * jj], av[2 * jj + 1], h[jj], l[jj]);
                                if (chk) nonfinite |= f16x2_nonfinite(h[jj]);
                            }
                            ptx::tmem_st8(a_hi + kq * (Cfg::KS / 2), h);
                            ptx::tmem_st8(a_lo + kq * (Cfg::KS / 2), l);
                        } else {
#pragma unroll
                            for (int c = 0; c < Cfg::KS / 8; ++c) {
                                uint32_t h[8], l[8];
#pragma unroll
                                for (int jj = 0; jj < 8; ++jj) split_tf32(av[8 * c + jj], h[jj], l[jj]);
                                ptx::tmem_st8(a_hi + kq * Cfg::KS + 8 * c, h);
                                ptx::tmem_st8(a_lo + kq * Cfg::KS + 8 * c, l);
                            }
                        }
                    }
                    // ---- B: split into the K-major operand tile in shared memory
                    if (!has_b) {
                    } else if (MODE == 0) {
                        // one 16-byte FP16 chunk (8 k), K-major SWIZZLE_64B rows
                        uint2 h0, l0, h1, l1;
                        split4_fp16(vb[0], h0, l0);
                        split4_fp16(vb[1], h1, l1);
                        if (chk)
                            nonfinite |= f16x2_nonfinite(h0.x) | f16x2_nonfinite(h0.y) | f16x2_nonfinite(h1.x) |
                                         f16x2_nonfinite(h1.y);
                        const uint32_t off = n * 64 + ((quarter ^ ((n >> 1) & 3)) << 4);
                        *reinterpret_cast<uint4*>(ob_hi + off) = make_uint4(h0.x, h0.y, h1.x, h1.y);
                        *reinterpret_cast<uint4*>(ob_lo + off) = make_uint4(l0.x, l0.y, l1.x, l1.y);
                    } else {
#pragma unroll
                        for (int c = 0; c < 2; ++c) {   // two 16-byte TF32 chunks, K-major SWIZZLE_128B rows
                            const uint32_t jj = 2 * quarter + c;
                            uint4 h, l;
                            split_tf32(vb[c].x, h.x, l.x);
                            split_tf32(vb[c].y, h.y, l.y);
                            split_tf32(vb[c].z, h.z, l.z);
                            split_tf32(vb[c].w, h.w, l.w);
                            const uint32_t off = n * 128 + ((jj ^ (n & 7)) << 4);
                            *reinterpret_cast<uint4*>(ob_hi + off) = h;
                            *reinterpret_cast<uint4*>(ob_lo + off) = l;
                        }
                    }
                    ptx::fence_proxy_async_smem();   // B tiles -> async proxy
                    if (doA) ptx::tmem_wait_st();    // A columns written
                    ptx::tc_fence_before();
                    __syncwarp();
                    PROF_ADD(P_SPL_WORK);
                    if (lane == 0) {
                        ptx::mbar_arrive_cluster(op_full_leader + 8 * sop);
                        ptx::mbar_arrive(&f32_empty[s32]);
                    }
                    if (warp == Cfg::SPLIT_WARP0 && lane == 0) TRACE_AT(2, 4, ks);
                    if (++s32 == Cfg::S32) { s32 = 0; ph32 ^= 1; }
                    if (++sop == Cfg::SOP) { sop = 0; phop ^= 1; }
                }
            }
        }
        if ((RANGE & 1) && p.range_flag) {
            nonfinite = __reduce_or_sync(0xffffffffu, nonfinite);
            if (nonfinite && lane == 0) atomicOr(p.range_flag, 1u);
        }
    } else {
        // ------------------------------------------------ combine + epilogue (both CTAs)
        ptx::setmaxnreg_inc<Cfg::REGS_EPI>();
        constexpr int HALF = Cfg::ECOLS;               // this warp's accumulator columns
        const uint32_t e = warp - Cfg::EPI_WARP0;
        const uint32_t q = warp & 3;
        const uint32_t h = e >> 2;                     // column group: tile columns [HALF h, +HALF)
        const float scale = MODE == 0 ? (1.0f / 2048.0f) : 1.0f;
        const uint32_t acc_empty_leader = ptx::mapa_shared(&acc_empty[0], 0);   // + 8 * buffer
        uint32_t acc_it = 0, ci = 0;
        for (long long u = cid; u >= 0 && u < num_units; u = clc ? clc_next(ci, lane == 0) : u + ncl) {
            for (int j = 0; j < R; ++j) {
                int b, mt, nt;
                ts_unit_tile<ASTAT>(p, u, j, b, mt, nt);
                float creg[HALF];
#pragma unroll
                for (int jj = 0; jj < HALF; ++jj) creg[jj] = 0.0f;
                if constexpr (Cfg::SPLITC) {
                    const uint32_t taddr = tmem_base + ((q * 32u) << 16) + h * HALF;
                    const uint32_t emp_hi = acc_empty_leader, emp_corr = acc_empty_leader + 8;
                    for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                        const uint32_t aph = acc_it & 1u;
                        // D_corr first (P2 + P3 are issued first); hold it while P1 runs
                        PROF_T0();
                        ptx::mbar_wait(&acc_full[1], aph);
                        PROF_ADD(P_EPI_WAIT_ACC);
                        if (lane == 0) TRACE_AT(3 + e, 10, kb);
                        PROF_T0();
                        ptx::tc_fence_after();
                        float vc[HALF / 16][16];   // x16 loads: fewer instructions on the drain
                        if (p.corr) {
#pragma unroll
                            for (int c = 0; c < HALF / 16; ++c) ptx::tmem_ld16(taddr + Cfg::BN + c * 16, vc[c]);
                            ptx::tmem_wait_ld();
                        }
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_cluster(emp_corr);
                        PROF_ADD(P_EPI_DRAIN);
                        if (lane == 0) TRACE_AT(3 + e, 11, kb);
                        PROF_T0();
                        ptx::mbar_wait(&acc_full[0], aph);
                        PROF_ADD(P_EPI_WAIT_ACC);
                        if (lane == 0) TRACE_AT(3 + e, 12, kb);
                        PROF_T0();
                        ptx::tc_fence_after();
#pragma unroll
                        for (int c0 = 0; c0 < HALF / 16; ++c0) {   // 16-column chunks of D_hi
                            float vh[16];
                            ptx::tmem_ld16(taddr + c0 * 16, vh);
                            ptx::tmem_wait_ld();
                            if (c0 + 1 == HALF / 16) {   // last chunk read: release D_hi before the math
                                ptx::tc_fence_before();
                                __syncwarp();
                                if (lane == 0) ptx::mbar_arrive_cluster(emp_hi);
                                if (lane == 0) TRACE_AT(3 + e, 13, kb);
                            }
                            float* cr = creg + c0 * 16;
                            const float* cc = vc[c0];
                            if (p.corr) {
#pragma unroll
                                for (int jj = 0; jj < 16; jj += 2)
                                    combine2(cr[jj], cr[jj + 1], vh[jj], vh[jj + 1], cc[jj], cc[jj + 1], scale);
                            } else {
#pragma unroll
                                for (int jj = 0; jj < 16; ++jj) cr[jj] = __fadd_rn(cr[jj], vh[jj]);
                            }
                        }
                        PROF_ADD(P_EPI_DRAIN);
                    }
                } else {
                    for (int kb = 0; kb < nkb; ++kb, ++acc_it) {
                        const uint32_t buf = Cfg::DBUF == 2 ? (acc_it & 1u) : 0u;
                        const uint32_t aph = Cfg::DBUF == 2 ? ((acc_it >> 1) & 1u) : (acc_it & 1u);
                        PROF_T0();
                        ptx::mbar_wait(&acc_full[buf], aph);   // on the critical path: spin, do not sleep
                        PROF_ADD(P_EPI_WAIT_ACC);
                        PROF_T0();
                        ptx::tc_fence_after();
                        const uint32_t taddr = tmem_base + ((q * 32u) << 16) + buf * 2 * Cfg::BN + h * HALF;
                        if constexpr (HALF % 16 == 0) {
                            // x16 loads: one instruction per 16 columns of each part
#pragma unroll
                            for (int c0 = 0; c0 < HALF / 16; ++c0) {
                                float vh[16], vc[16];
                                ptx::tmem_ld16(taddr + c0 * 16, vh);
                                ptx::tmem_ld16(taddr + Cfg::BN + c0 * 16, vc);
                                ptx::tmem_wait_ld();
                                float* cr = creg + c0 * 16;
                                if (p.corr) {
#pragma unroll
                                    for (int jj = 0; jj < 16; jj += 2)
                                        combine2(cr[jj], cr[jj + 1], vh[jj], vh[jj + 1], vc[jj], vc[jj + 1], scale);
                                } else {
#pragma unroll
                                    for (int jj = 0; jj < 16; ++jj) cr[jj] = __fadd_rn(cr[jj], vh[jj]);
                                }
                            }
                        } else {
                        // columns in chunks of 8; CPW chunks loaded per tcgen05.wait::ld
                        constexpr int NCH = HALF / 8, CPW = (HALF <= 24) ? NCH : 2;
#pragma unroll
                        for (int c0 = 0; c0 < NCH; c0 += CPW) {
                            float vh[CPW][8], vc[CPW][8];
#pragma unroll
                            for (int c = 0; c < CPW; ++c) {
                                ptx::tmem_ld8(taddr + (c0 + c) * 8, vh[c]);
                                ptx::tmem_ld8(taddr + Cfg::BN + (c0 + c) * 8, vc[c]);
                            }
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < CPW; ++c) {
                                float* cr = creg + (c0 + c) * 8;
                                if (p.corr) {
#pragma unroll
                                    for (int jj = 0; jj < 8; jj += 2)
                                        combine2(cr[jj], cr[jj + 1], vh[c][jj], vh[c][jj + 1], vc[c][jj], vc[c][jj + 1],
                                                 scale);
                                } else {
#pragma unroll
                                    for (int jj = 0; jj < 8; ++jj) cr[jj] = __fadd_rn(cr[jj], vh[c][jj]);
                                }
                            }
                        }
                        }
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive_cluster(acc_empty_leader + 8 * buf);
                        PROF_ADD(P_EPI_DRAIN);
                    }
                }
                PROF_T0();
                if (lane == 0) TRACE_AT(3 + e, 14, j);
                const int mrow0 = mt * 256 + (int)rank * Cfg::BM;
                if ((RANGE & 2) && p.row_max) {   // range-safe mode: C_acc * 2^(e_i + f_j), one rounding (R#22)
                    const int r = mrow0 + (int)(q * 32 + lane);
                    const int er = r < p.m ? range_exp_of(p.row_max[(long long)b * p.m + r]) : 0;
                    const int colb = nt * Cfg::BN + (int)(h * HALF);
#pragma unroll
                    for (int jj = 0; jj < HALF; ++jj) {
                        const int fc = colb + jj < p.n ? range_exp_of(p.col_max[(long long)b * p.n + colb + jj]) : 0;
                        creg[jj] = ldexp_rn(creg[jj], er + fc);
                    }
                }
                if (Ops::custom_store) {
                    const int r = mrow0 + (int)(q * 32 + lane);
                    const int col0 = nt * Cfg::BN + (int)(h * HALF);
                    if (r < p.m && col0 < p.n) ops.store(b, r, col0, creg, min(HALF, p.n - col0));
                } else if (p.tma_store && (p.l2_policy & 8)) {
                    // (TF32 default, EMU_C_BOX128) the 4 warps of a column group stage their 32-row
                    // blocks into one 128-row x HALF box, stored by one TMA store (512-byte
                    // column segments in global memory instead of 128-byte ones)
                    float* dstg = cstage + h * (128 * HALF);
                    if (q == 0 && lane == 0) ptx::bulk_wait_group_read0();   // the group's previous store
                    ptx::named_bar_sync(1 + h, 128);
#pragma unroll
                    for (int jj = 0; jj < HALF; ++jj) dstg[jj * 128 + q * 32 + lane] = fmaf(p.alpha, creg[jj], 0.0f);
                    ptx::fence_proxy_async_smem();
                    ptx::named_bar_sync(1 + h, 128);
                    if (q == 0 && lane == 0) {
                        ptx::tma_store_3d(&tmC, dstg, mrow0, nt * Cfg::BN + (int)(h * HALF), b);
                        ptx::bulk_commit_group();
                    }
                } else if (p.tma_store) {
                    // each warp stages and TMA-stores its own 32 rows x HALF columns (no
                    // CTA-wide barrier: a warp moves on to the next tile's drains at once)
                    float* dst = cstage + e * (32 * HALF);
                    if (lane == 0) ptx::bulk_wait_group_read0();   // this warp's previous store read its block
                    __syncwarp();
                    if (lane == 0) TRACE_AT(3 + e, 16, j);
#pragma unroll
                    for (int jj = 0; jj < HALF; ++jj) dst[jj * 32 + lane] = fmaf(p.alpha, creg[jj], 0.0f);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) TRACE_AT(3 + e, 17, j);
                    if (lane == 0) {   // box: 32 rows x HALF columns
                        if (p.l2_policy & 4)   // C stores evict_first (tuning, EMU_C_EVICT_FIRST)
                            ptx::tma_store_3d_hint(&tmC, dst, mrow0 + (int)(q * 32), nt * Cfg::BN + (int)(h * HALF), b,
                                                   ptx::l2_policy_evict_first());
                        else
                            ptx::tma_store_3d(&tmC, dst, mrow0 + (int)(q * 32), nt * Cfg::BN + (int)(h * HALF), b);
                        ptx::bulk_commit_group();
                    }
                } else {
                    const int r = mrow0 + (int)(q * 32 + lane);
                    const int col0 = nt * Cfg::BN + (int)(h * HALF);
                    if (r < p.m) {
                        float* cp = p.C + (long long)b * p.strideC + r + (long long)col0 * p.ldc;
                        if (p.beta != 0.0f) {
#pragma unroll
                            for (int jj = 0; jj < HALF; ++jj)
                                if (col0 + jj < p.n) {
                                    float* d = cp + (long long)jj * p.ldc;
                                    *d = fmaf(p.alpha, creg[jj], __fmul_rn(p.beta, *d));
                                }
                        } else {
#pragma unroll
                            for (int jj = 0; jj < HALF; ++jj)
                                if (col0 + jj < p.n) cp[(long long)jj * p.ldc] = fmaf(p.alpha, creg[jj], 0.0f);
                            // fused all-gather (NEXT row 3): the same tile to every other
                            // destination -- peer C buffers over NVLink on a multi-GPU run
                            if constexpr (MC) {
                                for (int d = 1; d < p.num_dst; ++d) {
                                    float* dp = p.dst[d] + r + (long long)col0 * p.ldc;
#pragma unroll
                                    for (int jj = 0; jj < HALF; ++jj)
                                        if (col0 + jj < p.n) dp[(long long)jj * p.ldc] = fmaf(p.alpha, creg[jj], 0.0f);
                                }
                            }
                        }
                    }
                }
                PROF_ADD(P_EPI_STORE);
                if (lane == 0) TRACE_AT(3 + e, 15, j);
            }
        }
        if (p.tma_store && lane == 0) ptx::bulk_wait_group0();
    }
#ifdef EMU_PROF
    if (lane == 0 && warp == 0) TRACE_END(0);
    if (lane == 0 && warp == 1) TRACE_END(1);
    if (lane == 0 && warp == Cfg::SPLIT_WARP0) TRACE_END(2);
    if (lane == 0 && warp >= Cfg::EPI_WARP0) TRACE_END(3 + warp - Cfg::EPI_WARP0);
    if (warp == 0 || warp == 1 || warp >= 4 || lane == 0) {
        prof_acc[P_CTA_TOTAL] = (warp == 4 && lane == 0) ? (unsigned long long)(clock64() - prof_start) : 0;
        if (warp != 2 && warp != 3) PROF_FLUSH();
    }
#endif

    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair<Cfg::TMEM_COLS>(tmem_base);
    }
}

}  // namespace emu
