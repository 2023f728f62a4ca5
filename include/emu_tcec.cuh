/*
 * emu_tcec.cuh -- device-level (in-kernel) API of the B200 emulated SGEMM:
 * the B200 analog of the paper's WMMAe-TCEC (§4.4, P:496-523;
 * SURVEY §8(f) NEXT 2) and of its structured-operand primitives foreach_ij /
 * map.  Header-only; compile with
 *   nvcc -gencode arch=compute_100a,code=sm_100a -I include -I paper_2308_15152_b200/csrc
 * and never with --use_fast_math (R#3: the split needs IEEE subnormals).
 *
 * What it computes.  A CTA of 128 threads owns a 128 x N block of an FP32
 * product C = A B and walks K in stages of BK elements (one 128-byte K row of
 * the low-precision operand: BK = 64 for FP16, 32 for TF32).  Per stage:
 *   load_a / load_b      FP32 operand tile (global or shared memory, column-major);
 *                        or fetch_a / fetch_b into a register fragment + split_a / split_b
 *                        (software pipelining: fetch the next stage before mma())
 *   generate_a / _b      or an operand tile computed from a rule f(i, p) (foreach_ij)
 *   fill_a / set_a ...   or a constant tile with single elements set (map)
 *     -- every path splits in registers straight into the hi / lo operand tiles
 *        (Eqs. corr-1..corr-4; R#6 for TF32) in the tcgen05 shared-
 *        memory layout: no FP32 or FP16 staging copy (Fig. 7)
 *   mma()                P1 = A_hi B_hi -> D_hi, P2 = A_lo B_hi and P3 = A_hi B_lo ->
 *                        D_corr (Eq. corr-5), tcgen05.mma into TMEM,
 *                        issued by one thread, asynchronous
 *   combine()            t = RN(D_hi + D_corr * 2^-11), C += t in FP32 RN on CUDA cores
 *                        (the accumulation outside the tensor core's RZ; R#7/R#8);
 *                        the next mma() restarts D_hi / D_corr
 *   store / acc(j)       C = RN(alpha*C + RN(beta*C_old)), or direct access to the
 *                        FP32 accumulator for a custom epilogue (after sync_acc())
 * TMEM holds two (D_hi, D_corr) buffers: a finished k-block is drained by the
 * next mma() after it has issued the following block, so the CUDA-core combine
 * overlaps the tensor core (4N columns).
 * The combine interval is the caller's: combine() after every KB/BK stages
 * (the library's kernels use KB = 64, R#7).
 *
 * Policies ("policy-based design"): tcec::policy<Op, Ec, Backend>
 *   Op      op_fp16 (kind::f16, FP16 hi + 2^11-scaled lo) | op_tf32 (kind::tf32, R#6)
 *   Ec      with_ec (three products) | without_ec (P1 only: the negative control)
 *   Backend tensor_core (tcgen05.mma) | simt (the same products from the same
 *           shared-memory hi / lo tiles with FP32 FMAs on CUDA cores, sequential
 *           in k: the paper's "software" alternative, for evaluation; N <= 64)
 *
 * Contract.  All member functions except set_a / set_b are CTA-collective:
 * every one of the 128 threads calls them in the same order with the same
 * arguments (like WMMA's warp-collective calls).  blockDim.x == 128.  One tile
 * object per CTA (it allocates 4N tensor-memory columns and relinquishes the
 * allocation permit); call release() before the kernel exits.  Dynamic shared
 * memory of at least tile::SMEM_BYTES must be passed to the constructor.
 * Thread t owns accumulator row t (acc(j) = C(t, j)).
 * set_a / set_b may be called by any subset of threads, only after fill_a /
 * fill_b of the same stage (which ends with a CTA barrier), and only on
 * elements no other thread sets in that stage.
 * Ownership: pointers passed in are read (load_*) or written (store) only
 * during the call; nothing is retained.  No error reporting: out-of-range
 * indices are the caller's bug (rows / cols / kvalid bound every access).
 */
#pragma once

#include <cstdint>

#include "sm100_ptx.cuh"
#include "split.cuh"

namespace emu {
namespace tcec {

// ------------------------------------------------------------------ policies
struct op_fp16 { static constexpr int mode = 0; };
struct op_tf32 { static constexpr int mode = 1; };
struct with_ec { static constexpr bool ec = true; };
struct without_ec { static constexpr bool ec = false; };
struct tensor_core { static constexpr bool tc = true; };
struct simt { static constexpr bool tc = false; };

template <class Op = op_fp16, class Ec = with_ec, class Backend = tensor_core>
struct policy {
    static constexpr int mode = Op::mode;
    static constexpr bool ec = Ec::ec;
    static constexpr bool tc = Backend::tc;
};

// ---------------------------------------------------------------------- tile
template <class Policy, int N>
struct tile {
    static constexpr int M = 128;                       // rows (TMEM lanes), one per thread
    static constexpr int THREADS = 128;
    static constexpr int MODE = Policy::mode;
    static constexpr bool EC = Policy::ec;
    static constexpr bool TC = Policy::tc;
    static constexpr int ESZ = MODE == 0 ? 2 : 4;       // operand bytes per element
    static constexpr int BK = 128 / ESZ;                // k per stage: one 128-byte K row
    static constexpr int EPC = 16 / ESZ;                // elements per 16-byte chunk
    static constexpr int KSTEP = MODE == 0 ? 16 : 8;    // UMMA K per instruction
    static constexpr int NSTEPS = BK / KSTEP;
    static constexpr uint32_t A_BYTES = M * 128;        // one part (hi or lo) of A
    static constexpr uint32_t B_BYTES = N * 128;
    static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr uint32_t TMEM_COLS = 4 * N;        // two buffers of D_hi | D_corr
    static constexpr uint32_t SMEM_BYTES = 1024 + 2 * STAGE_BYTES + 64;
    static_assert(N == 32 || N == 64 || N == 128, "N: 32, 64 or 128 (UMMA M = 128 needs N % 16 == 0; "
                                                  "4N TMEM columns must be a power of two <= 512)");
    static_assert(TC || N <= 64, "the simt backend keeps 3N accumulators per thread");
    static_assert(SMEM_BYTES <= 232448, "shared memory");

    // K-major SWIZZLE_128B operand layout (rows of 128 bytes = BK elements, 8-row
    // atoms of 1024 bytes, 16-byte chunk index XOR row % 8 -- what the UMMA
    // descriptor below decodes); row = m for A, n for B
    __device__ static uint32_t chunk_off(uint32_t row, uint32_t c)
    {
        return (row >> 3) * 1024u + (row & 7u) * 128u + ((c ^ (row & 7u)) << 4);
    }

    __device__ explicit tile(void* dyn_smem)
    {
        uint8_t* raw = static_cast<uint8_t*>(dyn_smem);
        op_ = raw + ((1024u - (ptx::smem_u32(raw) & 1023u)) & 1023u);
        bars_ = reinterpret_cast<uint64_t*>(op_ + 2 * STAGE_BYTES);
        if (threadIdx.x == 0) {
            ptx::mbar_init(&bars_[0], 1);   // MMAs of stage 0 done
            ptx::mbar_init(&bars_[1], 1);   // MMAs of stage 1 done
            ptx::mbar_init(&bars_[2], 1);   // k-block in accumulator buffer 0 done
            ptx::mbar_init(&bars_[3], 1);   // k-block in accumulator buffer 1 done
            ptx::fence_mbar_init();
        }
        uint32_t* slot = reinterpret_cast<uint32_t*>(bars_ + 4);
        if (TC && threadIdx.x < 32) ptx::tmem_alloc<TMEM_COLS>(slot);
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
        tmem_ = TC ? *slot : 0u;
#pragma unroll
        for (int j = 0; j < N; ++j) c_[j] = 0.0f;
    }

    // all MMAs drained, tensor memory freed (CTA-collective, last call)
    __device__ void release()
    {
        sync_acc();
        ptx::tc_fence_before();
        __syncthreads();
        ptx::tc_fence_after();
        if (TC && threadIdx.x < 32) ptx::tmem_dealloc<TMEM_COLS>(tmem_);
    }

    // ---------------------------------------------------------- operand staging
    // Register fragments of one stage (the FP32 values this thread splits): fetch_*
    // fills one from memory without touching shared memory, split_* splits it into
    // the current stage.  Fetching stage s+1 before mma() of stage s overlaps the
    // global-load latency with the barrier and the MMAs (tcec GEMM kernel).
    // B is staged in quads (4 consecutive k of one column = 16 bytes of FP32): quad
    // u = t + 128 q covers column u / (BK/4), k = 4 (u % (BK/4)) .. +3, so a warp
    // reads whole 128/256-byte column segments (coalesced) and stores 8/16-byte
    // pieces of the swizzled rows (conflict-free)
    static constexpr int QPC = BK / 4;                   // quads per column
    static constexpr int B_QUADS = N * QPC / THREADS;    // quads per thread
    struct a_frag { float x[8][EPC]; };                  // row t, k = 0..BK-1
    struct b_frag { float4 x[B_QUADS]; };

    // A(i, p) = A[i + p*lda] for i < rows, p < kvalid, else 0; A points at the
    // tile's first element (row m0, column k0).  Thread t holds row t.
    __device__ static void fetch_a(a_frag& f, const float* A, long long lda, int rows, int kvalid)
    {
        const int i = (int)threadIdx.x;
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int e = 0; e < EPC; ++e) {
                const int p = c * EPC + e;
                f.x[c][e] = (i < rows && p < kvalid) ? A[i + (long long)p * lda] : 0.0f;
            }
    }

    // B(p, j) = B[p + j*ldb] for p < kvalid, j < cols, else 0 (B at row k0, column n0);
    // one 16-byte load per quad when B and ldb keep quads 16-byte aligned
    __device__ static void fetch_b(b_frag& f, const float* B, long long ldb, int kvalid, int cols)
    {
        const bool vec = ((reinterpret_cast<uintptr_t>(B) | (uintptr_t)(ldb * 4)) & 15u) == 0;
#pragma unroll
        for (int q = 0; q < B_QUADS; ++q) {
            const int u = (int)threadIdx.x + THREADS * q, j = u / QPC, p = 4 * (u % QPC);
            const float* col = B + p + (long long)j * ldb;
            if (j < cols && vec && p + 4 <= kvalid) {
                f.x[q] = *reinterpret_cast<const float4*>(col);
            } else {
                const bool ok = j < cols;
                f.x[q] = make_float4(ok && p < kvalid ? col[0] : 0.0f, ok && p + 1 < kvalid ? col[1] : 0.0f,
                                     ok && p + 2 < kvalid ? col[2] : 0.0f, ok && p + 3 < kvalid ? col[3] : 0.0f);
            }
        }
    }

    __device__ void split_a(const a_frag& f)
    {
        acquire();
#pragma unroll
        for (int c = 0; c < 8; ++c) put_chunk(a_hi(), a_lo(), threadIdx.x, c, f.x[c]);
    }

    __device__ void split_b(const b_frag& f)
    {
        acquire();
#pragma unroll
        for (int q = 0; q < B_QUADS; ++q) {
            const int u = (int)threadIdx.x + THREADS * q;
            put_quad(b_hi(), b_lo(), (uint32_t)(u / QPC), (uint32_t)(4 * (u % QPC)), f.x[q]);
        }
    }

    __device__ void load_a(const float* A, long long lda, int rows, int kvalid)
    {
        a_frag f;
        fetch_a(f, A, lda, rows, kvalid);
        split_a(f);
    }

    __device__ void load_b(const float* B, long long ldb, int kvalid, int cols)
    {
        b_frag f;
        fetch_b(f, B, ldb, kvalid, cols);
        split_b(f);
    }

    // foreach_ij: A(i, p) = f(i, p) for the 128 x BK stage (tile-local
    // indices), computed and split in registers, never stored as FP32
    template <class F>
    __device__ void generate_a(F&& f)
    {
        a_frag g;
        const int i = (int)threadIdx.x;
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
            for (int e = 0; e < EPC; ++e) g.x[c][e] = f(i, c * EPC + e);
        split_a(g);
    }

    // B(p, j) = f(p, j) for the BK x N stage
    template <class F>
    __device__ void generate_b(F&& f)
    {
        b_frag g;
#pragma unroll
        for (int q = 0; q < B_QUADS; ++q) {
            const int u = (int)threadIdx.x + THREADS * q, j = u / QPC, p = 4 * (u % QPC);
            g.x[q] = make_float4(f(p, j), f(p + 1, j), f(p + 2, j), f(p + 3, j));
        }
        split_b(g);
    }

    // fill_fragment analog: every element of the stage's A (or B) operand = v;
    // ends with a CTA barrier so set_a / set_b may follow
    __device__ void fill_a(float v)
    {
        generate_a([&](int, int) { return v; });
        __syncthreads();
    }
    __device__ void fill_b(float v)
    {
        generate_b([&](int, int) { return v; });
        __syncthreads();
    }

    // map: the shared-memory location of element (i, p) of the A
    // operand (byte offset inside one part, plus the 16-bit / 32-bit slot), and
    // the single-element set built on it -- any thread, see the contract above
    __device__ static uint32_t map_a(int i, int p) { return chunk_off((uint32_t)i, (uint32_t)(p / EPC)) + (p % EPC) * ESZ; }
    __device__ static uint32_t map_b(int p, int j) { return chunk_off((uint32_t)j, (uint32_t)(p / EPC)) + (p % EPC) * ESZ; }
    __device__ void set_a(int i, int p, float v) { put_one(a_hi(), a_lo(), map_a(i, p), v); }
    __device__ void set_b(int p, int j, float v) { put_one(b_hi(), b_lo(), map_b(p, j), v); }

    // --------------------------------------------------------------- products
    // D_hi (+)= A_hi B_hi; D_corr (+)= A_lo B_hi + A_hi B_lo (Eq. corr-5) for the
    // current stage; the first mma() after a combine() restarts the accumulators
    __device__ void mma()
    {
        ptx::fence_proxy_async_smem();   // this thread's st.shared -> visible to the tensor core
        ptx::tc_fence_before();          // prior tcgen05.ld (combine) ordered before the barrier
        __syncthreads();
        uint8_t* base = op_ + stage_ * STAGE_BYTES;
        if (TC) {
            if (threadIdx.x == 0) {
                ptx::tc_fence_after();
                constexpr uint32_t idesc = ptx::instr_desc(MODE == 0 ? 0u : 2u, 0u, 0u, M, N);
                const uint32_t ah = ptx::smem_u32(base), al = ah + A_BYTES;
                const uint32_t bh = ah + 2 * A_BYTES, bl = bh + B_BYTES;
                const uint32_t d_hi = tmem_ + buf_ * 2 * N, d_corr = d_hi + N;
#pragma unroll
                for (int st = 0; st < NSTEPS; ++st) {
                    const uint32_t off = st * 32;   // KSTEP elements = 32 bytes along the swizzled row
                    const uint64_t dah = ptx::smem_desc(ah + off, 16, 1024, 2);
                    const uint64_t dbh = ptx::smem_desc(bh + off, 16, 1024, 2);
                    const uint32_t acc = (fresh_ && st == 0) ? 0u : 1u;
                    if (MODE == 0) ptx::mma_f16(d_hi, dah, dbh, idesc, acc);        // P1
                    else ptx::mma_tf32(d_hi, dah, dbh, idesc, acc);
                    if (EC) {
                        const uint64_t dal = ptx::smem_desc(al + off, 16, 1024, 2);
                        const uint64_t dbl = ptx::smem_desc(bl + off, 16, 1024, 2);
                        if (MODE == 0) {
                            ptx::mma_f16(d_corr, dal, dbh, idesc, acc);             // P2
                            ptx::mma_f16(d_corr, dah, dbl, idesc, 1u);              // P3
                        } else {
                            ptx::mma_tf32(d_corr, dal, dbh, idesc, acc);
                            ptx::mma_tf32(d_corr, dah, dbl, idesc, 1u);
                        }
                    }
                }
                ptx::tc_commit(&bars_[stage_]);   // stage free when these MMAs complete
            }
            outstanding_ |= 1u << stage_;
        } else {
            simt_mma(base);
        }
        stage_ ^= 1u;
        acquired_ = false;
        fresh_ = false;
        pending_ = true;
        drain();   // the previous k-block, while this one's MMAs run
    }

    // End of a k-block: C += RN(D_hi + D_corr * 2^-11) (TF32: scale 1), FP32 RN on
    // CUDA cores.  On the tensor cores the add is deferred: the block's
    // accumulators are committed and drained by the next mma() (after it has issued
    // the next block into the other buffer) or by sync_acc() / store() -- blocks are
    // still added in order, one at a time.
    __device__ void combine()
    {
        if (!pending_) return;
        constexpr float scale = MODE == 0 ? 1.0f / 2048.0f : 1.0f;
        if (TC) {
            drain();                                                 // at most one block in flight
            if (threadIdx.x == 0) ptx::tc_commit(&bars_[2 + buf_]);  // this block's MMAs
            drain_buf_ = buf_;
            drain_pending_ = true;
            buf_ ^= 1u;
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j)
                c_[j] = __fadd_rn(c_[j], EC ? __fmaf_rn(sco_[j], scale, shi_[j]) : shi_[j]);
        }
        fresh_ = true;
        pending_ = false;
    }

    // every k-block so far added into the FP32 accumulator (call before acc())
    __device__ void sync_acc()
    {
        combine();
        drain();
    }

  private:
    __device__ void drain()
    {
        if (!TC || !drain_pending_) return;
        constexpr float scale = MODE == 0 ? 1.0f / 2048.0f : 1.0f;
        {
            const uint32_t bit = 1u << drain_buf_;
            ptx::mbar_wait(&bars_[2 + drain_buf_], (acc_phase_ & bit) ? 1u : 0u);
            acc_phase_ ^= bit;
            ptx::tc_fence_after();
            const uint32_t lane0 = (threadIdx.x & ~31u) << 16;  // warp w reads TMEM lanes 32w..32w+31
            const uint32_t d = tmem_ + lane0 + drain_buf_ * 2 * N;
#pragma unroll
            for (int j0 = 0; j0 < N; j0 += 16) {
                float h[16], q[16];
                ptx::tmem_ld16(d + j0, h);
                if (EC) ptx::tmem_ld16(d + N + j0, q);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; e += 2) {
                    if (EC) combine2(c_[j0 + e], c_[j0 + e + 1], h[e], h[e + 1], q[e], q[e + 1], scale);
                    else { c_[j0 + e] = __fadd_rn(c_[j0 + e], h[e]); c_[j0 + e + 1] = __fadd_rn(c_[j0 + e + 1], h[e + 1]); }
                }
            }
            ptx::tc_fence_before();
        }
        drain_pending_ = false;
    }

  public:
    // ------------------------------------------------------------- accumulator
    // C(threadIdx.x, j); complete only after sync_acc() (k-blocks drain lazily)
    __device__ float& acc(int j) { return c_[j]; }
    __device__ static int acc_row() { return (int)threadIdx.x; }
    __device__ void fill_acc(float v)
    {
#pragma unroll
        for (int j = 0; j < N; ++j) c_[j] = v;
    }

    // C(i, j) = RN(alpha*acc + RN(beta*C(i, j))) for i < rows, j < cols (C at
    // row m0, column n0; beta == 0 never reads C).  Coalesced along each column.
    __device__ void store(float* C, long long ldc, float alpha, float beta, int rows, int cols)
    {
        sync_acc();
        const int i = (int)threadIdx.x;
        if (i >= rows) return;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            if (j < cols) {
                float* p = C + i + (long long)j * ldc;
                *p = beta == 0.0f ? __fmul_rn(alpha, c_[j]) : __fmaf_rn(alpha, c_[j], __fmul_rn(beta, *p));
            }
        }
    }

  private:
    __device__ uint8_t* a_hi() const { return op_ + stage_ * STAGE_BYTES; }
    __device__ uint8_t* a_lo() const { return a_hi() + A_BYTES; }
    __device__ uint8_t* b_hi() const { return a_hi() + 2 * A_BYTES; }
    __device__ uint8_t* b_lo() const { return b_hi() + B_BYTES; }

    // wait until the MMAs that last read the current stage have completed
    __device__ void acquire()
    {
        if (acquired_) return;
        const uint32_t bit = 1u << stage_;
        if (outstanding_ & bit) {
            ptx::mbar_wait(&bars_[stage_], (mma_phase_ >> stage_) & 1u);
            mma_phase_ ^= bit;
            outstanding_ &= ~bit;
        }
        acquired_ = true;
    }

    // split EPC consecutive-k values of one operand row into its hi / lo chunk
    __device__ static void put_chunk(uint8_t* hi, uint8_t* lo, uint32_t row, uint32_t c, const float (&x)[EPC])
    {
        const uint32_t off = chunk_off(row, c);
        uint4 h, l;
        if constexpr (MODE == 0) {
            split_fp16x2x2(x[0], x[1], x[2], x[3], h.x, h.y, l.x, l.y);
            split_fp16x2x2(x[4], x[5], x[6], x[7], h.z, h.w, l.z, l.w);
        } else {
            split_tf32(x[0], h.x, l.x);
            split_tf32(x[1], h.y, l.y);
            split_tf32(x[2], h.z, l.z);
            split_tf32(x[3], h.w, l.w);
        }
        *reinterpret_cast<uint4*>(hi + off) = h;
        if (EC) *reinterpret_cast<uint4*>(lo + off) = l;
    }

    // split 4 consecutive-k values (k4 .. k4+3) of one operand row: 8-byte (FP16)
    // or 16-byte (TF32) pieces of its hi / lo chunk
    __device__ static void put_quad(uint8_t* hi, uint8_t* lo, uint32_t row, uint32_t k4, const float4 v)
    {
        const uint32_t off = chunk_off(row, k4 / EPC) + (k4 % EPC) * ESZ;
        if constexpr (MODE == 0) {
            uint2 h, l;
            split_fp16x2x2(v.x, v.y, v.z, v.w, h.x, h.y, l.x, l.y);
            *reinterpret_cast<uint2*>(hi + off) = h;
            if (EC) *reinterpret_cast<uint2*>(lo + off) = l;
        } else {
            uint4 h, l;
            split_tf32(v.x, h.x, l.x);
            split_tf32(v.y, h.y, l.y);
            split_tf32(v.z, h.z, l.z);
            split_tf32(v.w, h.w, l.w);
            *reinterpret_cast<uint4*>(hi + off) = h;
            if (EC) *reinterpret_cast<uint4*>(lo + off) = l;
        }
    }

    __device__ static void put_one(uint8_t* hi, uint8_t* lo, uint32_t off, float v)
    {
        if constexpr (MODE == 0) {
            uint32_t h, l;
            split_fp16x2(v, 0.0f, h, l);
            *reinterpret_cast<uint16_t*>(hi + off) = (uint16_t)(h & 0xffffu);
            *reinterpret_cast<uint16_t*>(lo + off) = (uint16_t)(l & 0xffffu);
        } else {
            uint32_t h, l;
            split_tf32(v, h, l);
            *reinterpret_cast<uint32_t*>(hi + off) = h;
            *reinterpret_cast<uint32_t*>(lo + off) = l;
        }
    }

    __device__ static float part(const uint8_t* buf, uint32_t off)
    {
        if constexpr (MODE == 0) {
            const uint16_t b = *reinterpret_cast<const uint16_t*>(buf + off);
            float x0, x1;
            f16x2_to_f32x2((uint32_t)b, x0, x1);
            return x0;
        }
        return __uint_as_float(*reinterpret_cast<const uint32_t*>(buf + off));
    }

    // simt backend: the three products of Eq. corr-5 from the same split tiles,
    // FP32 FMA (each product exact: <= 11 x 11 significant bits), k ascending
    __device__ void simt_mma(const uint8_t* base)
    {
        const uint8_t* ah = base;
        const uint8_t* al = base + A_BYTES;
        const uint8_t* bh = base + 2 * A_BYTES;
        const uint8_t* bl = bh + B_BYTES;
        if (fresh_) {
#pragma unroll
            for (int j = 0; j < N; ++j) { shi_[j] = 0.0f; sco_[j] = 0.0f; }
        }
        const int i = (int)threadIdx.x;
#pragma unroll 1
        for (int p = 0; p < BK; ++p) {
            const float xh = part(ah, map_a(i, p));
            const float xl = part(al, map_a(i, p));
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const float yh = part(bh, map_b(p, j));
                shi_[j] = __fmaf_rn(xh, yh, shi_[j]);
                if (EC) {
                    sco_[j] = __fmaf_rn(xl, yh, sco_[j]);
                    sco_[j] = __fmaf_rn(xh, part(bl, map_b(p, j)), sco_[j]);
                }
            }
        }
    }

    uint8_t* op_;
    uint64_t* bars_;
    uint32_t tmem_;
    uint32_t stage_ = 0, outstanding_ = 0, mma_phase_ = 0, acc_phase_ = 0, buf_ = 0, drain_buf_ = 0;
    bool acquired_ = false, fresh_ = true, pending_ = false, drain_pending_ = false;
    float c_[N];
    float shi_[TC ? 1 : N], sco_[TC ? 1 : N];
};

}  // namespace tcec
}  // namespace emu
