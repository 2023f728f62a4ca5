/*
 * emu_sgemm.h -- C ABI of the B200 (sm_100a) emulated SGEMM library
 * (libemusgemm.so), the hot path of arXiv 2308.15152 (Ootomo & Yokota,
 * "Reducing shared memory footprint to leverage high throughput on Tensor
 * Cores and its flexible API extension library", §4.4 "WMMAe-TCEC").
 *
 * What is computed (citations: P:n = /root/reference/PAPER.md line n;
 * R#n = reading n in DESIGN.md §3):
 *   The paper computes C_F32 = A_F32 B_F32 as
 *     A_F16  = toFP16(A_F32)                                   Eq. corr-1
 *     dA_F16 = toFP16((A_F32 - toFP32(A_F16)) * 2^11)          Eq. corr-2
 *     (same for B)                                             Eqs. corr-3/4
 *     C = A_F16 B_F16 + (dA_F16 B_F16 + A_F16 dB_F16) / 2^11   Eq. corr-5
 *   with the accumulation moved outside the Tensor Core's RZ rounding:
 *   the main product and the two correction products are accumulated in two
 *   separate tensor-core accumulators over one k-block of KB elements, then
 *   combined in FP32 round-to-nearest on CUDA cores, t = RN(D_hi + D_corr*2^-11),
 *   C_acc = RN(C_acc + t), block after block (R#7, R#8).  EMU_SPLIT_TF32 is the
 *   TF32 hi/lo variant of north_star (R#6: hi = RNE_tf32(x), lo = RNE_tf32(x-hi),
 *   scale 1).  Finally C = RN(alpha*C_acc + RN(beta*C)) (BLAS, R#17); beta == 0
 *   never reads C (R#19).  The batched form runs `batch` independent problems
 *   (P:552): X_b = X + b*strideX for X in {A, B, C}.
 *
 * Conventions: column-major throughout, no transposes (A(i,p) = A[i + p*lda],
 * m x k; B(p,j) = B[p + j*ldb], k x n; C(i,j) = C[i + j*ldc], m x n).  All
 * pointers are DEVICE pointers owned by the caller (except the _host entry),
 * all sizes are elements.  `stream` is a cudaStream_t (NULL = legacy default
 * stream); every call is asynchronous on it unless stated.  Results are
 * deterministic: identical inputs and configuration give bit-identical C
 * (no split-K, no atomics on C).
 *
 * Errors: arguments are validated synchronously before anything is launched;
 * on any non-SUCCESS return C is untouched.  Faults during kernel execution
 * surface as CUDA errors at the caller's next synchronisation.
 *
 * Memory: the device entries allocate no global memory (tensor memory is
 * allocated and freed inside each CTA; the range-safe entry uses a caller-owned
 * workspace); per-device attributes are cached.
 * Thread-safe.  sm_100a only (B200); other devices -> EMU_STATUS_ARCH_MISMATCH.
 */
#ifndef EMU_SGEMM_H_
#define EMU_SGEMM_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EMU_SPLIT_FP16 = 0, /* FP16 hi + 2^11-scaled FP16 lo, kind::f16 MMAs */
    EMU_SPLIT_TF32 = 1  /* TF32 hi + TF32 lo, kind::tf32 MMAs (north_star, R#6)    */
} emu_split_mode;

typedef enum {
    EMU_STATUS_SUCCESS = 0,
    EMU_STATUS_INVALID_VALUE = 1,  /* a size, leading dimension, stride, pointer or mode is invalid */
    EMU_STATUS_NOT_SUPPORTED = 2,  /* valid BLAS call outside this version's domain (see below)     */
    EMU_STATUS_ARCH_MISMATCH = 3,  /* current device is not sm_100                                  */
    EMU_STATUS_LAUNCH_FAILED = 4,  /* kernel launch returned an error                               */
    EMU_STATUS_CUDA_ERROR = 5      /* another CUDA runtime/driver call failed                       */
} emu_status;

/* Flags for emu_sgemm_batched_ex. */
#define EMU_FLAG_NO_CORRECTION 1u  /* policy "error correction off": drop both
                                      correction products; a negative control only */
#define EMU_FLAG_SIMT 2u           /* emu_tcec_* only: the device API's "simt" backend,
                                      the same three products on CUDA cores, for evaluation */
#define EMU_FLAG_PIPELINED 4u      /* emu_tcec_gemm_batched / emu_tcec_householder_batched only: the
                                      pipelined (warp-specialized) form of the device API
                                      (include/emu_tcec_pipeline.cuh) instead of the synchronous
                                      tile -- the library's kernel with the caller's operand hooks.
                                      Tensor-core backend only (with EMU_FLAG_SIMT ->
                                      EMU_STATUS_NOT_SUPPORTED); FP32 operands read from memory must
                                      be in the TMA domain (16-byte aligned, ld and stride multiples
                                      of 4) else EMU_STATUS_NOT_SUPPORTED.  Same results as
                                      emu_sgemm_batched_ex with the same kblock, bit for bit. */

/*
 * emu_sgemm_batched -- C_b = alpha * A_b B_b + beta * C_b for b in [0, batch).
 *   m, n, k, batch >= 0; lda >= max(1, m); ldb >= max(1, k); ldc >= max(1, m).
 *   strideA / strideB may be 0 (one operand shared by every problem); strideC
 *   must make the outputs disjoint when batch > 1 (|strideC| >= ldc*n).
 *   A and B may be NULL only when they are not read (k == 0 or alpha == 0);
 *   C may be NULL only when m == 0, n == 0 or batch == 0.  C must not
 *   overlap A or B.
 *   Quick returns: m == 0 || n == 0 || batch == 0 -> SUCCESS, nothing
 *   launched; k == 0 || alpha == 0 -> C = RN(beta*C) (beta == 0 writes +0).
 *   Any alignment and leading dimension is accepted.  When A and B are
 *   16-byte aligned and lda, ldb, strideA, strideB are multiples of 4
 *   elements, FP32 tiles are staged by TMA (tensor-map strides are 16-byte
 *   units); otherwise the splitter warps load them directly (slower path,
 *   identical results).
 *   FP16 mode: |A|, |B| < 65520 and finite, else those outputs are
 *   non-finite (R#4); pass d_range_flag to emu_sgemm_batched_ex to detect it.
 */
emu_status emu_sgemm_batched(int m, int n, int k, float alpha,
                             const float* A, int lda, long long strideA,
                             const float* B, int ldb, long long strideB,
                             float beta, float* C, int ldc, long long strideC,
                             int batch, emu_split_mode mode, void* stream);

/* emu_sgemm -- the single-problem form (batch = 1). */
emu_status emu_sgemm(int m, int n, int k, float alpha,
                     const float* A, int lda, const float* B, int ldb,
                     float beta, float* C, int ldc, emu_split_mode mode, void* stream);

/*
 * emu_sgemm_batched_ex -- emu_sgemm_batched plus:
 *   d_range_flag: NULL, or a device unsigned int that the kernel ORs with 1
 *     (sticky, never cleared) when an FP16-mode operand element has
 *     |x| >= 65520 or is not finite (its hi part is +-Inf/NaN, R#4);
 *   kblock: the combine interval KB in k (R#7; 0 = the default: 64 for
 *     k <= 8192, doubled for every further factor 4 of k -- 128 for k <= 32768,
 *     256 for k <= 131072, ...; otherwise a positive multiple of 32, at most 4096);
 *   flags: EMU_FLAG_* bits (0 = the paper's method).
 */
emu_status emu_sgemm_batched_ex(int m, int n, int k, float alpha,
                                const float* A, int lda, long long strideA,
                                const float* B, int ldb, long long strideB,
                                float beta, float* C, int ldc, long long strideC,
                                int batch, emu_split_mode mode, void* stream,
                                unsigned int* d_range_flag, int kblock, unsigned int flags);

/*
 * emu_sgemm_batched_t -- C_b = alpha * op(A_b) op(B_b) + beta * C_b with BLAS
 * transpose arguments (the paper's problem is C = A B):
 *   transa 'N'/'n': op(A) = A, stored m x k (lda >= max(1, m));
 *          'T'/'t' (or 'C'/'c', real data): op(A) = A^T, A stored k x m (lda >= max(1, k));
 *   transb 'N': op(B) = B, stored k x n (ldb >= max(1, k));
 *          'T': op(B) = B^T, B stored n x k (ldb >= max(1, n)).
 * The method, the other arguments and the errors are those of emu_sgemm_batched_ex;
 * an invalid trans character -> EMU_STATUS_INVALID_VALUE.  Transposed operands are
 * read by TMA only: a transposed operand outside the TMA domain (base not 16-byte
 * aligned, ld or stride not a multiple of 4) -> EMU_STATUS_NOT_SUPPORTED.
 * ('N', 'N') is exactly emu_sgemm_batched_ex.
 */
emu_status emu_sgemm_batched_t(char transa, char transb, int m, int n, int k, float alpha,
                               const float* A, int lda, long long strideA,
                               const float* B, int ldb, long long strideB,
                               float beta, float* C, int ldc, long long strideC,
                               int batch, emu_split_mode mode, void* stream,
                               unsigned int* d_range_flag, int kblock, unsigned int flags);

/*
 * emu_sgemm_batched_layout -- emu_sgemm_batched_t with a storage order (NEXT row 2,
 * "row-major at the C ABI"; cblas_sgemm's Order argument):
 *   EMU_COL_MAJOR: exactly emu_sgemm_batched_t.
 *   EMU_ROW_MAJOR: every matrix is row-major: X(i, j) = X[i*ldX + j]; op(A) is m x k,
 *     op(B) k x n, C m x n with ldc >= max(1, n); 'N' A needs lda >= max(1, k), 'T' A
 *     (stored k x m) lda >= max(1, m); 'N' B ldb >= max(1, n), 'T' B (stored n x k)
 *     ldb >= max(1, k).  Computed as the column-major C^T = op(B)^T op(A)^T (same
 *     arithmetic per element; no data is moved).
 * Another layout value -> EMU_STATUS_INVALID_VALUE; other errors as emu_sgemm_batched_t.
 */
typedef enum { EMU_COL_MAJOR = 0, EMU_ROW_MAJOR = 1 } emu_layout;
emu_status emu_sgemm_batched_layout(emu_layout layout, char transa, char transb, int m, int n, int k,
                                    float alpha, const float* A, int lda, long long strideA,
                                    const float* B, int ldb, long long strideB,
                                    float beta, float* C, int ldc, long long strideC,
                                    int batch, emu_split_mode mode, void* stream,
                                    unsigned int* d_range_flag, int kblock, unsigned int flags);

/*
 * Range-safe mode (DESIGN R#22).  The paper splits raw
 * values, so FP16 mode overflows for |x| >= 65520 (R#4).  This
 * entry first scales row i of A_b by 2^-e_i and column j of B_b by 2^-f_j,
 *   e = clamp(ilogb(max finite |x| over the row / column) - 14, -125, 125)
 *   (0 when the row / column has no finite non-zero element),
 * so every scaled row / column peaks in [2^14, 2^15); runs the unchanged
 * method (split, three products, per-k-block combine) on the scaled operands;
 * and un-scales the combined accumulator: C = RN(alpha*RN(C'*2^(e_i+f_j)) +
 * RN(beta*C)).  Power-of-two scaling is exact except where a scaled value is
 * subnormal or overflows.  The exponents come from one max-|x| pass over A
 * and B (a second kernel, recorded by emu_last_launch_count).
 *
 * emu_range_workspace_size: bytes of device workspace the call needs,
 *   4 * batch * (m + n) (returns 0 for negative arguments).
 * emu_sgemm_batched_range: arguments as emu_sgemm_batched_ex, plus
 *   d_workspace / workspace_bytes: caller-owned device memory, 16-byte aligned,
 *     >= emu_range_workspace_size(m, n, batch); not aliased with A, B, C; it may
 *     be reused once the call's work on `stream` has completed.
 *   Errors: as emu_sgemm_batched_ex; workspace NULL, misaligned or too small ->
 *   EMU_STATUS_INVALID_VALUE; operands outside the TMA domain (base not 16-byte
 *   aligned, lda/ldb/strides not multiples of 4) -> EMU_STATUS_NOT_SUPPORTED.
 */
size_t emu_range_workspace_size(int m, int n, int batch);
emu_status emu_sgemm_batched_range(int m, int n, int k, float alpha,
                                   const float* A, int lda, long long strideA,
                                   const float* B, int ldb, long long strideB,
                                   float beta, float* C, int ldc, long long strideC,
                                   int batch, emu_split_mode mode, void* stream,
                                   void* d_workspace, size_t workspace_bytes,
                                   unsigned int* d_range_flag, int kblock, unsigned int flags);

/*
 * emu_sgemm_batched_host -- the same operation on HOST buffers (pinned or
 * pageable, column-major as above, C read only if beta != 0): stages the
 * operands into a per-device device workspace the library keeps (grow-only),
 * runs the device path, copies C back and synchronises `stream` before
 * returning.  Batches of >= 16 problems are processed in 8 chunks on two
 * internal streams so the copies of one chunk overlap the kernel of the next
 * (work is ordered after prior work on `stream`).  Calls are serialised per
 * device.  Same errors; allocation failure -> EMU_STATUS_CUDA_ERROR.
 */
emu_status emu_sgemm_batched_host(int m, int n, int k, float alpha,
                                  const float* A, int lda, long long strideA,
                                  const float* B, int ldb, long long strideB,
                                  float beta, float* C, int ldc, long long strideC,
                                  int batch, emu_split_mode mode, void* stream);

/*
 * emu_split -- the split of Eqs. corr-1..corr-4 (FP16: P:481-488) or R#6
 * (TF32), elementwise over `count` contiguous device floats, with the SAME
 * device code the GEMM kernels use for operand staging.  FP16: hi and lo are
 * device arrays of `count` uint16 binary16 bit patterns.  TF32: hi and lo are
 * device arrays of `count` float (binary32 patterns with the low 13 bits 0).
 * count >= 0; x, hi, lo non-NULL when count > 0 and 4-byte aligned.
 */
emu_status emu_split(const float* x, long long count, emu_split_mode mode,
                     void* hi, void* lo, void* stream);

/*
 * emu_sgemm_multicast -- one GEMM C = alpha A B (beta = 0: C is never read) whose
 * result is stored to num_dst (1..8) destinations C_dst[0..num_dst-1], each m x n
 * with leading dimension ldc.  C_dst is a HOST array of
 * device pointers; a pointer may be a peer GPU's memory mapped into this process
 * (CUDA IPC / symmetric memory over NVLink): then the kernel's epilogue writes
 * every finished tile to every peer while later tiles are still computing -- the
 * all-gather of an n-sharded GEMM fused into the GEMM (rank r passes its column
 * block B_r and C_dst[q] = C_q + n0_r*ldc).  Same method and arithmetic as
 * emu_sgemm (bit-identical per element).  Requires the TMA domain (A, B 16-byte
 * aligned, lda, ldb multiples of 4) else EMU_STATUS_NOT_SUPPORTED; num_dst out of
 * range or a NULL destination -> EMU_STATUS_INVALID_VALUE; other errors as
 * emu_sgemm_batched_ex.  Destinations must not overlap each other, A or B.
 */
emu_status emu_sgemm_multicast(int m, int n, int k, float alpha,
                               const float* A, int lda, const float* B, int ldb,
                               float* const* C_dst, int num_dst, int ldc,
                               emu_split_mode mode, void* stream, int kblock, unsigned int flags);

/*
 * Device-level API users (include/emu_tcec.cuh).  Each
 * entry is ONE kernel written against the in-kernel tile API emu::tcec::tile
 * (the B200 analog of WMMAe-TCEC): 128 x 64 output blocks per
 * 128-thread CTA (128 x 32 with EMU_FLAG_SIMT), k in stages of 64 (FP16) / 32
 * (TF32) split on load, three tcgen05 products per stage, combine every 64 k.
 * flags: EMU_FLAG_NO_CORRECTION (policy without_ec, P1 only) and/or
 * EMU_FLAG_SIMT (policy simt: the products on CUDA cores).  Column-major,
 * device pointers owned by the caller, asynchronous on `stream`; any alignment.
 * Errors as emu_sgemm_batched; unknown flag bits -> EMU_STATUS_INVALID_VALUE;
 * more than 65535 column blocks -> EMU_STATUS_NOT_SUPPORTED.
 *
 * emu_tcec_gemm_batched: C_b = alpha A_b B_b + beta C_b, arguments as
 *   emu_sgemm_batched_ex (kblock: combine interval, 0 = 64, else a multiple of
 *   the stage k (64 FP16 / 32 TF32), at most 4096).  The paper's "Code 1 with the
 *   namespace swapped".
 * emu_tcec_householder_batched: C_b = H_b X_b, H_b = I_m - 2 v_b v_b^T
 *   (Eq. householder, read as v v^T for a unit column v, R#23),
 *   H(i, p) = RN(RN(RN(v_i v_p) * -2) + [i == p]) generated inside the kernel by
 *   the foreach_ij analog (Code 4); H is never stored.  v_b =
 *   V + b*strideV (m floats); X_b m x n (ldx >= m); C_b m x n (ldc >= m).
 * emu_tcec_givens_batched: C_b = G(i, j, theta_b) X_b (R#24): G = I_m
 *   except G(i,i) = G(j,j) = c_b, G(i,j) = -s_b, G(j,i) = s_b with (c_b, s_b) =
 *   (CS[2b], CS[2b+1]); built with the map analog.  0 <= i, j < m,
 *   i != j, else EMU_STATUS_INVALID_VALUE.
 * emu_tcec_scan: inclusive prefix sums of `count` arrays of n floats, array c at
 *   X + c*ldx, result at Y + c*ldy: y = L x, L(i, p) = [p <= i] (the transpose of
 *   the paper's U, Eqs. scan-mat / u-rule, R#25), L generated by rule.
 */
emu_status emu_tcec_gemm_batched(int m, int n, int k, float alpha,
                                 const float* A, int lda, long long strideA,
                                 const float* B, int ldb, long long strideB,
                                 float beta, float* C, int ldc, long long strideC,
                                 int batch, emu_split_mode mode, void* stream,
                                 int kblock, unsigned int flags);
emu_status emu_tcec_householder_batched(int m, int n, const float* V, long long strideV,
                                        const float* X, int ldx, long long strideX,
                                        float* C, int ldc, long long strideC,
                                        int batch, emu_split_mode mode, void* stream,
                                        unsigned int flags);
emu_status emu_tcec_givens_batched(int m, int n, int i, int j, const float* CS,
                                   const float* X, int ldx, long long strideX,
                                   float* C, int ldc, long long strideC,
                                   int batch, emu_split_mode mode, void* stream,
                                   unsigned int flags);
emu_status emu_tcec_scan(int n, int count, const float* X, int ldx, float* Y, int ldy,
                         emu_split_mode mode, void* stream, unsigned int flags);

/* Number of kernel launches the last successful call on this host thread
 * issued (0 for a quick return without a scale kernel); for launch accounting. */
int emu_last_launch_count(void);

/* Name of the GEMM kernel (and its template configuration) the last call on
 * this host thread dispatched; "" before any launch.  Never NULL; the string
 * is owned by the library and stays valid.  For reports (bench.py) and
 * diagnostics; the dispatch itself is described in DESIGN.md §6. */
const char* emu_last_kernel_name(void);

/* Human-readable status. Never NULL. */
const char* emu_status_string(emu_status status);

/* Library version: major*10000 + minor*100 + patch. */
int emu_version(void);

#ifdef __cplusplus
}
#endif

#endif /* EMU_SGEMM_H_ */
