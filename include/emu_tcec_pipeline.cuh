/*
 * emu_tcec_pipeline.cuh -- the PIPELINED (warp-specialized) form of the
 * device-level API: the library's own batched-SGEMM kernel with operand and
 * epilogue hooks (§4.4, P:496-523:
 * WMMAe-TCEC is an API that user kernels are built on, and the paper's
 * 54.2 TFlop/s batched SGEMM is one such user).
 *
 * include/emu_tcec.cuh's emu::tcec::tile is the synchronous form: one
 * 128-thread CTA that loads, splits, multiplies and combines in program order
 * -- the shape of the paper's WMMA-style API, convenient for custom fused
 * kernels, but with no overlap between the roles.  This header is the
 * throughput form: a persistent CTA pair (cta_group::2, M = 256) whose warps
 * specialise --
 *
 *   producer   TMA loads of the FP32 operand tiles into a shared-memory ring
 *              (skipped for a generated operand);
 *   splitters  8 warps: each FP32 value -> hi/lo (Eqs. corr-1..4, P:481-488;
 *              R#6 for TF32) in registers, A straight into tensor memory
 *              (tcgen05.st), B into the K-major operand ring -- or the value
 *              of a generated operand, evaluated right there;
 *   MMA        one thread: P2 + P3 -> D_corr, then P1 -> D_hi per k-block
 *              (Eq. corr-5; tcgen05.mma.cta_group::2, A from TMEM);
 *   combine    16 warps: t = RN(D_hi + D_corr 2^-11), C += t in FP32 RN on
 *              CUDA cores (R#7/R#8), then the store (or the user's);
 *
 * i.e. emu::emu_sgemm_pair_ts_kernel (paper_2308_15152_b200/csrc/
 * gemm_pair_ts_sm100.cuh; design in DESIGN.md §6).  Its last template
 * argument is the hook type `Ops`:
 *
 *   struct my_operands {
 *       static constexpr bool gen_a = ..., gen_b = ..., custom_store = ...;
 *       // gen_a: the A operand is the rule a(batch, i, p) = A_b(i, p), evaluated by
 *       //        the splitter warps for i < m, p < k (0 is used outside); no memory
 *       //        read of A happens (foreach_ij)
 *       __device__ float a(int batch, int i, int p) const;
 *       // gen_b: likewise B_b(p, j) for p < k, j < n
 *       __device__ float b(int batch, int p, int j) const;
 *       // custom_store: receives the finished FP32 accumulator of row i, columns
 *       //        j0 .. j0 + cols - 1 (alpha / beta are then the hook's business)
 *       __device__ void store(int batch, int i, int j0, const float* c, int cols) const;
 *       // ... any kernel-parameter data the rules need (pointers, sizes)
 *   };
 *
 * The hooks do not change the method: every operand value, generated or
 * loaded, goes through the same split, the same three products and the same
 * combine, so a generated operand gives the bits the explicit operand would.
 * The object is passed by value as a kernel parameter (param space; keep it
 * small and trivially copyable).
 *
 * Users in this repository (C ABI, include/emu_sgemm.h, flag EMU_FLAG_PIPELINED):
 *   emu_tcec_gemm_batched        Ops = operands_from_memory (the defaults): the
 *                                library's kernel itself -- the c2 workload through
 *                                the API runs at the library's speed
 *   emu_tcec_householder_batched Ops = householder_operands (csrc/tcec_api.cuh): the
 *                                reflector H = I - 2 v v^T generated from v by the
 *                                splitter warps (R#23), H never in memory
 * Host launch: run_pipelined<MODE, Ops>() in csrc/api.cu selects the tile shape
 * exactly like the library's entries (A-stationary, long-k rings, 64-wide tiles)
 * and builds the tensor maps of the non-generated operands.
 */
#pragma once

#include "gemm_pair_ts_sm100.cuh"

namespace emu {
namespace tcec {

// the defaults: both FP32 operands from global memory (TMA), the library's store
using operands_from_memory = emu::lib_operands;

}  // namespace tcec
}  // namespace emu
