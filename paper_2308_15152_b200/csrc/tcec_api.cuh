// tcec_api.cuh -- C-ABI entries built on the device-level API (include/emu_tcec.cuh):
// the "custom kernels" of the paper's WMMAe-TCEC and its
// structured-operand benchmarks (foreach_ij: Householder and scan, map: Givens;
// P:311-470).  Included at the end of api.cu (shares its device checks and
// launch accounting).  Every kernel here is a plain user of emu::tcec::tile.
#pragma once

#include "emu_tcec.cuh"
#include "emu_tcec_pipeline.cuh"

namespace emu {
namespace tcec_kernels {

using namespace emu::tcec;

struct GemmArgs {
    int m, n, k, batch;
    float alpha, beta;
    const float* A; long long lda, strideA;
    const float* B; long long ldb, strideB;
    float* C; long long ldc, strideC;
    int kb_stages;   // combine every kb_stages stages (KB / BK)
};

// the generic batched GEMM written against the tile API: the paper's Code 1 with
// the namespace swapped, one 128 x N block per CTA
template <class Pol, int N>
__global__ void __launch_bounds__(128) tcec_gemm_kernel(const GemmArgs a)
{
    extern __shared__ uint8_t smem[];
    using T = tile<Pol, N>;
    T t(smem);
    const int m0 = blockIdx.x * T::M, n0 = blockIdx.y * N;
    const int rows = min(T::M, a.m - m0), cols = min(N, a.n - n0);
    for (int b = blockIdx.z; b < a.batch; b += gridDim.z) {
        const float* A = a.A + b * a.strideA + m0;
        const float* B = a.B + b * a.strideB + (long long)n0 * a.ldb;
        if constexpr (!Pol::tc) {   // simt: registers go to the 3N accumulators, no lookahead
            int s = 0;
            for (int k0 = 0; k0 < a.k; k0 += T::BK) {
                const int kv = min(T::BK, a.k - k0);
                t.load_a(A + (long long)k0 * a.lda, a.lda, rows, kv);
                t.load_b(B + k0, a.ldb, kv, cols);
                t.mma();
                if (++s == a.kb_stages) { t.combine(); s = 0; }
            }
            t.store(a.C + b * a.strideC + m0 + (long long)n0 * a.ldc, a.ldc, a.alpha, a.beta, rows, cols);
            t.fill_acc(0.0f);
            continue;
        }
        // software-pipelined: the FP32 values of stage k0 + BK are in flight while
        // stage k0 is split and its MMAs issued
        typename T::a_frag fa;
        typename T::b_frag fb;
        T::fetch_a(fa, A, a.lda, rows, min(T::BK, a.k));
        T::fetch_b(fb, B, a.ldb, min(T::BK, a.k), cols);
        int s = 0;
        for (int k0 = 0; k0 < a.k; k0 += T::BK) {
            t.split_a(fa);
            t.split_b(fb);
            const int k1 = k0 + T::BK;
            if (k1 < a.k) {
                T::fetch_a(fa, A + (long long)k1 * a.lda, a.lda, rows, min(T::BK, a.k - k1));
                T::fetch_b(fb, B + k1, a.ldb, min(T::BK, a.k - k1), cols);
            }
            t.mma();
            if (++s == a.kb_stages) { t.combine(); s = 0; }
        }
        t.store(a.C + b * a.strideC + m0 + (long long)n0 * a.ldc, a.ldc, a.alpha, a.beta, rows, cols);
        t.fill_acc(0.0f);
    }
    t.release();
}

// Householder (Eq. householder, R#23): C_b = H_b X_b, H = I_m - 2 v v^T
// generated element by element from v (Code 4) straight into the split
// operand -- H never exists in memory:
//   H(i, p) = RN(RN(RN(v_i * v_p) * -2) + [i == p])
struct HouseArgs {
    int m, n, batch, kb_stages;
    const float* V; long long strideV;
    const float* X; long long ldx, strideX;
    float* C; long long ldc, strideC;
};

__device__ __forceinline__ float householder_elem(float vi, float vp, bool diag)
{
    const float e = __fmul_rn(__fmul_rn(vi, vp), -2.0f);
    return diag ? __fadd_rn(e, 1.0f) : e;
}

// the same operand for the pipelined form (include/emu_tcec_pipeline.cuh): the
// library's warp-specialized kernel evaluates H(i, p) in its splitter warps
struct householder_operands {
    static constexpr bool gen_a = true, gen_b = false, custom_store = false;
    const float* V;
    long long strideV;
    __device__ float a(int b, int i, int p) const
    {
        const float* v = V + b * strideV;
        return householder_elem(__ldg(v + i), __ldg(v + p), i == p);
    }
    __device__ float b(int, int, int) const { return 0.0f; }
    __device__ void store(int, int, int, const float*, int) const {}
};

template <class Pol, int N>
__global__ void __launch_bounds__(128) tcec_householder_kernel(const HouseArgs a)
{
    extern __shared__ uint8_t smem[];
    using T = tile<Pol, N>;
    T t(smem);
    const int m0 = blockIdx.x * T::M, n0 = blockIdx.y * N;
    const int rows = min(T::M, a.m - m0), cols = min(N, a.n - n0);
    for (int b = blockIdx.z; b < a.batch; b += gridDim.z) {
        const float* v = a.V + b * a.strideV;
        const float* X = a.X + b * a.strideX + (long long)n0 * a.ldx;
        const float vi = (int)threadIdx.x < rows ? v[m0 + threadIdx.x] : 0.0f;
        int s = 0;
        for (int k0 = 0; k0 < a.m; k0 += T::BK) {
            const int kv = min(T::BK, a.m - k0);
            t.generate_a([&](int i, int p) {
                return (i < rows && p < kv) ? householder_elem(vi, v[k0 + p], m0 + i == k0 + p) : 0.0f;
            });
            t.load_b(X + k0, a.ldx, kv, cols);
            t.mma();
            if (++s == a.kb_stages) { t.combine(); s = 0; }
        }
        t.store(a.C + b * a.strideC + m0 + (long long)n0 * a.ldc, a.ldc, 1.0f, 0.0f, rows, cols);
        t.fill_acc(0.0f);
    }
    t.release();
}

// Givens rotation (R#24): C_b = G(i, j, theta_b) X_b, G = identity except
// G(i,i) = G(j,j) = c_b, G(i,j) = -s_b, G(j,i) = s_b.  The operand is built with the
// map primitive: fill with 0, then single elements set where they live.
struct GivensArgs {
    int m, n, batch, gi, gj, kb_stages;
    const float* CS;                       // (c_b, s_b) pairs, 2*batch floats
    const float* X; long long ldx, strideX;
    float* C; long long ldc, strideC;
};

template <class Pol, int N>
__global__ void __launch_bounds__(128) tcec_givens_kernel(const GivensArgs a)
{
    extern __shared__ uint8_t smem[];
    using T = tile<Pol, N>;
    T t(smem);
    const int m0 = blockIdx.x * T::M, n0 = blockIdx.y * N;
    const int rows = min(T::M, a.m - m0), cols = min(N, a.n - n0);
    const int r = m0 + (int)threadIdx.x;   // this thread's row of G
    for (int b = blockIdx.z; b < a.batch; b += gridDim.z) {
        const float c = a.CS[2 * b], sn = a.CS[2 * b + 1];
        const float* X = a.X + b * a.strideX + (long long)n0 * a.ldx;
        int s = 0;
        for (int k0 = 0; k0 < a.m; k0 += T::BK) {
            const int kv = min(T::BK, a.m - k0);
            t.fill_a(0.0f);
            if ((int)threadIdx.x < rows && r >= k0 && r < k0 + kv)            // diagonal
                t.set_a((int)threadIdx.x, r - k0, (r == a.gi || r == a.gj) ? c : 1.0f);
            if (threadIdx.x == 0) {                                           // the two off-diagonal entries
                if (a.gi >= m0 && a.gi < m0 + rows && a.gj >= k0 && a.gj < k0 + kv)
                    t.set_a(a.gi - m0, a.gj - k0, -sn);
                if (a.gj >= m0 && a.gj < m0 + rows && a.gi >= k0 && a.gi < k0 + kv)
                    t.set_a(a.gj - m0, a.gi - k0, sn);
            }
            t.load_b(X + k0, a.ldx, kv, cols);
            t.mma();
            if (++s == a.kb_stages) { t.combine(); s = 0; }
        }
        t.store(a.C + b * a.strideC + m0 + (long long)n0 * a.ldc, a.ldc, 1.0f, 0.0f, rows, cols);
        t.fill_acc(0.0f);
    }
    t.release();
}

// Scan (Eq. scan-mat / u-rule, R#25): inclusive prefix sums of each
// column x of X (length n, contiguous) as y = L x with L(i, p) = [p <= i] = U^T,
// generated by rule (foreach_ij, Code 2 P:351-360).  count columns.
struct ScanArgs {
    int n, count, kb_stages;
    const float* X; long long ldx;
    float* Y; long long ldy;
};

template <class Pol, int N>
__global__ void __launch_bounds__(128) tcec_scan_kernel(const ScanArgs a)
{
    extern __shared__ uint8_t smem[];
    using T = tile<Pol, N>;
    T t(smem);
    const int m0 = blockIdx.x * T::M, n0 = blockIdx.y * N;
    const int rows = min(T::M, a.n - m0), cols = min(N, a.count - n0);
    const float* X = a.X + (long long)n0 * a.ldx;
    int s = 0;
    const int kend = min(a.n, m0 + rows);   // L(i, p) = 0 for p > i: later k-stages are all zero
    for (int k0 = 0; k0 < kend; k0 += T::BK) {
        const int kv = min(T::BK, a.n - k0);
        t.generate_a([&](int i, int p) { return (i < rows && p < kv && k0 + p <= m0 + i) ? 1.0f : 0.0f; });
        t.load_b(X + k0, a.ldx, kv, cols);
        t.mma();
        if (++s == a.kb_stages) { t.combine(); s = 0; }
    }
    t.store(a.Y + m0 + (long long)n0 * a.ldy, a.ldy, 1.0f, 0.0f, rows, cols);
    t.release();
}

}  // namespace tcec_kernels
}  // namespace emu

// ---------------------------------------------------------------- host side
namespace {

using emu::tcec::policy;
using emu::tcec::op_fp16;
using emu::tcec::op_tf32;
using emu::tcec::with_ec;
using emu::tcec::without_ec;
using emu::tcec::tensor_core;
using emu::tcec::simt;

constexpr unsigned kTcecFlags = EMU_FLAG_NO_CORRECTION | EMU_FLAG_SIMT | EMU_FLAG_PIPELINED;

// launch `Kern<Pol, N>` for the policy the (mode, flags) pair selects; N = 64
// on the tensor cores (two CTAs' operand rings and TMEM fit one SM), 32 on SIMT
template <template <class, int> class Launch, class Args>
emu_status tcec_dispatch(emu_split_mode mode, unsigned flags, dim3 grid, cudaStream_t s, const Args& a)
{
    const bool ec = !(flags & EMU_FLAG_NO_CORRECTION), sw = (flags & EMU_FLAG_SIMT) != 0;
    if (mode == EMU_SPLIT_FP16) {
        if (!sw) return ec ? Launch<policy<op_fp16, with_ec, tensor_core>, 64>::run(grid, s, a)
                           : Launch<policy<op_fp16, without_ec, tensor_core>, 64>::run(grid, s, a);
        return ec ? Launch<policy<op_fp16, with_ec, simt>, 32>::run(grid, s, a)
                  : Launch<policy<op_fp16, without_ec, simt>, 32>::run(grid, s, a);
    }
    if (!sw) return ec ? Launch<policy<op_tf32, with_ec, tensor_core>, 64>::run(grid, s, a)
                       : Launch<policy<op_tf32, without_ec, tensor_core>, 64>::run(grid, s, a);
    return ec ? Launch<policy<op_tf32, with_ec, simt>, 32>::run(grid, s, a)
              : Launch<policy<op_tf32, without_ec, simt>, 32>::run(grid, s, a);
}

template <class Kern>
emu_status tcec_set_smem(Kern kern, unsigned smem)
{
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return EMU_STATUS_CUDA_ERROR;
    return EMU_STATUS_SUCCESS;
}

#define TCEC_LAUNCHER(NAME, KERNEL, ARGS)                                                        \
    template <class Pol, int N>                                                                  \
    struct NAME {                                                                                \
        static emu_status run(dim3 grid, cudaStream_t s, const ARGS& a)                          \
        {                                                                                        \
            using T = emu::tcec::tile<Pol, N>;                                                   \
            auto kern = emu::tcec_kernels::KERNEL<Pol, N>;                                       \
            emu_status st = tcec_set_smem(kern, T::SMEM_BYTES);                           \
            if (st != EMU_STATUS_SUCCESS) return st;                                             \
            kern<<<grid, 128, T::SMEM_BYTES, s>>>(a);                                            \
            g_last_launches = 1;                                                                 \
            return launch_status(cudaGetLastError());                                            \
        }                                                                                        \
    };
TCEC_LAUNCHER(GemmLaunch, tcec_gemm_kernel, emu::tcec_kernels::GemmArgs)
TCEC_LAUNCHER(HouseLaunch, tcec_householder_kernel, emu::tcec_kernels::HouseArgs)
TCEC_LAUNCHER(GivensLaunch, tcec_givens_kernel, emu::tcec_kernels::GivensArgs)
TCEC_LAUNCHER(ScanLaunch, tcec_scan_kernel, emu::tcec_kernels::ScanArgs)
#undef TCEC_LAUNCHER

// (m-tiles, n-tiles, batch slices) of 128 x N blocks; N = 64 (tensor cores) or 32 (SIMT);
// false when the n-tiles exceed the grid's y limit
bool tcec_grid(int rows, int cols, int batch, unsigned flags, dim3& g)
{
    const int N = (flags & EMU_FLAG_SIMT) ? 32 : 64;
    const int ny = (cols + N - 1) / N;
    if (ny > 65535) return false;
    g = dim3((unsigned)((rows + 127) / 128), (unsigned)ny, (unsigned)std::min(batch, 65535));
    return true;
}

// KB (combine interval, elements) -> stages of BK (64 FP16 / 32 TF32); 0 = 64
bool tcec_kb_stages(int kblock, emu_split_mode mode, int& stages)
{
    const int bk = mode == EMU_SPLIT_FP16 ? 64 : 32;
    const int kb = kblock == 0 ? 64 : kblock;
    if (kb < bk || kb % bk != 0 || kb > 4096) return false;
    stages = kb / bk;
    return true;
}

bool tcec_common_ok(emu_split_mode mode, unsigned flags)
{
    return (mode == EMU_SPLIT_FP16 || mode == EMU_SPLIT_TF32) && !(flags & ~kTcecFlags);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) emu_status emu_tcec_gemm_batched(
    int m, int n, int k, float alpha, const float* A, int lda, long long strideA, const float* B, int ldb,
    long long strideB, float beta, float* C, int ldc, long long strideC, int batch, emu_split_mode mode,
    void* stream, int kblock, unsigned int flags)
{
    g_last_launches = 0;
    int kbs = 0;
    if (m < 0 || n < 0 || k < 0 || batch < 0 || !tcec_common_ok(mode, flags) || !tcec_kb_stages(kblock, mode, kbs))
        return EMU_STATUS_INVALID_VALUE;
    if (lda < std::max(1, m) || ldb < std::max(1, k) || ldc < std::max(1, m)) return EMU_STATUS_INVALID_VALUE;
    if (strideA < 0 || strideB < 0 || strideC < 0) return EMU_STATUS_INVALID_VALUE;
    if (m == 0 || n == 0 || batch == 0) return EMU_STATUS_SUCCESS;
    if (C == nullptr || (batch > 1 && strideC < (long long)ldc * n)) return EMU_STATUS_INVALID_VALUE;
    const bool reads_ab = k > 0 && alpha != 0.0f;
    if (reads_ab && (A == nullptr || B == nullptr)) return EMU_STATUS_INVALID_VALUE;
    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!reads_ab) {
        const long long cols = (long long)n * batch;
        scale_c_kernel<<<(unsigned)std::min<long long>(cols, 65535LL * 8), 256, 0, s>>>(C, m, n, ldc, strideC, batch,
                                                                                       beta);
        g_last_launches = 1;
        return launch_status(cudaGetLastError());
    }
    if (flags & EMU_FLAG_PIPELINED) {   // the warp-specialized form (= the library kernel, default operands)
        if (flags & EMU_FLAG_SIMT) return EMU_STATUS_NOT_SUPPORTED;
        if (!tma_domain(A, lda, batch > 1 ? strideA : 0) || !tma_domain(B, ldb, batch > 1 ? strideB : 0))
            return EMU_STATUS_NOT_SUPPORTED;
        const int kb = kblock ? kblock : default_kblock(k);
        const unsigned f = flags & EMU_FLAG_NO_CORRECTION;
        return mode == EMU_SPLIT_FP16
                   ? run_pipelined<0>(dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                                      batch, s, kb, f, emu::lib_operands())
                   : run_pipelined<1>(dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC,
                                      batch, s, kb, f, emu::lib_operands());
    }
    emu::tcec_kernels::GemmArgs a{m, n, k, batch, alpha, beta, A, lda, batch > 1 ? strideA : 0, B, ldb,
                                  batch > 1 ? strideB : 0, C, ldc, strideC, kbs};
    dim3 g;
    if (!tcec_grid(m, n, batch, flags, g)) return EMU_STATUS_NOT_SUPPORTED;
    return tcec_dispatch<GemmLaunch>(mode, flags, g, s, a);
}

__attribute__((visibility("default"))) emu_status emu_tcec_householder_batched(
    int m, int n, const float* V, long long strideV, const float* X, int ldx, long long strideX, float* C, int ldc,
    long long strideC, int batch, emu_split_mode mode, void* stream, unsigned int flags)
{
    g_last_launches = 0;
    int kbs = 0;
    if (m < 0 || n < 0 || batch < 0 || !tcec_common_ok(mode, flags) || !tcec_kb_stages(0, mode, kbs))
        return EMU_STATUS_INVALID_VALUE;
    if (ldx < std::max(1, m) || ldc < std::max(1, m) || strideV < 0 || strideX < 0 || strideC < 0)
        return EMU_STATUS_INVALID_VALUE;
    if (m == 0 || n == 0 || batch == 0) return EMU_STATUS_SUCCESS;
    if (V == nullptr || X == nullptr || C == nullptr) return EMU_STATUS_INVALID_VALUE;
    if (batch > 1 && strideC < (long long)ldc * n) return EMU_STATUS_INVALID_VALUE;
    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    if (flags & EMU_FLAG_PIPELINED) {   // H generated by the library kernel's splitter warps
        if (flags & EMU_FLAG_SIMT) return EMU_STATUS_NOT_SUPPORTED;
        if (!tma_domain(X, ldx, batch > 1 ? strideX : 0)) return EMU_STATUS_NOT_SUPPORTED;
        const emu::tcec_kernels::householder_operands ops{V, batch > 1 ? strideV : 0};
        const unsigned f = flags & EMU_FLAG_NO_CORRECTION;
        cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
        return mode == EMU_SPLIT_FP16
                   ? run_pipelined<0>(dev, sms, m, n, m, 1.0f, nullptr, m, 0, X, ldx, strideX, 0.0f, C, ldc, strideC,
                                      batch, s, 64, f, ops)
                   : run_pipelined<1>(dev, sms, m, n, m, 1.0f, nullptr, m, 0, X, ldx, strideX, 0.0f, C, ldc, strideC,
                                      batch, s, 64, f, ops);
    }
    emu::tcec_kernels::HouseArgs a{m, n, batch, kbs, V, batch > 1 ? strideV : 0, X, ldx, batch > 1 ? strideX : 0,
                                   C, ldc, strideC};
    dim3 g;
    if (!tcec_grid(m, n, batch, flags, g)) return EMU_STATUS_NOT_SUPPORTED;
    return tcec_dispatch<HouseLaunch>(mode, flags, g, reinterpret_cast<cudaStream_t>(stream), a);
}

__attribute__((visibility("default"))) emu_status emu_tcec_givens_batched(
    int m, int n, int i, int j, const float* CS, const float* X, int ldx, long long strideX, float* C, int ldc,
    long long strideC, int batch, emu_split_mode mode, void* stream, unsigned int flags)
{
    g_last_launches = 0;
    int kbs = 0;
    if (m < 0 || n < 0 || batch < 0 || !tcec_common_ok(mode, flags) || !tcec_kb_stages(0, mode, kbs))
        return EMU_STATUS_INVALID_VALUE;
    if (ldx < std::max(1, m) || ldc < std::max(1, m) || strideX < 0 || strideC < 0) return EMU_STATUS_INVALID_VALUE;
    if (m == 0 || n == 0 || batch == 0) return EMU_STATUS_SUCCESS;
    if (i < 0 || j < 0 || i >= m || j >= m || i == j) return EMU_STATUS_INVALID_VALUE;
    if (flags & EMU_FLAG_PIPELINED) return EMU_STATUS_NOT_SUPPORTED;   // tile form only
    if (CS == nullptr || X == nullptr || C == nullptr) return EMU_STATUS_INVALID_VALUE;
    if (batch > 1 && strideC < (long long)ldc * n) return EMU_STATUS_INVALID_VALUE;
    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    emu::tcec_kernels::GivensArgs a{m, n, batch, i, j, kbs, CS, X, ldx, batch > 1 ? strideX : 0, C, ldc, strideC};
    dim3 g;
    if (!tcec_grid(m, n, batch, flags, g)) return EMU_STATUS_NOT_SUPPORTED;
    return tcec_dispatch<GivensLaunch>(mode, flags, g, reinterpret_cast<cudaStream_t>(stream), a);
}

__attribute__((visibility("default"))) emu_status emu_tcec_scan(int n, int count, const float* X, int ldx, float* Y,
                                                                 int ldy, emu_split_mode mode, void* stream,
                                                                 unsigned int flags)
{
    g_last_launches = 0;
    int kbs = 0;
    if (n < 0 || count < 0 || !tcec_common_ok(mode, flags) || !tcec_kb_stages(0, mode, kbs))
        return EMU_STATUS_INVALID_VALUE;
    if (ldx < std::max(1, n) || ldy < std::max(1, n)) return EMU_STATUS_INVALID_VALUE;
    if (n == 0 || count == 0) return EMU_STATUS_SUCCESS;
    if (X == nullptr || Y == nullptr) return EMU_STATUS_INVALID_VALUE;
    if (flags & EMU_FLAG_PIPELINED) return EMU_STATUS_NOT_SUPPORTED;   // tile form only
    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    emu::tcec_kernels::ScanArgs a{n, count, kbs, X, ldx, Y, ldy};
    dim3 g;
    if (!tcec_grid(n, count, 1, flags, g)) return EMU_STATUS_NOT_SUPPORTED;
    return tcec_dispatch<ScanLaunch>(mode, flags, g, reinterpret_cast<cudaStream_t>(stream), a);
}

}  // extern "C"
