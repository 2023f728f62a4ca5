// api.cu -- the C ABI of libemusgemm.so (declared and documented in
// include/emu_sgemm.h): argument validation, tensor-map encoding, launch.
// Every arithmetic step of the method runs in the kernels of this library.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "emu_sgemm.h"
#include "gemm_pair_sm100.cuh"
#include "gemm_pair_ts_sm100.cuh"
#include "gemm_sm100.cuh"
#include "split.cuh"

#define EMU_VERSION 100  // 0.1.0

namespace {

thread_local int g_last_launches = 0;
// name of the GEMM kernel the last call on this host thread dispatched (diagnostics)
thread_local const char* g_last_kernel = "";

// one static name per kernel instantiation, built once
template <typename F>
const char* kernel_name_once(F build)
{
    static char buf[192];
    static std::once_flag once;
    std::call_once(once, [&] { build(buf, sizeof(buf)); });
    return buf;
}

// extra result destinations of the emu_sgemm_multicast call in progress on this
// host thread (nullptr otherwise); read by the TS-kernel launcher
struct MultiDst {
    int n;
    float* d[8];
};
thread_local const MultiDst* g_mdst = nullptr;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn()
{
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

struct DeviceInfo {
    int ok = -1;  // -1 unknown, 0 not sm_100, 1 sm_100
    int sms = 0;
    bool attr_set[32] = {};
    bool pair_attr_set[16] = {};
};

constexpr int kMaxDevices = 64;
DeviceInfo g_dev[kMaxDevices];
std::mutex g_dev_mu;

// host-buffer entry: per-device internal streams and a grow-only workspace
struct HostCtx {
    std::mutex mu;
    bool init = false;
    cudaStream_t st[2] = {nullptr, nullptr};
    cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
    float* ws = nullptr;
    size_t ws_bytes = 0;
};
HostCtx g_host[kMaxDevices];

emu_status device_check(int& dev, int& sms)
{
    if (cudaGetDevice(&dev) != cudaSuccess) return EMU_STATUS_CUDA_ERROR;
    if (dev < 0 || dev >= kMaxDevices) return EMU_STATUS_CUDA_ERROR;
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DeviceInfo& d = g_dev[dev];
    if (d.ok < 0) {
        int major = 0, minor = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            return EMU_STATUS_CUDA_ERROR;
        d.ok = (major == 10 && minor == 0) ? 1 : 0;
    }
    sms = d.sms;
    return d.ok == 1 ? EMU_STATUS_SUCCESS : EMU_STATUS_ARCH_MISMATCH;
}

template <int MODE, int BN, int ALAY, bool RANGE, bool LDG>
emu_status ensure_smem_attr(int dev)
{
    std::lock_guard<std::mutex> lk(g_dev_mu);
    const int slot = ((MODE * 4 + ALAY) * 2 + (RANGE ? 1 : 0)) * 2 + (LDG ? 1 : 0);
    if (g_dev[dev].attr_set[slot]) return EMU_STATUS_SUCCESS;
    if (cudaFuncSetAttribute(emu::emu_sgemm_kernel<MODE, BN, ALAY, RANGE, LDG>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)emu::GemmCfg<MODE, BN, ALAY>::SMEM_BYTES) != cudaSuccess)
        return EMU_STATUS_CUDA_ERROR;
    g_dev[dev].attr_set[slot] = true;
    return EMU_STATUS_SUCCESS;
}

// 3-D FP32 tensor map {dim0 contiguous, dim1, batch}
bool make_map(CUtensorMap* map, const float* base, uint64_t d0, uint64_t d1, uint64_t ld,
              uint64_t nbatch, uint64_t bstride, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw)
{
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, nbatch};
    cuuint64_t strides[2] = {ld * 4, bstride * 4};
    cuuint32_t box[3] = {box0, box1, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// k == 0 or alpha == 0: C = RN(beta*C) (beta == 0 writes +0 and never reads C)
__global__ void scale_c_kernel(float* C, int m, int n, long long ldc, long long strideC, int batch, float beta)
{
    const long long cols = (long long)n * batch;
    for (long long cj = blockIdx.x; cj < cols; cj += gridDim.x) {
        const long long b = cj / n, j = cj - b * n;
        float* col = C + b * strideC + j * ldc;
        for (int i = threadIdx.x; i < m; i += blockDim.x) col[i] = beta != 0.0f ? __fmul_rn(beta, col[i]) : 0.0f;
    }
}

// range-safe mode (R#22): bit patterns of the max finite |x| of every row of A_b and
// column of B_b (non-negative binary32 values order like their bit patterns, so an
// integer atomicMax merges the k-chunks).  One block per (item, A row block of 256 x
// k-chunk of ka) or (item, B column block of 8 warps x k-chunk of kb): short A chunks
// give the row pass (one strided column read per k) enough blocks to reach HBM rates.
__global__ void range_max_kernel(const float* __restrict__ A, long long lda, long long strideA,
                                 const float* __restrict__ B, long long ldb, long long strideB, int m, int n, int k,
                                 int a_blocks, int b_blocks, int ka, int kb, unsigned* __restrict__ row_max,
                                 unsigned* __restrict__ col_max)
{
    const int a_ch = (k + ka - 1) / ka, b_ch = (k + kb - 1) / kb;
    const long long per_item = (long long)a_blocks * a_ch + (long long)b_blocks * b_ch;
    const long long item = blockIdx.x / per_item;
    long long w = blockIdx.x - item * per_item;
    if (w < (long long)a_blocks * a_ch) {
        const int blk = (int)(w / a_ch), p0 = (int)(w % a_ch) * ka, p1 = min(k, p0 + ka);
        const int r = blk * 256 + (int)threadIdx.x;
        if (r >= m) return;
        const float* a = A + item * strideA + r;
        float mx = 0.0f;
#pragma unroll 8
        for (int p = p0; p < p1; ++p) {
            const float v = fabsf(__ldg(a + (long long)p * lda));
            if (v <= 3.402823466e38f) mx = fmaxf(mx, v);   // finite values only (NaN compares false)
        }
        if (mx > 0.0f) atomicMax(row_max + item * m + r, __float_as_uint(mx));
    } else {
        w -= (long long)a_blocks * a_ch;
        const int blk = (int)(w / b_ch), p0 = (int)(w % b_ch) * kb, p1 = min(k, p0 + kb);
        const int c = blk * 8 + (int)(threadIdx.x >> 5);
        if (c >= n) return;
        const float* bcol = B + item * strideB + (long long)c * ldb;
        float mx = 0.0f;
        for (int p = p0 + (int)(threadIdx.x & 31); p < p1; p += 32) {
            const float v = fabsf(__ldg(bcol + p));
            if (v <= 3.402823466e38f) mx = fmaxf(mx, v);
        }
        const unsigned bits = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
        if ((threadIdx.x & 31) == 0 && bits) atomicMax(col_max + item * n + c, bits);
    }
}

__global__ void split_fp16_kernel(const float* __restrict__ x, long long count, uint16_t* __restrict__ hi,
                                  uint16_t* __restrict__ lo)
{
    const long long pairs = count / 2;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride) {
        const float2 v = reinterpret_cast<const float2*>(x)[i];
        uint32_t h, l;
        emu::split_fp16x2(v.x, v.y, h, l);
        reinterpret_cast<uint32_t*>(hi)[i] = h;
        reinterpret_cast<uint32_t*>(lo)[i] = l;
    }
    if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        uint32_t h, l;
        emu::split_fp16x2(x[count - 1], 0.0f, h, l);
        hi[count - 1] = (uint16_t)(h & 0xffffu);
        lo[count - 1] = (uint16_t)(l & 0xffffu);
    }
}

__global__ void split_tf32_kernel(const float* __restrict__ x, long long count, uint32_t* __restrict__ hi,
                                  uint32_t* __restrict__ lo)
{
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        uint32_t h, l;
        emu::split_tf32(x[i], h, l);
        hi[i] = h;
        lo[i] = l;
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// an FP32 operand the TMA path can read: 16-byte aligned base, leading dimension and
// batch stride in 16-byte units
bool tma_domain(const float* X, long long ld, long long stride)
{
    return aligned16(X) && ld % 4 == 0 && stride % 4 == 0;
}

// L2 prefetch distance (k-stages) of the TMA producer; EMU_PREFETCH overrides (tuning only)
int env_int(const char* name, int dflt, int lo, int hi)
{
    const char* e = getenv(name);
    return e ? std::max(lo, std::min(hi, atoi(e))) : dflt;
}

// Launch with programmatic stream serialization (PDL): the GEMM kernels call
// griddepcontrol.wait before touching global memory, so their prologue overlaps
// the previous kernel's tail and the launch latency is hidden (sm100_ptx.cuh).
// EMU_PDL=0 launches them plainly (A/B measurements).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args... args)
{
    static const int pdl = env_int("EMU_PDL", 1, 0, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

int prefetch_distance()
{
    static const int pf = [] {
        const char* e = getenv("EMU_PREFETCH");
        return e ? std::max(0, std::min(64, atoi(e))) : 0;   // measured: prefetch slows c2 (PF 8: -6 %)
    }();
    return pf;
}

emu_status launch_status(cudaError_t e)
{
    if (e == cudaSuccess) return EMU_STATUS_SUCCESS;
    return EMU_STATUS_LAUNCH_FAILED;
}

template <int MODE, int ALAY, bool RANGE, bool LDG>
emu_status run_gemm(int dev, int sms, int m, int n, int k, float alpha, const float* A, int lda, long long strideA,
                    const float* B, int ldb, long long strideB, float beta, float* C, int ldc, long long strideC,
                    int batch, cudaStream_t stream, unsigned* range_flag, int kblock, unsigned flags)
{
    constexpr int BN = 128;
    using Cfg = emu::GemmCfg<MODE, BN, ALAY>;
    emu_status st = ensure_smem_attr<MODE, BN, ALAY, RANGE, LDG>(dev);
    if (st != EMU_STATUS_SUCCESS) return st;

    const bool a_b = batch > 1 && strideA != 0;
    const bool b_b = batch > 1 && strideB != 0;
    CUtensorMap tmA, tmB, tmC;
    std::memset(&tmA, 0, sizeof(tmA));
    std::memset(&tmB, 0, sizeof(tmB));
    std::memset(&tmC, 0, sizeof(tmC));
    // TMA-store epilogue: beta == 0 and a 16-byte-unit C layout
    const bool c_b = batch > 1;
    int tma_store = Cfg::CSTAGE_BYTES != 0 && beta == 0.0f && aligned16(C) && ldc % 4 == 0 &&
                    (!c_b || strideC % 4 == 0) && (unsigned long long)strideC * 4 < (1ull << 40);
    if (tma_store) {
        const uint64_t sC = c_b ? (uint64_t)strideC : (((uint64_t)ldc * (uint64_t)n + 3) & ~uint64_t(3));
        if (!make_map(&tmC, C, (uint64_t)m, (uint64_t)n, (uint64_t)ldc, c_b ? (uint64_t)batch : 1, sC, Cfg::BM, 32,
                      CU_TENSOR_MAP_SWIZZLE_NONE))
            tma_store = 0;
    }
    // dim-2 stride: any valid value when the batch extent is 1
    const uint64_t sA = a_b ? (uint64_t)strideA : (((uint64_t)lda * (uint64_t)k + 3) & ~uint64_t(3));
    const uint64_t sB = b_b ? (uint64_t)strideB : (((uint64_t)ldb * (uint64_t)n + 3) & ~uint64_t(3));
    if (!LDG && !make_map(&tmA, A, (uint64_t)m, (uint64_t)k, (uint64_t)lda, a_b ? (uint64_t)batch : 1, sA, Cfg::BM,
                          Cfg::BK, CU_TENSOR_MAP_SWIZZLE_NONE))
        return EMU_STATUS_NOT_SUPPORTED;
    if (!LDG && !make_map(&tmB, B, (uint64_t)k, (uint64_t)n, (uint64_t)ldb, b_b ? (uint64_t)batch : 1, sB, Cfg::BK,
                          BN, CU_TENSOR_MAP_SWIZZLE_128B))
        return EMU_STATUS_NOT_SUPPORTED;

    emu::GemmParams p;
    p.m = m; p.n = n; p.k = k;
    p.a_batched = a_b; p.b_batched = b_b;
    p.alpha = alpha; p.beta = beta;
    p.C = C; p.ldc = ldc; p.strideC = strideC;
    p.tiles_m = (m + Cfg::BM - 1) / Cfg::BM;
    p.tiles_n = (n + BN - 1) / BN;
    p.num_tiles = (long long)p.tiles_m * p.tiles_n * batch;
    p.num_k_stages = (k + Cfg::BK - 1) / Cfg::BK;
    p.kb_stages = (kblock > 0 ? kblock : 64) / Cfg::BK;
    p.corr = (flags & EMU_FLAG_NO_CORRECTION) ? 0 : 1;
    p.range_flag = MODE == 0 ? range_flag : nullptr;
    p.tma_store = tma_store;
    p.prefetch = prefetch_distance();
    {
        static const int gm = env_int("EMU_GROUP_M", 2, 1, 1 << 20);    // tuning only (c3 DRAM bytes: 2 < 4 < 8 < 16, profiles/r01_summary.md)
        static const int pol = env_int("EMU_L2_POLICY", 0, 0, 3);      // tuning only
        p.group_m = gm;
        p.l2_policy = pol;
    }
    p.A = A; p.B = B; p.lda = lda; p.ldb = ldb;
    p.strideA = a_b ? strideA : 0; p.strideB = b_b ? strideB : 0;

    const long long grid = std::min<long long>(p.num_tiles, sms);
    const cudaError_t le = launch_pdl(emu::emu_sgemm_kernel<MODE, BN, ALAY, RANGE, LDG>, (unsigned)grid, Cfg::NUM_THREADS,
                                      Cfg::SMEM_BYTES, stream, tmA, tmB, tmC, p);
    if (le != cudaSuccess) return launch_status(le);
    g_last_launches = 1;
    g_last_kernel = kernel_name_once([](char* b, size_t nb) {
        snprintf(b, nb, "emu_sgemm_kernel<%s, BN=%d, A layout %d%s%s> (single CTA, M=128)", MODE == 0 ? "FP16" : "TF32",
                 BN, ALAY, RANGE ? ", range flag" : "", LDG ? ", direct loads" : "");
    });
    return launch_status(cudaGetLastError());
}

template <int MODE, int ALAY, bool RANGE>
emu_status run_gemm_pair(int dev, int sms, int m, int n, int k, float alpha, const float* A, int lda,
                         long long strideA, const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                         long long strideC, int batch, cudaStream_t stream, unsigned* range_flag, int kblock,
                         unsigned flags)
{
    using Cfg = emu::PairCfg<MODE, ALAY>;
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        const int slot = (MODE * 4 + ALAY) * 2 + (RANGE ? 1 : 0);
        if (!g_dev[dev].pair_attr_set[slot]) {
            if (cudaFuncSetAttribute(emu::emu_sgemm_pair_kernel<MODE, ALAY, RANGE>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM_BYTES) != cudaSuccess)
                return EMU_STATUS_CUDA_ERROR;
            g_dev[dev].pair_attr_set[slot] = true;
        }
    }
    const bool a_b = batch > 1 && strideA != 0;
    const bool b_b = batch > 1 && strideB != 0;
    const bool c_b = batch > 1;
    CUtensorMap tmA, tmB, tmC;
    std::memset(&tmA, 0, sizeof(tmA));
    std::memset(&tmB, 0, sizeof(tmB));
    std::memset(&tmC, 0, sizeof(tmC));
    const uint64_t sA = a_b ? (uint64_t)strideA : (((uint64_t)lda * (uint64_t)k + 3) & ~uint64_t(3));
    const uint64_t sB = b_b ? (uint64_t)strideB : (((uint64_t)ldb * (uint64_t)n + 3) & ~uint64_t(3));
    if (!make_map(&tmA, A, (uint64_t)m, (uint64_t)k, (uint64_t)lda, a_b ? (uint64_t)batch : 1, sA, Cfg::BM, Cfg::BK,
                  CU_TENSOR_MAP_SWIZZLE_NONE))
        return EMU_STATUS_NOT_SUPPORTED;
    if (!make_map(&tmB, B, (uint64_t)k, (uint64_t)n, (uint64_t)ldb, b_b ? (uint64_t)batch : 1, sB, Cfg::BK, Cfg::BNC,
                  CU_TENSOR_MAP_SWIZZLE_128B))
        return EMU_STATUS_NOT_SUPPORTED;
    int tma_store = beta == 0.0f && aligned16(C) && ldc % 4 == 0 && (!c_b || strideC % 4 == 0) &&
                    (unsigned long long)strideC * 4 < (1ull << 40);
    if (tma_store) {
        const uint64_t sC = c_b ? (uint64_t)strideC : (((uint64_t)ldc * (uint64_t)n + 3) & ~uint64_t(3));
        if (!make_map(&tmC, C, (uint64_t)m, (uint64_t)n, (uint64_t)ldc, c_b ? (uint64_t)batch : 1, sC, Cfg::BM, 32,
                      CU_TENSOR_MAP_SWIZZLE_NONE))
            tma_store = 0;
    }
    emu::GemmParams p;
    std::memset(&p, 0, sizeof(p));
    p.m = m; p.n = n; p.k = k;
    p.a_batched = a_b; p.b_batched = b_b;
    p.alpha = alpha; p.beta = beta;
    p.C = C; p.ldc = ldc; p.strideC = strideC;
    p.tiles_m = (m + 255) / 256;
    p.tiles_n = (n + Cfg::BN - 1) / Cfg::BN;
    p.num_tiles = (long long)p.tiles_m * p.tiles_n * batch;
    p.num_k_stages = (k + Cfg::BK - 1) / Cfg::BK;
    p.kb_stages = (kblock > 0 ? kblock : 64) / Cfg::BK;
    p.corr = (flags & EMU_FLAG_NO_CORRECTION) ? 0 : 1;
    p.tma_store = tma_store;
    p.prefetch = prefetch_distance();
    {
        static const int gm = env_int("EMU_GROUP_M", 2, 1, 1 << 20);    // tuning only (c3 DRAM bytes: 2 < 4 < 8 < 16, profiles/r01_summary.md)
        static const int pol = env_int("EMU_L2_POLICY", 0, 0, 3);      // tuning only
        p.group_m = gm;
        p.l2_policy = pol;
    }
    p.range_flag = MODE == 0 ? range_flag : nullptr;
    const long long clusters = std::min<long long>(p.num_tiles, sms / 2);
    const cudaError_t le = launch_pdl(emu::emu_sgemm_pair_kernel<MODE, ALAY, RANGE>, (unsigned)(2 * clusters),
                                      Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream, tmA, tmB, tmC, p);
    if (le != cudaSuccess) return launch_status(le);
    g_last_launches = 1;
    g_last_kernel = kernel_name_once([](char* b, size_t nb) {
        snprintf(b, nb, "emu_sgemm_pair_kernel<%s, A layout %d%s> (CTA pair, both operands in SMEM)",
                 MODE == 0 ? "FP16" : "TF32", ALAY, RANGE ? ", range flag" : "");
    });
    return launch_status(cudaGetLastError());
}

template <int MODE, int RANGE, int BN, bool SPLITC, bool ASTAT, bool TA = false, bool TB = false, bool LONGK = false,
          class Ops = emu::lib_operands>
emu_status run_gemm_pair_ts(int dev, int sms, int m, int n, int k, float alpha, const float* A, int lda,
                         long long strideA, const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                         long long strideC, int batch, cudaStream_t stream, unsigned* range_flag, int kblock,
                         unsigned flags, const unsigned* row_max, const unsigned* col_max, const Ops& ops = Ops())
{
    using Cfg = emu::PairTsCfg<MODE, BN, SPLITC, ASTAT, LONGK>;
    {
        // the dynamic shared-memory attribute, once per device and instantiation
        static bool attr_set[kMaxDevices] = {};
        std::lock_guard<std::mutex> lk(g_dev_mu);
        if (!attr_set[dev]) {
            if (cudaFuncSetAttribute(emu::emu_sgemm_pair_ts_kernel<MODE, RANGE, BN, SPLITC, ASTAT, TA, TB, false, LONGK, Ops>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM_BYTES) != cudaSuccess)
                return EMU_STATUS_CUDA_ERROR;
            if constexpr (!RANGE && !TA && !TB) {
                if (cudaFuncSetAttribute(emu::emu_sgemm_pair_ts_kernel<MODE, RANGE, BN, SPLITC, ASTAT, TA, TB, true, LONGK, Ops>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cfg::SMEM_BYTES) != cudaSuccess)
                    return EMU_STATUS_CUDA_ERROR;
            }
            attr_set[dev] = true;
        }
    }
    const bool a_b = batch > 1 && strideA != 0;
    const bool b_b = batch > 1 && strideB != 0;
    const bool c_b = batch > 1;
    CUtensorMap tmA, tmB, tmC;
    std::memset(&tmA, 0, sizeof(tmA));
    std::memset(&tmB, 0, sizeof(tmB));
    std::memset(&tmC, 0, sizeof(tmC));
    const uint64_t sA = a_b ? (uint64_t)strideA : (((uint64_t)lda * (uint64_t)(TA ? m : k) + 3) & ~uint64_t(3));
    const uint64_t sB = b_b ? (uint64_t)strideB : (((uint64_t)ldb * (uint64_t)(TB ? k : n) + 3) & ~uint64_t(3));
    // op(A) = A (m x k, m contiguous) or A^T (A stored k x m); op(B) = B (k x n) or B^T (B stored n x k)
    // generated operands (Ops::gen_a / gen_b) need no tensor map
    const bool mapA = Ops::gen_a ? true : TA ? make_map(&tmA, A, (uint64_t)k, (uint64_t)m, (uint64_t)lda, a_b ? (uint64_t)batch : 1, sA,
                                    Cfg::BK, Cfg::BM, CU_TENSOR_MAP_SWIZZLE_128B)
                         : make_map(&tmA, A, (uint64_t)m, (uint64_t)k, (uint64_t)lda, a_b ? (uint64_t)batch : 1, sA,
                                    Cfg::BM, Cfg::BK, CU_TENSOR_MAP_SWIZZLE_NONE);
    const bool mapB = Ops::gen_b ? true : TB ? make_map(&tmB, B, (uint64_t)n, (uint64_t)k, (uint64_t)ldb, b_b ? (uint64_t)batch : 1, sB,
                                    Cfg::BNC, Cfg::BK, CU_TENSOR_MAP_SWIZZLE_NONE)
                         : make_map(&tmB, B, (uint64_t)k, (uint64_t)n, (uint64_t)ldb, b_b ? (uint64_t)batch : 1, sB,
                                    Cfg::BK, Cfg::BNC, CU_TENSOR_MAP_SWIZZLE_128B);
    if (!mapA || !mapB) return EMU_STATUS_NOT_SUPPORTED;
    int tma_store = beta == 0.0f && aligned16(C) && ldc % 4 == 0 && (!c_b || strideC % 4 == 0) &&
                    (unsigned long long)strideC * 4 < (1ull << 40);
    bool c_box128 = false;
    if (g_mdst && g_mdst->n > 1) tma_store = 0;   // multicast: st.global to every destination
    if (Cfg::CSTAGE_BYTES == 0) tma_store = 0;     // long-k variant: no C staging area
    if (Ops::custom_store) tma_store = 0;          // the user's epilogue stores
    // tuning only (0: st.global from the combine warps; c2 fp16 204.7 vs 236.2 TF, ABBA)
    static const int tma_store_env = env_int("EMU_TMA_STORE", 1, 0, 1);
    if (!tma_store_env) tma_store = 0;
    if (tma_store) {
        const uint64_t sC = c_b ? (uint64_t)strideC : (((uint64_t)ldc * (uint64_t)n + 3) & ~uint64_t(3));
        // one 32-row x ECOLS block per combine warp (each warp stores its own columns), or
        // one 128-row block per column group of 4 warps: TF32 +1.1 %, FP16 -0.3 % (c2, ABBA),
        // so the default for TF32 only (EMU_C_BOX128=0/1 overrides, tuning)
        static const int box128_env = env_int("EMU_C_BOX128", -1, -1, 1);
        const int box128 = box128_env >= 0 ? box128_env : (MODE == 1 ? 1 : 0);
        if (!make_map(&tmC, C, (uint64_t)m, (uint64_t)n, (uint64_t)ldc, c_b ? (uint64_t)batch : 1, sC,
                      box128 ? Cfg::BM : 32, Cfg::ECOLS, CU_TENSOR_MAP_SWIZZLE_NONE))
            tma_store = 0;
        c_box128 = box128 != 0;
    }
    emu::GemmParams p;
    std::memset(&p, 0, sizeof(p));
    p.m = m; p.n = n; p.k = k;
    p.a_batched = a_b; p.b_batched = b_b;
    p.alpha = alpha; p.beta = beta;
    p.C = C; p.ldc = ldc; p.strideC = strideC;
    p.tiles_m = (m + 255) / 256;
    p.tiles_n = (n + Cfg::BN - 1) / Cfg::BN;
    p.num_tiles = (long long)p.tiles_m * p.tiles_n * batch;
    p.num_k_stages = (k + Cfg::BK - 1) / Cfg::BK;
    p.kb_stages = (kblock > 0 ? kblock : 64) / Cfg::BK;
    p.corr = (flags & EMU_FLAG_NO_CORRECTION) ? 0 : 1;
    p.tma_store = tma_store;
    p.prefetch = prefetch_distance();
    // long-k streaming tiles: one cluster per tile; the running (persistent) clusters take over
    // the rest by cluster launch control, in launch order, each claiming its next tile p.clc
    // k-stages before its current one's loads end (EMU_TS_CLC; 0: static order, cluster c
    // takes tiles c, c + 74, ...).  The clusters that share an operand panel then start it
    // close together instead of drifting apart over the launch, so the panel is reused in L2:
    // c3 DRAM reads 70 -> 37 GB per launch (profiles/r02_summary.md)
    static const int clc_env = env_int("EMU_TS_CLC", 8, 0, 1 << 20);   // tuning only
    static const int clc_as_env = env_int("EMU_TS_CLC_ASTAT", 0, 0, 1);   // tuning only
    const long long units = ASTAT ? (long long)p.tiles_m * batch : p.num_tiles;
    p.clc = (LONGK || (ASTAT && clc_as_env)) && units <= (1LL << 30) ? clc_env : 0;
    {
        // raster group: m-tiles per group walking the n-tiles together (EMU_GROUP_M, tuning);
        // dynamic order: 3 (each B panel is read by 3 row blocks close together)
        static const int gm = env_int("EMU_GROUP_M", 0, 0, 1 << 20);
        static const int pol = env_int("EMU_L2_POLICY", -1, -1, 31);   // tuning only (-1: default below)
        p.group_m = gm ? gm : (p.clc ? 3 : 2);
        // streaming tiles (grouped raster), static order: B evict_first (each B tile is used by the
        // two row blocks of a group at about the same time, then not again), A evict_last (a
        // group's rows are reread by every n-tile): c3 fp16 +5 %, tf32 +3.5 % from lower DRAM
        // power under the power cap (profiles/r01_summary.md).  Dynamic order: B normal (the
        // group's readers come within ~10 us of each other), A evict_last.  A-stationary units
        // read A and B once: default policy.  Bit 4 (tuning): B evict_last.
        p.l2_policy = pol >= 0 ? pol : (ASTAT ? 0 : (p.clc ? 2 : 3));
        if (c_box128) p.l2_policy |= 8;
        static const int c_ef = env_int("EMU_C_EVICT_FIRST", 0, 0, 1);   // tuning only
        if (c_ef) p.l2_policy |= 4;
    }
    p.range_flag = MODE == 0 ? range_flag : nullptr;
    p.row_max = row_max;
    p.col_max = col_max;
    if (g_mdst) {
        p.num_dst = g_mdst->n;
        for (int d = 0; d < g_mdst->n; ++d) p.dst[d] = g_mdst->d[d];
    }
    p.num_units = ASTAT ? (long long)p.tiles_m * batch : p.num_tiles;
    p.unit_tiles = ASTAT ? p.tiles_n : 1;
    if (ASTAT && p.num_k_stages > Cfg::ASLOTS) return EMU_STATUS_NOT_SUPPORTED;   // dispatch guarantees it
    const long long clusters = p.clc ? p.num_units : std::min<long long>(p.num_units, sms / 2);
    // the multicast epilogue is its own instantiation (MC): the plain kernels carry no
    // per-destination loop
    bool launched = false;
    if constexpr (!RANGE && !TA && !TB) {
        if (p.num_dst > 1) {
            const cudaError_t le = launch_pdl(emu::emu_sgemm_pair_ts_kernel<MODE, RANGE, BN, SPLITC, ASTAT, TA, TB, true, LONGK, Ops>,
                                              (unsigned)(2 * clusters), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream, tmA,
                                              tmB, tmC, p, ops);
            if (le != cudaSuccess) return launch_status(le);
            launched = true;
        }
    }
    if (!launched) {
        if (p.num_dst > 1) return EMU_STATUS_NOT_SUPPORTED;
        const cudaError_t le = launch_pdl(emu::emu_sgemm_pair_ts_kernel<MODE, RANGE, BN, SPLITC, ASTAT, TA, TB, false, LONGK, Ops>,
                                          (unsigned)(2 * clusters), Cfg::NUM_THREADS, Cfg::SMEM_BYTES, stream, tmA, tmB,
                                          tmC, p, ops);
        if (le != cudaSuccess) return launch_status(le);
    }
    g_last_launches = 1;
    // (the tile order is fixed per process: p.clc follows static tuning knobs)
    const bool dyn = p.clc != 0;
    g_last_kernel = kernel_name_once([dyn](char* b, size_t nb) {
        snprintf(b, nb, "emu_sgemm_pair_ts_kernel<%s, %d cols%s%s%s%s%s%s%s%s> (CTA pair, A in TMEM)",
                 MODE == 0 ? "FP16" : "TF32", BN, SPLITC ? ", split commit" : "", ASTAT ? ", A-stationary" : "",
                 Cfg::LONGK ? ", long-k rings" : "", dyn ? ", dynamic tile order" : "",
                 (RANGE & 2) ? ", range-safe" : "", (RANGE & 1) ? ", range flag" : "", TA ? ", op(A)=T" : "",
                 TB ? ", op(B)=T" : "");
    });
    if (launched) g_last_kernel = "emu_sgemm_pair_ts_kernel<multicast epilogue> (CTA pair, A in TMEM)";
    return launch_status(cudaGetLastError());
}

// TS-kernel variant for a problem (shared by the library entries and the pipelined
// device-API entries): tile width, split commit, A-stationary, long-k rings
struct TsPlan {
    int n;
    bool sc, as, lk;
};

TsPlan ts_plan(int mode, int m, int n, int k, int batch, int sms, bool multicast)
{
    static const int ts_n_env = env_int("EMU_TS_N", 0, 0, 128);   // tuning only
    // few tiles (fewer 256 x 128 tiles than clusters, e.g. c4's 1024^2 output): 64-wide
    // tiles with double-buffered accumulators put twice as many clusters to work
    const long long ts_tiles128 = (long long)((m + 255) / 256) * ((n + 127) / 128) * batch;
    TsPlan t;
    t.n = ts_n_env ? ts_n_env : (ts_tiles128 < sms / 2 && n > 64 && !multicast ? 64 : 128);
    static const int ts_sc_env = env_int("EMU_TS_SPLITC", 1, 0, 1);   // tuning only (default on)
    static const int ts_as_env = env_int("EMU_TS_ASTAT", 1, 0, 1);    // tuning only (default on)
    t.sc = t.n == 128 && ts_sc_env;
    // A-stationary: all of k fits the TMEM A slots, at least two n-tiles share the split
    // A, and there are enough (batch, m-pair) row blocks to keep every cluster busy
    const long long ts_units = (long long)((m + 255) / 256) * batch;
    const int ts_aslots = mode == EMU_SPLIT_FP16 ? emu::PairTsCfg<0, 128, true, true>::ASLOTS
                                                 : emu::PairTsCfg<1, 128, true, true>::ASLOTS;
    t.as = t.sc && ts_as_env && (k + 31) / 32 <= ts_aslots && (n + 127) / 128 >= 2 && ts_units >= 2LL * (sms / 2);
    // long k, streaming tiles: deeper operand / FP32 rings instead of the C staging area
    static const int ts_lk_env = env_int("EMU_TS_LONGK", 1, 0, 1);   // tuning only (default on)
    t.lk = t.sc && !t.as && ts_lk_env && (k + 31) / 32 >= 64;
    return t;
}

// the pipelined (warp-specialized) form of the device API (include/emu_tcec_pipeline.cuh):
// the library's TS kernel with the caller's operand / epilogue hooks (no range mode,
// no transposes; column-major, alpha / beta as the library)
template <int MODE, class Ops>
emu_status run_pipelined(int dev, int sms, int m, int n, int k, float alpha, const float* A, int lda,
                         long long strideA, const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                         long long strideC, int batch, cudaStream_t s, int kblock, unsigned flags, const Ops& ops)
{
    const TsPlan t = ts_plan(MODE, m, n, k, batch, sms, false);
#define EMU_RUN_P(BN_, SC_, AS_, LK_)                                                                            \
    return run_gemm_pair_ts<MODE, 0, BN_, SC_, AS_, false, false, LK_, Ops>(                                     \
        dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, s, nullptr,    \
        kblock, flags, nullptr, nullptr, ops)
    if (t.as) EMU_RUN_P(128, true, true, false);
    if (t.lk) EMU_RUN_P(128, true, false, true);
    if (t.sc) EMU_RUN_P(128, true, false, false);
    if (t.n == 64) EMU_RUN_P(64, false, false, false);
    EMU_RUN_P(128, false, false, false);
#undef EMU_RUN_P
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* emu_status_string(emu_status s)
{
    switch (s) {
        case EMU_STATUS_SUCCESS: return "EMU_STATUS_SUCCESS";
        case EMU_STATUS_INVALID_VALUE: return "EMU_STATUS_INVALID_VALUE";
        case EMU_STATUS_NOT_SUPPORTED: return "EMU_STATUS_NOT_SUPPORTED";
        case EMU_STATUS_ARCH_MISMATCH: return "EMU_STATUS_ARCH_MISMATCH";
        case EMU_STATUS_LAUNCH_FAILED: return "EMU_STATUS_LAUNCH_FAILED";
        case EMU_STATUS_CUDA_ERROR: return "EMU_STATUS_CUDA_ERROR";
    }
    return "EMU_STATUS_UNKNOWN";
}

__attribute__((visibility("default"))) int emu_version(void) { return EMU_VERSION; }

__attribute__((visibility("default"))) int emu_last_launch_count(void) { return g_last_launches; }

__attribute__((visibility("default"))) const char* emu_last_kernel_name(void) { return g_last_kernel; }

// default combine interval KB (R#7): 64 up to k = 8192, doubled for every further
// factor 4 of k (128 up to 32768, ...).  With the measured tensor-core model the
// error at k = 16384 is 0.12x (FP16) / 0.17x (TF32) plain SGEMM at KB = 128 against
// 0.14x / 0.15x at 64 (tools/kb_accuracy.py): the cross-block FP32 additions
// dominate there, so the longer interval costs nothing in accuracy and halves the
// combine work
static int default_kblock(int k)
{
    int kb = 64;
    long long lim = 8192;
    while (k > lim && kb < 4096) {
        kb *= 2;
        lim *= 4;
    }
    return kb;
}

// the device entries; range_ws != nullptr selects the range-safe mode (R#22)

static emu_status gemm_impl(int m, int n, int k, float alpha, const float* A, int lda, long long strideA,
                            const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                            long long strideC, int batch, emu_split_mode mode, void* stream,
                            unsigned int* d_range_flag, int kblock, unsigned int flags, void* range_ws,
                            size_t range_ws_bytes, bool ta = false, bool tb = false)
{
    g_last_launches = 0;
    // ---- synchronous validation (C untouched on error) ----
    if (m < 0 || n < 0 || k < 0 || batch < 0) return EMU_STATUS_INVALID_VALUE;
    if (mode != EMU_SPLIT_FP16 && mode != EMU_SPLIT_TF32) return EMU_STATUS_INVALID_VALUE;
    if (lda < std::max(1, ta ? k : m) || ldb < std::max(1, tb ? n : k) || ldc < std::max(1, m))
        return EMU_STATUS_INVALID_VALUE;
    if (range_ws != nullptr && (ta || tb)) return EMU_STATUS_NOT_SUPPORTED;
    if (strideA < 0 || strideB < 0 || strideC < 0) return EMU_STATUS_INVALID_VALUE;
    if (kblock < 0 || (kblock > 0 && (kblock % 32 != 0 || kblock > 4096))) return EMU_STATUS_INVALID_VALUE;
    if (flags & ~EMU_FLAG_NO_CORRECTION) return EMU_STATUS_INVALID_VALUE;
    if (kblock == 0) kblock = default_kblock(k);
    if (m == 0 || n == 0 || batch == 0) return EMU_STATUS_SUCCESS;
    if (C == nullptr) return EMU_STATUS_INVALID_VALUE;
    if (batch > 1 && strideC < (long long)ldc * n) return EMU_STATUS_INVALID_VALUE;
    const bool reads_ab = k > 0 && alpha != 0.0f;
    if (reads_ab && (A == nullptr || B == nullptr)) return EMU_STATUS_INVALID_VALUE;
    const bool range = range_ws != nullptr;
    if (range && (!aligned16(range_ws) || range_ws_bytes < (size_t)4 * (size_t)batch * ((size_t)m + (size_t)n)))
        return EMU_STATUS_INVALID_VALUE;

    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

    if (!reads_ab) {
        const long long cols = (long long)n * batch;
        const unsigned grid = (unsigned)std::min<long long>(cols, 65535LL * 8);
        scale_c_kernel<<<grid, 256, 0, s>>>(C, m, n, ldc, strideC, batch, beta);
        g_last_launches = 1;
        return launch_status(cudaGetLastError());
    }
    // ---- TMA path when its alignment domain holds, else the direct-load path ----
    const bool tma_ok = aligned16(A) && aligned16(B) && lda % 4 == 0 && ldb % 4 == 0 &&
                        (batch <= 1 || strideA == 0 || strideA % 4 == 0) &&
                        (batch <= 1 || strideB == 0 || strideB % 4 == 0) &&
                        (unsigned long long)strideA * 4 < (1ull << 40) && (unsigned long long)strideB * 4 < (1ull << 40);
    static const int force_ldg = [] {
        const char* e = getenv("EMU_FORCE_LDG");   // testing/diagnostics only
        return e && strcmp(e, "1") == 0;
    }();
    const bool ldg = !tma_ok || force_ldg;
    const unsigned* row_max = nullptr;
    const unsigned* col_max = nullptr;
    if (range) {
        // range-safe mode: TS kernel only (any m); exponents from one max-|x| pass
        if (!tma_ok) return EMU_STATUS_NOT_SUPPORTED;
        unsigned* ws = static_cast<unsigned*>(range_ws);
        if (cudaMemsetAsync(ws, 0, (size_t)4 * batch * ((size_t)m + n), s) != cudaSuccess)
            return EMU_STATUS_CUDA_ERROR;
        const int a_blocks = (m + 255) / 256, b_blocks = (n + 7) / 8, ka = 16, kb = 512;
        const long long blocks = (long long)batch * ((long long)a_blocks * ((k + ka - 1) / ka) +
                                                     (long long)b_blocks * ((k + kb - 1) / kb));
        if (blocks > 0x7fffffffLL) return EMU_STATUS_NOT_SUPPORTED;
        const long long sAr = batch > 1 ? strideA : 0, sBr = batch > 1 ? strideB : 0;
        if (blocks > 0)
            range_max_kernel<<<(unsigned)blocks, 256, 0, s>>>(A, lda, sAr, B, ldb, sBr, m, n, k, a_blocks, b_blocks,
                                                               ka, kb, ws, ws + (size_t)batch * m);
        const emu_status ls = launch_status(cudaGetLastError());
        if (ls != EMU_STATUS_SUCCESS) return ls;
        row_max = ws;
        col_max = ws + (size_t)batch * m;
    }
    // CTA-pair kernel for problems with more than one 128-row block
    static const int kernel_pref = [] {
        const char* e = getenv("EMU_KERNEL");   // "single" | "pair" | "ts": tuning/diagnostics only
        if (e && strcmp(e, "single") == 0) return 1;
        if (e && strcmp(e, "pair") == 0) return 2;
        if (e && strcmp(e, "ts") == 0) return 3;
        return 0;
    }();
    // A-in-TMEM pair kernel (fewest shared-memory bytes per MMA) for every problem
    // with more than one 128-row block; the SMEM-operand pair kernel stays selectable
    // (EMU_KERNEL=pair) for comparison.
    if ((ta || tb) && !tma_ok) return EMU_STATUS_NOT_SUPPORTED;   // transposed operands: TS kernel only
    if (g_mdst && (!tma_ok || ldg)) return EMU_STATUS_NOT_SUPPORTED;   // multicast: TS kernel only (also under EMU_FORCE_LDG)
    const bool ts = !ldg && (range || ta || tb || g_mdst || kernel_pref == 3 || (kernel_pref == 0 && m > 128));
    const bool pair = !ldg && !ts && (kernel_pref == 2 || kernel_pref == 3 || (kernel_pref == 0 && m > 128));
    // tile width of the TS kernel (profiles/r01_summary.md): 128 with one accumulator
    // buffer whose D_corr and D_hi drains overlap the other part's MMAs (SPLITC); the
    // double-buffered 96-wide tile (EMU_TS_N=96) and the plain single buffer
    // (EMU_TS_SPLITC=0) stay selectable for comparison.
    const TsPlan plan = ts_plan(mode, m, n, k, batch, sms, g_mdst != nullptr);
    const int ts_n = plan.n;
    const bool ts_sc = plan.sc, ts_as = plan.as, ts_lk = plan.lk;
#define EMU_RUN_TS(MODE_, RANGE_)                                                                                      \
    do {                                                                                                               \
        if (ts_as)                                                                                                     \
            { rs = run_gemm_pair_ts<MODE_, RANGE_, 128, true, true>(dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, \
                                                                    strideB, beta, C, ldc, strideC, batch, s,          \
                                                                    d_range_flag, kblock, flags, row_max, col_max); break; }    \
        if (ts_lk)                                                                                                     \
            { rs = run_gemm_pair_ts<MODE_, RANGE_, 128, true, false, false, false, true>(dev, sms, m, n, k, alpha, A,  \
                                     lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, s, d_range_flag,     \
                                     kblock, flags, row_max, col_max); break; }                                        \
        if (ts_sc)                                                                                                     \
            { rs = run_gemm_pair_ts<MODE_, RANGE_, 128, true, false>(dev, sms, m, n, k, alpha, A, lda, strideA, B,     \
                                                                     ldb, strideB, beta, C, ldc, strideC, batch, s,    \
                                                                     d_range_flag, kblock, flags, row_max, col_max); break; }   \
        if (ts_n == 64)                                                                                                \
            { rs = run_gemm_pair_ts<MODE_, RANGE_, 64, false, false>(dev, sms, m, n, k, alpha, A, lda, strideA, B,     \
                                                                     ldb, strideB, beta, C, ldc, strideC, batch, s,    \
                                                                     d_range_flag, kblock, flags, row_max, col_max); break; }   \
        if (ts_n == 128)                                                                                               \
            { rs = run_gemm_pair_ts<MODE_, RANGE_, 128, false, false>(dev, sms, m, n, k, alpha, A, lda, strideA, B,    \
                                                                      ldb, strideB, beta, C, ldc, strideC, batch, s,   \
                                                                      d_range_flag, kblock, flags, row_max, col_max); break; }  \
        { rs = run_gemm_pair_ts<MODE_, RANGE_, 96, false, false>(dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb,    \
                                                                 strideB, beta, C, ldc, strideC, batch, s,             \
                                                                 d_range_flag, kblock, flags, row_max, col_max); break; }       \
    } while (0)
#define EMU_RUN_TT(MODE_, RANGE_, TA_, TB_)                                                                            \
    do {                                                                                                               \
        if (ts_as)                                                                                                     \
            rs = run_gemm_pair_ts<MODE_, RANGE_, 128, true, true, TA_, TB_>(                                           \
                dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, s,           \
                d_range_flag, kblock, flags, nullptr, nullptr);                                                        \
        else                                                                                                           \
            rs = run_gemm_pair_ts<MODE_, RANGE_, 128, true, false, TA_, TB_>(                                          \
                dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, s,           \
                d_range_flag, kblock, flags, nullptr, nullptr);                                                        \
    } while (0)
#define EMU_RUN_T3(MODE_, RANGE_)                                                                                      \
    do {                                                                                                               \
        if (ta && tb) EMU_RUN_TT(MODE_, RANGE_, true, true);                                                           \
        else if (ta) EMU_RUN_TT(MODE_, RANGE_, true, false);                                                           \
        else EMU_RUN_TT(MODE_, RANGE_, false, true);                                                                   \
    } while (0)
    if (ta || tb) {   // op(A) / op(B) transposed (NEXT row 2): split-commit TS kernel, 128-wide tiles
        emu_status rs;
        if (mode == EMU_SPLIT_FP16) {
            if (d_range_flag) EMU_RUN_T3(0, 1);
            else EMU_RUN_T3(0, 0);
        } else {
            EMU_RUN_T3(1, 0);
        }
        return rs;
    }
#undef EMU_RUN_T3
#undef EMU_RUN_TT
    if (ts) {
        // RANGE mask: 1 = the overflow flag code, 2 = the range-safe scaling; the plain
        // instantiations (the paper's method) carry neither
        emu_status rs;
        if (mode == EMU_SPLIT_FP16) {
            const int rmask = (d_range_flag ? 1 : 0) | (range ? 2 : 0);
            if (rmask == 3) EMU_RUN_TS(0, 3);
            else if (rmask == 2) EMU_RUN_TS(0, 2);
            else if (rmask == 1) EMU_RUN_TS(0, 1);
            else EMU_RUN_TS(0, 0);
        } else {
            if (range) EMU_RUN_TS(1, 2);
            else EMU_RUN_TS(1, 0);
        }
        if (range && rs == EMU_STATUS_SUCCESS) g_last_launches = 2;   // max-|x| pass + GEMM
        return rs;
    }
#undef EMU_RUN_TS
#define EMU_RUN_PAIR(MODE_, ALAY_, RANGE_)                                                                          \
    return run_gemm_pair<MODE_, ALAY_, RANGE_>(dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, \
                                               ldc, strideC, batch, s, d_range_flag, kblock, flags)
    if (pair) {
        if (mode == EMU_SPLIT_FP16) {
            if (d_range_flag) EMU_RUN_PAIR(0, emu::A_MN_SW128, true);
            EMU_RUN_PAIR(0, emu::A_MN_SW128, false);
        }
        EMU_RUN_PAIR(1, emu::A_K_SW128, false);
    }
#undef EMU_RUN_PAIR
#define EMU_RUN(MODE_, ALAY_, RANGE_, LDG_)                                                                         \
    return run_gemm<MODE_, ALAY_, RANGE_, LDG_>(dev, sms, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, \
                                                ldc, strideC, batch, s, d_range_flag, kblock, flags)
    if (mode == EMU_SPLIT_FP16) {
        if (d_range_flag) {
            if (ldg) EMU_RUN(0, emu::A_MN_SW128, true, true);
            EMU_RUN(0, emu::A_MN_SW128, true, false);
        }
        if (ldg) EMU_RUN(0, emu::A_MN_SW128, false, true);
        EMU_RUN(0, emu::A_MN_SW128, false, false);
    }
    static const bool tf32_mn = [] {
        const char* e = getenv("EMU_TF32_A_LAYOUT");   // tuning/diagnostics only
        return e && strcmp(e, "mn32") == 0;
    }();
    if (ldg) EMU_RUN(1, emu::A_K_SW128, false, true);
    if (tf32_mn) EMU_RUN(1, emu::A_MN_SW128_32B, false, false);
    EMU_RUN(1, emu::A_K_SW128, false, false);
#undef EMU_RUN
}

__attribute__((visibility("default"))) emu_status emu_sgemm_batched_ex(int m, int n, int k, float alpha, const float* A, int lda, long long strideA,
                                const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                                long long strideC, int batch, emu_split_mode mode, void* stream,
                                unsigned int* d_range_flag, int kblock, unsigned int flags)
{
    return gemm_impl(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, mode, stream,
                     d_range_flag, kblock, flags, nullptr, 0);
}

__attribute__((visibility("default"))) emu_status emu_sgemm_batched_t(char transa, char transb, int m, int n, int k, float alpha,
                               const float* A, int lda, long long strideA, const float* B, int ldb,
                               long long strideB, float beta, float* C, int ldc, long long strideC,
                               int batch, emu_split_mode mode, void* stream, unsigned int* d_range_flag,
                               int kblock, unsigned int flags)
{
    auto op = [](char t, bool& tr) {
        if (t == 'N' || t == 'n') { tr = false; return true; }
        if (t == 'T' || t == 't' || t == 'C' || t == 'c') { tr = true; return true; }
        return false;
    };
    bool ta = false, tb = false;
    g_last_launches = 0;
    if (!op(transa, ta) || !op(transb, tb)) return EMU_STATUS_INVALID_VALUE;
    return gemm_impl(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, mode, stream,
                     d_range_flag, kblock, flags, nullptr, 0, ta, tb);
}

// row-major storage (NEXT row 2): a row-major X with leading dimension ld is the
// column-major X^T with the same ld, so C = op(A) op(B) row-major is
// C^T = op(B)^T op(A)^T column-major -- the operands swap, the trans flags stay
__attribute__((visibility("default"))) emu_status emu_sgemm_batched_layout(
    emu_layout layout, char transa, char transb, int m, int n, int k, float alpha, const float* A, int lda,
    long long strideA, const float* B, int ldb, long long strideB, float beta, float* C, int ldc, long long strideC,
    int batch, emu_split_mode mode, void* stream, unsigned int* d_range_flag, int kblock, unsigned int flags)
{
    g_last_launches = 0;
    if (layout == EMU_COL_MAJOR)
        return emu_sgemm_batched_t(transa, transb, m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc,
                                   strideC, batch, mode, stream, d_range_flag, kblock, flags);
    if (layout != EMU_ROW_MAJOR) return EMU_STATUS_INVALID_VALUE;
    return emu_sgemm_batched_t(transb, transa, n, m, k, alpha, B, ldb, strideB, A, lda, strideA, beta, C, ldc,
                               strideC, batch, mode, stream, d_range_flag, kblock, flags);
}

__attribute__((visibility("default"))) size_t emu_range_workspace_size(int m, int n, int batch)
{
    if (m < 0 || n < 0 || batch < 0) return 0;
    return (size_t)4 * (size_t)batch * ((size_t)m + (size_t)n);
}

__attribute__((visibility("default"))) emu_status emu_sgemm_batched_range(int m, int n, int k, float alpha, const float* A, int lda,
                                   long long strideA, const float* B, int ldb, long long strideB, float beta,
                                   float* C, int ldc, long long strideC, int batch, emu_split_mode mode,
                                   void* stream, void* d_workspace, size_t workspace_bytes,
                                   unsigned int* d_range_flag, int kblock, unsigned int flags)
{
    if (d_workspace == nullptr) return EMU_STATUS_INVALID_VALUE;
    return gemm_impl(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch, mode, stream,
                     d_range_flag, kblock, flags, d_workspace, workspace_bytes);
}

__attribute__((visibility("default"))) emu_status emu_sgemm_batched(int m, int n, int k, float alpha, const float* A, int lda, long long strideA,
                             const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                             long long strideC, int batch, emu_split_mode mode, void* stream)
{
    return emu_sgemm_batched_ex(m, n, k, alpha, A, lda, strideA, B, ldb, strideB, beta, C, ldc, strideC, batch,
                                mode, stream, nullptr, 0, 0u);
}

__attribute__((visibility("default"))) emu_status emu_sgemm(int m, int n, int k, float alpha, const float* A, int lda, const float* B, int ldb, float beta,
                     float* C, int ldc, emu_split_mode mode, void* stream)
{
    return emu_sgemm_batched_ex(m, n, k, alpha, A, lda, 0, B, ldb, 0, beta, C, ldc, 0, 1, mode, stream, nullptr, 0,
                                0u);
}

__attribute__((visibility("default"))) emu_status emu_split(const float* x, long long count, emu_split_mode mode, void* hi, void* lo, void* stream)
{
    g_last_launches = 0;
    if (count < 0) return EMU_STATUS_INVALID_VALUE;
    if (mode != EMU_SPLIT_FP16 && mode != EMU_SPLIT_TF32) return EMU_STATUS_INVALID_VALUE;
    if (count == 0) return EMU_STATUS_SUCCESS;
    if (!x || !hi || !lo) return EMU_STATUS_INVALID_VALUE;
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 3u)
        return EMU_STATUS_INVALID_VALUE;
    if (mode == EMU_SPLIT_FP16 && (reinterpret_cast<uintptr_t>(x) & 7u)) return EMU_STATUS_NOT_SUPPORTED;
    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const unsigned grid = (unsigned)std::max(1, sms * 8);
    if (mode == EMU_SPLIT_FP16)
        split_fp16_kernel<<<grid, 256, 0, s>>>(x, count, static_cast<uint16_t*>(hi), static_cast<uint16_t*>(lo));
    else
        split_tf32_kernel<<<grid, 256, 0, s>>>(x, count, static_cast<uint32_t*>(hi), static_cast<uint32_t*>(lo));
    g_last_launches = 1;
    return launch_status(cudaGetLastError());
}

__attribute__((visibility("default"))) emu_status emu_sgemm_batched_host(int m, int n, int k, float alpha, const float* A, int lda, long long strideA,
                                  const float* B, int ldb, long long strideB, float beta, float* C, int ldc,
                                  long long strideC, int batch, emu_split_mode mode, void* stream)
{
    g_last_launches = 0;
    if (m < 0 || n < 0 || k < 0 || batch < 0) return EMU_STATUS_INVALID_VALUE;
    if (mode != EMU_SPLIT_FP16 && mode != EMU_SPLIT_TF32) return EMU_STATUS_INVALID_VALUE;
    if (lda < std::max(1, m) || ldb < std::max(1, k) || ldc < std::max(1, m)) return EMU_STATUS_INVALID_VALUE;
    if (strideA < 0 || strideB < 0 || strideC < 0) return EMU_STATUS_INVALID_VALUE;
    if (m == 0 || n == 0 || batch == 0) return EMU_STATUS_SUCCESS;
    if (C == nullptr) return EMU_STATUS_INVALID_VALUE;
    if (batch > 1 && strideC < (long long)ldc * n) return EMU_STATUS_INVALID_VALUE;
    const bool reads_ab = k > 0 && alpha != 0.0f;
    if (reads_ab && (A == nullptr || B == nullptr)) return EMU_STATUS_INVALID_VALUE;
    int dev = 0, sms = 0;
    emu_status st = device_check(dev, sms);
    if (st != EMU_STATUS_SUCCESS) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);

    // Problems are processed in chunks on two internal streams: the host->device
    // copy of chunk c+1 and the device->host copy of chunk c-1 overlap the kernel
    // of chunk c.  Device buffers mirror the host layout of one chunk; only the
    // m x k / k x n / m x n parts are copied (2-D copies), gaps are left alone.
    HostCtx& hc = g_host[dev];
    std::lock_guard<std::mutex> lk(hc.mu);
    if (!hc.init) {
        if (cudaStreamCreateWithFlags(&hc.st[0], cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&hc.st[1], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&hc.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&hc.join[0], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&hc.join[1], cudaEventDisableTiming) != cudaSuccess)
            return EMU_STATUS_CUDA_ERROR;
        hc.init = true;
    }
    auto span = [](long long ld, long long cols, long long rows, long long stride, int nb) {
        return (long long)(nb - 1) * stride + ld * (cols - 1) + rows;
    };
    auto copy = [](float* dst, const float* src, long long ld, long long cols, long long rows, long long stride, int nb,
                   cudaMemcpyKind kind, cudaStream_t cs) -> bool {
        if (nb == 1 || stride == ld * cols) {
            const long long h = (long long)nb * cols;
            if (ld == rows)   // contiguous: one linear copy
                return cudaMemcpyAsync(dst, src, (size_t)(h * rows * 4), kind, cs) == cudaSuccess;
            return cudaMemcpy2DAsync(dst, ld * 4, src, ld * 4, rows * 4, h, kind, cs) == cudaSuccess;
        }
        for (int i = 0; i < nb; ++i)
            if (cudaMemcpy2DAsync(dst + i * stride, ld * 4, src + i * stride, ld * 4, rows * 4, cols, kind, cs) !=
                cudaSuccess)
                return false;
        return true;
    };
    // chunks: the first chunk's upload and the last one's download are not overlapped; the c2
    // e2e step is PCIe-bound (~47 GB/s host->device), 8 / 16 / 32 chunks: 3.04 / 3.03 / 2.85 TF
    static const int chunks_env = env_int("EMU_HOST_CHUNKS", 8, 1, 64);   // tuning only
    const int nchunks = batch >= 2 * chunks_env ? chunks_env : (batch >= 16 ? 8 : 1);
    const int per = (batch + nchunks - 1) / nchunks;
    const bool shA = strideA == 0 || batch == 1, shB = strideB == 0 || batch == 1;
    const long long spanA = reads_ab ? span(lda, k, m, shA ? 0 : strideA, shA ? 1 : per) : 0;
    const long long spanB = reads_ab ? span(ldb, n, k, shB ? 0 : strideB, shB ? 1 : per) : 0;
    const long long spanC = span(ldc, n, m, strideC, per);
    const int nslot = nchunks > 1 ? 2 : 1;
    const size_t need = sizeof(float) * (size_t)((shA ? spanA : nslot * spanA) + (shB ? spanB : nslot * spanB) +
                                                 nslot * spanC + 64);
    if (hc.ws_bytes < need) {
        if (hc.ws) cudaFree(hc.ws);
        hc.ws = nullptr;
        hc.ws_bytes = 0;
        if (cudaMalloc((void**)&hc.ws, need) != cudaSuccess) return EMU_STATUS_CUDA_ERROR;
        hc.ws_bytes = need;
    }
    auto align16f = [](float* q) { return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(q) + 15) & ~uintptr_t(15)); };
    float* cur = hc.ws;
    float* dA = cur; cur = align16f(cur + (shA ? spanA : nslot * spanA));
    float* dB = cur; cur = align16f(cur + (shB ? spanB : nslot * spanB));
    float* dC = cur;
    bool ok = cudaEventRecord(hc.fork, s) == cudaSuccess && cudaStreamWaitEvent(hc.st[0], hc.fork, 0) == cudaSuccess &&
              cudaStreamWaitEvent(hc.st[1], hc.fork, 0) == cudaSuccess;
    if (ok && reads_ab && shA) ok = copy(dA, A, lda, k, m, 0, 1, cudaMemcpyHostToDevice, hc.st[0]);
    if (ok && reads_ab && shB) ok = copy(dB, B, ldb, n, k, 0, 1, cudaMemcpyHostToDevice, hc.st[0]);
    if (ok && nslot > 1 && (shA || shB)) {   // stream 1 must see the shared operands
        ok = cudaEventRecord(hc.join[0], hc.st[0]) == cudaSuccess &&
             cudaStreamWaitEvent(hc.st[1], hc.join[0], 0) == cudaSuccess;
    }
    int launches = 0;
    for (int c = 0; c < nchunks && ok && st == EMU_STATUS_SUCCESS; ++c) {
        const int b0 = c * per;
        const int nb = std::min(per, batch - b0);
        if (nb <= 0) break;
        const int slot = c % nslot;
        cudaStream_t cs = hc.st[slot];
        float* a = shA ? dA : dA + slot * spanA;
        float* bb = shB ? dB : dB + slot * spanB;
        float* cc = dC + slot * spanC;
        if (reads_ab && !shA) ok = ok && copy(a, A + (long long)b0 * strideA, lda, k, m, strideA, nb, cudaMemcpyHostToDevice, cs);
        if (reads_ab && !shB) ok = ok && copy(bb, B + (long long)b0 * strideB, ldb, n, k, strideB, nb, cudaMemcpyHostToDevice, cs);
        if (beta != 0.0f) ok = ok && copy(cc, C + (long long)b0 * strideC, ldc, n, m, strideC, nb, cudaMemcpyHostToDevice, cs);
        if (!ok) break;
        st = emu_sgemm_batched_ex(m, n, k, alpha, reads_ab ? a : nullptr, lda, shA ? 0 : strideA,
                                  reads_ab ? bb : nullptr, ldb, shB ? 0 : strideB, beta, cc, ldc, strideC, nb, mode,
                                  cs, nullptr, 0, 0u);
        launches += g_last_launches;
        if (st == EMU_STATUS_SUCCESS)
            ok = copy(C + (long long)b0 * strideC, cc, ldc, n, m, strideC, nb, cudaMemcpyDeviceToHost, cs);
    }
    for (int i = 0; i < nslot; ++i) {
        cudaEventRecord(hc.join[i], hc.st[i]);
        cudaStreamWaitEvent(s, hc.join[i], 0);
    }
    if (!ok && st == EMU_STATUS_SUCCESS) st = EMU_STATUS_CUDA_ERROR;
    if (cudaStreamSynchronize(s) != cudaSuccess && st == EMU_STATUS_SUCCESS) st = EMU_STATUS_CUDA_ERROR;
    g_last_launches = launches;
    return st;
}

#ifdef EMU_PROF
// profiling build only (tools/prof_roles.py): read and reset the role counters
__attribute__((visibility("default"))) int emu_prof_read(unsigned long long* host, int n)
{
    cudaDeviceSynchronize();
    return cudaMemcpyFromSymbol(host, emu::g_prof, sizeof(unsigned long long) * (n < 16 ? n : 16)) == cudaSuccess ? 0 : 1;
}
__attribute__((visibility("default"))) int emu_prof_reset(void)
{
    unsigned long long z[16] = {};
    unsigned int zc[emu::TRACE_ROLES] = {};
    if (cudaMemcpyToSymbol(emu::g_trace_cnt, zc, sizeof(zc)) != cudaSuccess) return 1;
    return cudaMemcpyToSymbol(emu::g_prof, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
// trace of CTA 0 since the last reset: host receives TRACE_N (t, ev) pairs and the
// per-role counts; returns the number of roles
__attribute__((visibility("default"))) int emu_trace_read(long long* host, unsigned int* counts)
{
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(counts, emu::g_trace_cnt, sizeof(unsigned int) * emu::TRACE_ROLES) != cudaSuccess)
        return -1;
    if (cudaMemcpyFromSymbol(host, emu::g_trace, sizeof(long long) * 2 * emu::TRACE_N) != cudaSuccess) return -1;
    return emu::TRACE_ROLES;
}
#endif

}  // extern "C"

extern "C" {

// one GEMM, result stored to several destinations (NEXT row 3: the epilogue of an
// n-sharded GEMM with its all-gather fused in)
__attribute__((visibility("default"))) emu_status emu_sgemm_multicast(
    int m, int n, int k, float alpha, const float* A, int lda, const float* B, int ldb, float* const* C_dst,
    int num_dst, int ldc, emu_split_mode mode, void* stream, int kblock, unsigned int flags)
{
    g_last_launches = 0;
    if (C_dst == nullptr || num_dst < 1 || num_dst > 8) return EMU_STATUS_INVALID_VALUE;
    MultiDst md;
    md.n = num_dst;
    for (int d = 0; d < num_dst; ++d) {
        if (C_dst[d] == nullptr) return EMU_STATUS_INVALID_VALUE;
        md.d[d] = C_dst[d];
    }
    struct Guard {
        explicit Guard(const MultiDst* p) { g_mdst = p; }
        ~Guard() { g_mdst = nullptr; }
    } guard(&md);
    // k == 0 / alpha == 0 quick path writes C_dst[0] only: route every destination through it
    if (k == 0 || alpha == 0.0f) {
        for (int d = 0; d < num_dst; ++d) {
            const emu_status st = gemm_impl(m, n, k, alpha, A, lda, 0, B, ldb, 0, 0.0f, C_dst[d], ldc, 0, 1, mode,
                                            stream, nullptr, kblock, flags, nullptr, 0);
            if (st != EMU_STATUS_SUCCESS) return st;
        }
        if (m > 0 && n > 0) g_last_launches = num_dst;
        return EMU_STATUS_SUCCESS;
    }
    return gemm_impl(m, n, k, alpha, A, lda, 0, B, ldb, 0, 0.0f, C_dst[0], ldc, 0, 1, mode, stream, nullptr, kblock,
                     flags, nullptr, 0);
}

}  // extern "C"

// device-level API users (include/emu_tcec.cuh): tcec GEMM, Householder, Givens, scan
#include "tcec_api.cuh"
