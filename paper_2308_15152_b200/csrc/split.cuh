// split.cuh -- the operand split of Eqs. corr-1..corr-4
// and its TF32 variant (R#6), as register-level device functions.
// The same functions run inside the GEMM's splitter warps and in the
// emu_split export, so the bit-exact split test covers the GEMM's staging.
//
// FP16: hi = toFP16(x) (RNE, IEEE subnormals, overflow -> Inf: R#1, R#3, R#4)
//       lo = toFP16((x - toFP32(hi)) * 2^11)
//   cvt.rn.f16x2.f32 does both roundings; x - hi and the 2^11 scaling use the
//   _rn intrinsics so they can never be contracted into an FMA.
// TF32: hi = RNE_tf32(x), lo = RNE_tf32(x - hi), with the low 13 bits cleared
//   explicitly so the tensor core's treatment of them is irrelevant (R#6).
//   The hardware cvt.rn.tf32.f32 is used; tf32_rn_bits is the integer form it
//   was checked against.
#pragma once

#include <cstdint>

namespace emu {

// two floats -> packed binary16 pair, element x0 in the low half
__device__ __forceinline__ uint32_t f32x2_to_f16x2_rn(float x0, float x1)
{
    uint32_t h;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(x1), "f"(x0));
    return h;
}

__device__ __forceinline__ void f16x2_to_f32x2(uint32_t h, float& x0, float& x1)
{
    asm("{\n\t.reg .f16 a, b;\n\t"
        "mov.b32 {a, b}, %2;\n\t"
        "cvt.f32.f16 %0, a;\n\t"
        "cvt.f32.f16 %1, b;\n\t}"
        : "=f"(x0), "=f"(x1) : "r"(h));
}

// (x0 - h0, x1 - h1) * 2^11 on the packed FP32x2 pipe (FADD2, FMUL2): each lane
// is one IEEE binary32 operation with round-to-nearest, never contracted
__device__ __forceinline__ void sub_mul2048_f32x2(float x0, float x1, float h0, float h1, float& r0, float& r1)
{
    asm("{\n\t.reg .b64 a, b, d;\n\t"
        "mov.b64 a, {%2, %3};\n\t"
        "mov.b64 b, {%4, %5};\n\t"
        "sub.rn.f32x2 d, a, b;\n\t"
        "mov.b64 b, {%6, %6};\n\t"
        "mul.rn.f32x2 d, d, b;\n\t"
        "mov.b64 {%0, %1}, d;\n\t}"
        : "=f"(r0), "=f"(r1) : "f"(x0), "f"(x1), "f"(h0), "f"(h1), "f"(2048.0f));
}

// x - toFP32(h) for both halves of a packed binary16 pair with the mixed-precision
// FMA (fma.rn.f32.f16: h * (-1) + x, one FHFMA per element, no separate unpack).
// The exact difference x - h is representable, so this equals __fsub_rn(x, h).
__device__ __forceinline__ void sub_f16x2_from_f32x2(uint32_t h, float x0, float x1, float& r0, float& r1)
{
    asm("{\n\t.reg .f16 a, b, m;\n\t"
        "mov.b32 {a, b}, %2;\n\t"
        "mov.b16 m, 0xBC00;\n\t"
        "fma.rn.f32.f16 %0, a, m, %3;\n\t"
        "fma.rn.f32.f16 %1, b, m, %4;\n\t}"
        : "=f"(r0), "=f"(r1) : "r"(h), "f"(x0), "f"(x1));
}

// r0 *= s, r1 *= s with one packed FMUL2 (each product rounded exactly like __fmul_rn)
__device__ __forceinline__ void scale_f32x2(float& r0, float& r1, float s)
{
    asm("{\n\t.reg .b64 d, b;\n\t"
        "mov.b64 d, {%0, %1};\n\t"
        "mov.b64 b, {%2, %2};\n\t"
        "mul.rn.f32x2 d, d, b;\n\t"
        "mov.b64 {%0, %1}, d;\n\t}"
        : "+f"(r0), "+f"(r1) : "f"(s));
}

__device__ __forceinline__ void mul2048_f32x2(float& r0, float& r1)
{
    asm("{\n\t.reg .b64 d, b;\n\t"
        "mov.b64 d, {%0, %1};\n\t"
        "mov.b64 b, {%2, %2};\n\t"
        "mul.rn.f32x2 d, d, b;\n\t"
        "mov.b64 {%0, %1}, d;\n\t}"
        : "+f"(r0), "+f"(r1) : "f"(2048.0f));
}

// Eqs. corr-1/corr-2 for two elements: packed hi and packed lo (low half = x0).
// Per element: 1/2 F2FP (hi), 1 FHFMA (x - hi), 1/2 FMUL2 (* 2^11), 1/2 F2FP (lo).
__device__ __forceinline__ void split_fp16x2(float x0, float x1, uint32_t& hi, uint32_t& lo)
{
    hi = f32x2_to_f16x2_rn(x0, x1);
    float r0, r1;
    sub_f16x2_from_f32x2(hi, x0, x1, r0, r1);
    mul2048_f32x2(r0, r1);
    lo = f32x2_to_f16x2_rn(r0, r1);
}

// the earlier form (unpack hi to FP32, FADD2, FMUL2) -- kept for the tools' A/B
__device__ __forceinline__ void split_fp16x2_unpack(float x0, float x1, uint32_t& hi, uint32_t& lo)
{
    hi = f32x2_to_f16x2_rn(x0, x1);
    float h0, h1;
    f16x2_to_f32x2(hi, h0, h1);
    float r0, r1;
    sub_mul2048_f32x2(x0, x1, h0, h1, r0, r1);
    lo = f32x2_to_f16x2_rn(r0, r1);
}

// combine step on two accumulator columns at once (R#8):
//   t = RN(d_corr * scale + d_hi)  (one rounding: the FMA of Eq. corr-5's sum)
//   c = RN(c + t)
// on the packed FP32x2 pipe (FFMA2, FADD2), lane-wise identical to fmaf / __fadd_rn
__device__ __forceinline__ void combine2(float& c0, float& c1, float hi0, float hi1, float co0, float co1, float scale)
{
    asm("{\n\t.reg .b64 h, k, s, t, c;\n\t"
        "mov.b64 h, {%2, %3};\n\t"
        "mov.b64 k, {%4, %5};\n\t"
        "mov.b64 s, {%6, %6};\n\t"
        "fma.rn.f32x2 t, k, s, h;\n\t"
        "mov.b64 c, {%0, %1};\n\t"
        "add.rn.f32x2 c, c, t;\n\t"
        "mov.b64 {%0, %1}, c;\n\t}"
        : "+f"(c0), "+f"(c1) : "f"(hi0), "f"(hi1), "f"(co0), "f"(co1), "f"(scale));
}

// four elements: (x0, x1) -> h01/l01, (x2, x3) -> h23/l23
__device__ __forceinline__ void split_fp16x2x2(float x0, float x1, float x2, float x3, uint32_t& h01,
                                               uint32_t& h23, uint32_t& l01, uint32_t& l23)
{
    split_fp16x2(x0, x1, h01, l01);
    split_fp16x2(x2, x3, h23, l23);
}

// 1 if either binary16 half of `h` is +-Inf or NaN (exponent field all ones)
__device__ __forceinline__ uint32_t f16x2_nonfinite(uint32_t h)
{
    const uint32_t e = h & 0x7c007c00u;
    return ((e & 0xffffu) == 0x7c00u) | ((e >> 16) == 0x7c00u);
}

// binary32 -> TF32 (RNE at fraction bit 13); Inf stays Inf, NaN stays a quiet NaN
__device__ __forceinline__ uint32_t tf32_rn_bits(uint32_t u)
{
    const uint32_t r = (u + 0xfffu + ((u >> 13) & 1u)) & 0xffffe000u;
    const bool special = (u & 0x7f800000u) == 0x7f800000u;
    const uint32_t s = (u & 0x7fffffu) ? ((u | 0x400000u) & 0xffffe000u) : u;
    return special ? s : r;
}

// cvt.rn.tf32.f32 (one F2FP.TF32.F32.PACK_B) -- verified on a B200 to equal
// tf32_rn_bits on all 2^32 inputs (tools/probe_tf32_cvt.cu, NaN by NaN-ness)
__device__ __forceinline__ uint32_t tf32_rn_cvt(float x)
{
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo)
{
    hi = tf32_rn_cvt(x);
    lo = tf32_rn_cvt(__fsub_rn(x, __uint_as_float(hi)));
}

}  // namespace emu
