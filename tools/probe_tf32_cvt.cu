// Exhaustive device check: does cvt.rn.tf32.f32 (F2FP.TF32.F32.PACK_B) equal
// the integer RNE formula of split.cuh (bit-exact with the oracle, R#6) on all
// 2^32 inputs?  Prints mismatch counts per input class.
#include <cstdio>
#include <cstdint>
#include "../paper_2308_15152_b200/csrc/split.cuh"

__global__ void probe(unsigned long long* cnt, uint32_t* example)
{
    const uint64_t total = 1ull << 32;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = (uint32_t)i;
        uint32_t c;
        asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(c) : "f"(__uint_as_float(u)));
        const uint32_t r = emu::tf32_rn_bits(u);
        const uint32_t e = (u >> 23) & 0xff;
        const int cls = e == 0xff ? ((u & 0x7fffff) ? 3 : 2) : (e == 0 ? 1 : 0);
        bool ok = (c == r);
        if (cls == 3) ok = ((c & 0x7f800000u) == 0x7f800000u) && (c & 0x7fffffu);  // NaN-ness
        if (!ok) {
            atomicAdd(&cnt[cls], 1ull);
            example[cls] = u;
        }
        // also the lo part of the split: tf32(x - hi)
        const float x = __uint_as_float(u);
        uint32_t c2;
        asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(c2) : "f"(__fsub_rn(x, __uint_as_float(r))));
        const uint32_t r2 = emu::tf32_rn_bits(__float_as_uint(__fsub_rn(x, __uint_as_float(r))));
        bool ok2 = (c2 == r2) || (((c2 & 0x7f800000u) == 0x7f800000u) && (c2 & 0x7fffffu) && ((r2 & 0x7f800000u) == 0x7f800000u) && (r2 & 0x7fffffu));
        if (!ok2) atomicAdd(&cnt[4], 1ull);
    }
}

int main()
{
    unsigned long long* cnt;
    uint32_t* ex;
    cudaMallocManaged(&cnt, 8 * sizeof(unsigned long long));
    cudaMallocManaged(&ex, 8 * sizeof(uint32_t));
    for (int i = 0; i < 8; ++i) { cnt[i] = 0; ex[i] = 0; }
    probe<<<148 * 8, 256>>>(cnt, ex);
    cudaDeviceSynchronize();
    printf("{\"normal\": %llu, \"subnormal\": %llu, \"inf\": %llu, \"nan\": %llu, \"lo_part\": %llu, "
           "\"ex_normal\": \"0x%08x\", \"ex_sub\": \"0x%08x\", \"ex_inf\": \"0x%08x\", \"ex_nan\": \"0x%08x\"}\n",
           cnt[0], cnt[1], cnt[2], cnt[3], cnt[4], ex[0], ex[1], ex[2], ex[3]);
    return 0;
}
