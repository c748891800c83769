// ex2x2.cuh -- paired fp32 arithmetic (FFMA2 / FADD2, PTX f32x2) and a polynomial
// exp2 on the FMA pipe, so that the row-wise loss kernels can split their exponentials
// between the MUFU unit (16 results per clock per SM on sm_100) and the FMA pipe.
//
// ex2_poly<D>(x): 2^x = 2^j * 2^f with j = rint(x) (the 1.5*2^23 rounding trick) and
// f = x - j in [-1/2, 1/2]; 2^f by a degree-D polynomial whose coefficients minimise the
// maximum relative error on [-1/2, 1/2] with c0 = 1 (fit by linear programming, then
// rounded to fp32): D = 5 -> 6.8e-8 (2.2e-7 with fp32 Horner rounding, the accuracy
// of ex2.approx), D = 3 -> 1.0e-4 (enough for a bf16 result, half an ulp = 2.0e-3).
// 2^j is added to the exponent field: bits(t) << 23 == j << 23 (mod 2^32) since t's
// mantissa holds j + 2^22 and its upper bits shift out.  x is clamped to -127 first:
// -inf -> j = -127, f = 0, p = 1 -> exactly +0; results below 2^-126 are tiny
// denormals where ex2.approx.ftz gives 0 (both are far below any tolerance).
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace grpo {
namespace x2 {

__device__ __forceinline__ uint64_t pk(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(uint64_t r, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__host__ __device__ constexpr uint64_t splat(uint32_t bits) { return ((uint64_t)bits << 32) | bits; }

constexpr uint64_t kLog2e2 = splat(0x3FB8AA3Bu);     // log2(e) rounded to fp32

constexpr uint64_t kMagic2 = splat(0x4B400000u);     // 1.5 * 2^23
constexpr uint64_t kNegMagic2 = splat(0xCB400000u);  // -1.5 * 2^23
constexpr uint64_t kNegOne2 = splat(0xBF800000u);

// the bf16 pair of one 32-bit word as an fp32 pair (lo element in the low half)
__device__ __forceinline__ uint64_t bf_pair(uint32_t w) { return pk(bf_lo(w), bf_hi(w)); }

__device__ __forceinline__ uint64_t ex2_mufu(uint64_t a) {
    float x0, x1;
    upk(a, x0, x1);
    return pk(ex2(x0), ex2(x1));
}

template <int D>
__device__ __forceinline__ uint64_t ex2_poly(uint64_t a) {
    static_assert(D == 3 || D == 5, "degree 3 or 5");
    float x0, x1;
    upk(a, x0, x1);
    const uint64_t xc = pk(fmaxf(x0, -127.0f), fmaxf(x1, -127.0f));
    const uint64_t t = add2(xc, kMagic2);       // j + 1.5*2^23, j = rint(x)
    const uint64_t j = add2(t, kNegMagic2);     // j (exact)
    const uint64_t f = fma2(j, kNegOne2, xc);   // x - j in [-1/2, 1/2] (exact)
    uint64_t p;
    if (D == 5) {
        p = fma2(splat(0x3AAD0DDBu), f, splat(0x3C1E83B1u));
        p = fma2(p, f, splat(0x3D635EF3u));
        p = fma2(p, f, splat(0x3E75FCABu));
        p = fma2(p, f, splat(0x3F31720Eu));
    } else {
        p = fma2(splat(0x3D61512Eu), f, splat(0x3E780627u));
        p = fma2(p, f, splat(0x3F317AFDu));
    }
    p = fma2(p, f, splat(0x3F800000u));
    float p0, p1, t0, t1;
    upk(p, p0, p1);
    upk(t, t0, t1);
    return pk(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23)),
              __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23)));
}

// sum over U masked 8-element vectors of 2^(z*log2e - ref); K of the 4U bf16 pairs,
// evenly spread, go through the degree-5 polynomial, the rest through MUFU
template <int U, int K>
__device__ __forceinline__ float sum_exp2(const uint4 (&x)[U], float ref) {
    const uint64_t nref = pk(-ref, -ref);
    uint64_t acc0 = 0ull, acc1 = 0ull;
#pragma unroll
    for (int j = 0; j < U; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t arg = fma2(bf_pair(word_of(x[j], q)), kLog2e2, nref);
            const uint64_t e = ((j * 4 + q) * K) % (4 * U) < K ? ex2_poly<5>(arg) : ex2_mufu(arg);
            if (q & 1) acc1 = add2(acc1, e);
            else acc0 = add2(acc0, e);
        }
    }
    float lo, hi;
    upk(add2(acc0, acc1), lo, hi);
    return lo + hi;
}

// sign * 2^(z*log2e - ref) of one 8-element vector packed to bf16 (the gradient with the
// token scale folded into ref, rowwise.cuh); the first P pairs by the degree-3 polynomial
template <int P>
__device__ __forceinline__ uint4 grad_scaled(const uint4 &x, float ref, uint32_t sign) {
    const uint64_t nref = pk(-ref, -ref);
    uint32_t d[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint64_t arg = fma2(bf_pair(word_of(x, q)), kLog2e2, nref);
        const uint64_t e = q < P ? ex2_poly<3>(arg) : ex2_mufu(arg);
        float lo, hi;
        upk(e, lo, hi);
        d[q] = pack_bf16x2(lo, hi) ^ sign;
    }
    return make_uint4(d[0], d[1], d[2], d[3]);
}

}  // namespace x2
}  // namespace grpo
