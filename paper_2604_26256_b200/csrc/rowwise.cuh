// rowwise.cuh -- per-batch math shared by the row-wise loss kernels (loss_aux.cu,
// loss_vp.cu): the log2-domain softmax partial of U 8-element vectors and the
// gradient s * 2^(z*log2e - lse2) of one vector packed to bf16.
#pragma once

#include "common.cuh"
#include "ex2x2.cuh"

namespace grpo {

template <int NT, int U>
struct RowwiseBatch {
    // sum of 2^(z*log2e - ref) over U vectors (already loaded and masked): paired fp32
    // arithmetic (FFMA2 / FADD2), every exponential on MUFU.  x2::sum_exp2<U, K> can move
    // K pairs to the FMA-pipe polynomial instead: +2.5 % for a single K3c launch, but
    // -0.6 % in the sustained, power-capped loop (a polynomial exponential costs more
    // energy than a MUFU one), so K = 0
    static __device__ __forceinline__ float sum_exp2(const uint4 (&x)[U], float ref) {
        return x2::sum_exp2<U, 0>(x, ref);
    }
    // log2-domain partial of U vectors (already loaded and masked) into (a, s): a is the
    // running max of the thread's elements (bf16 max of the batch, 16 HMNMX2 per 32
    // elements), rounded up into log2 units, so every exponent is <= 0 and the terms that
    // dominate the row's sum have exponents near 0, where fp32 rounds them finely.  (A
    // lazy reference -- the first batch's max, raised only on overflow -- saved the max
    // reduction but left the row's top elements exponents of +10..+20 against a thread's
    // first-batch max on LM-like rows, whose fp32 rounding cost logp 3e-7.)
    // The running sum s is fp64: each 32-element batch sum (fp32) is added with one DADD.
    static __device__ __forceinline__ void reduce(const uint4 (&x)[U], float &a, double &s) {
        uint32_t mx2 = kBf16NegInfPair;
#pragma unroll
        for (int j = 0; j < U; ++j)
            mx2 = bmax2(bmax2(mx2, bmax2(x[j].x, x[j].y)), bmax2(x[j].z, x[j].w));
        // the new reference (integer-valued) and the exact power-of-two rescale of the sum so
        // far, branch-free: a warp's lanes raise their maxima in different batches, and a
        // divergent rescale block would run for the whole warp in nearly every batch
        const float va = fmaxf(a, log2_ref(fmaxf(bf_lo(mx2), bf_hi(mx2))));
        s = scale_pow2(s, a - va);  // a = va: s unchanged; a = -inf: s (= 0) stays 0
        a = va;
        // with a = -inf every element so far is -inf: reference 0 keeps the terms 0
        s += (double)sum_exp2(x, a == -INFINITY ? 0.0f : a);
    }
    // reduce of the first k vectors only (1 <= k <= U, the same k across the warp): a ragged
    // last chunk's batches past the row's end cost nothing
    static __device__ __forceinline__ void reduce_first(const uint4 (&x)[U], int k, float &a, double &s) {
        if constexpr (U == 1) {
            reduce(x, a, s);
        } else {
            if (k >= U) {
                reduce(x, a, s);
                return;
            }
            uint4 y[U - 1];
#pragma unroll
            for (int j = 0; j < U - 1; ++j) y[j] = x[j];
            RowwiseBatch<NT, U - 1>::reduce_first(y, k, a, s);
        }
    }
    // s * 2^(z*log2e - lse2) = sign(s) * 2^(z*log2e - (lse2 - log2|s|)): the token scale
    // folds into the exponent's reference, so an element costs one FFMA and one EX2 (no
    // FMUL) and the sign is applied to the packed bf16 pair
    struct GradRef {
        float ref;
        uint32_t sign;
    };
    static __device__ __forceinline__ GradRef grad_ref(float sc, float lse2) {
        return GradRef{lse2 - log2f(fabsf(sc)), sc < 0.0f ? 0x80008000u : 0u};
    }
    static __device__ __forceinline__ uint4 grad_scaled(const uint4 &x, const GradRef &g) {
        return x2::grad_scaled<0>(x, g.ref, g.sign);
    }
    // s * 2^(z*log2e - lse2) for the 8 elements of one vector, packed to bf16
    static __device__ __forceinline__ uint4 grad(const uint4 &x, float sc, float lse2) {
        uint4 d;
        d.x = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.x), kLog2e, -lse2)),
                          sc * ex2(fmaf(bf_hi(x.x), kLog2e, -lse2)));
        d.y = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.y), kLog2e, -lse2)),
                          sc * ex2(fmaf(bf_hi(x.y), kLog2e, -lse2)));
        d.z = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.z), kLog2e, -lse2)),
                          sc * ex2(fmaf(bf_hi(x.z), kLog2e, -lse2)));
        d.w = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.w), kLog2e, -lse2)),
                          sc * ex2(fmaf(bf_hi(x.w), kLog2e, -lse2)));
        return d;
    }
};

}  // namespace grpo
