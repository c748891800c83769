// rowwise.cuh -- per-batch math shared by the row-wise loss kernels (loss_aux.cu,
// loss_vp.cu): the log2-domain softmax partial of U 8-element vectors and the
// gradient s * 2^(z*log2e - lse2) of one vector packed to bf16.
#pragma once

#include "common.cuh"

namespace grpo {

template <int NT, int U>
struct RowwiseBatch {
    // log2-domain partial of U vectors (already loaded and masked)
    static __device__ __forceinline__ void reduce(const uint4 (&x)[U], float &a, float &s) {
        uint32_t mx2 = kBf16NegInfPair;
#pragma unroll
        for (int j = 0; j < U; ++j)
            mx2 = bmax2(bmax2(mx2, bmax2(x[j].x, x[j].y)), bmax2(x[j].z, x[j].w));
        const float va = log2_ref(fmaxf(bf_lo(mx2), bf_hi(mx2)));
        if (va == -INFINITY) return;
        float t0 = 0.f, t1 = 0.f, t2 = 0.f, t3 = 0.f;
#pragma unroll
        for (int j = 0; j < U; ++j) {
            t0 += ex2(fmaf(bf_lo(x[j].x), kLog2e, -va)) + ex2(fmaf(bf_hi(x[j].x), kLog2e, -va));
            t1 += ex2(fmaf(bf_lo(x[j].y), kLog2e, -va)) + ex2(fmaf(bf_hi(x[j].y), kLog2e, -va));
            t2 += ex2(fmaf(bf_lo(x[j].z), kLog2e, -va)) + ex2(fmaf(bf_hi(x[j].z), kLog2e, -va));
            t3 += ex2(fmaf(bf_lo(x[j].w), kLog2e, -va)) + ex2(fmaf(bf_hi(x[j].w), kLog2e, -va));
        }
        lse2_merge(a, s, va, (t0 + t1) + (t2 + t3));
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
        uint4 d;
        d.x = pack_bf16x2(ex2(fmaf(bf_lo(x.x), kLog2e, -g.ref)), ex2(fmaf(bf_hi(x.x), kLog2e, -g.ref))) ^ g.sign;
        d.y = pack_bf16x2(ex2(fmaf(bf_lo(x.y), kLog2e, -g.ref)), ex2(fmaf(bf_hi(x.y), kLog2e, -g.ref))) ^ g.sign;
        d.z = pack_bf16x2(ex2(fmaf(bf_lo(x.z), kLog2e, -g.ref)), ex2(fmaf(bf_hi(x.z), kLog2e, -g.ref))) ^ g.sign;
        d.w = pack_bf16x2(ex2(fmaf(bf_lo(x.w), kLog2e, -g.ref)), ex2(fmaf(bf_hi(x.w), kLog2e, -g.ref))) ^ g.sign;
        return d;
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
