// common.cuh -- sm_100a PTX helpers and shared declarations of the GRPO-async
// CUDA path (mbarrier, 1-D bulk TMA, cluster/DSMEM, bf16 packing, MUFU ex2).
// Product code: shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "grpo_async.h"

namespace grpo {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr uint32_t kBf16NegInfPair = 0xFF80FF80u;

// Per-row metadata staged by the row-info kernel (16 bytes, one vector load).
struct __align__(16) RowInfo {
    int32_t target;   // y_t (validated to be in [0, V))
    float logp_w;     // log pi_{w_j}(y_t)
    float adv;        // A_i of the row's trajectory
    float inv_norm;   // 1 / (P * G_p * L_i)
};

// A log2-domain softmax partial: the sum s of 2^(z*log2e - a) over a part of a row, with
// s in fp64 (16 bytes, one st.async / 128-bit shared access).
struct __align__(16) RowPart {
    float a;
    float pad;
    double s;
};

// A shard's partial of one row as 16 bytes (vocabulary- and tensor-parallel exchanges):
// (a, z_y, s fp64 with "this shard holds y_t" in its sign bit; s >= 0 otherwise).
__host__ __device__ __forceinline__ float4 pack_shard_part(float a, double s, float zy, bool holds) {
    unsigned long long sb;
    memcpy(&sb, &s, 8);
    sb |= holds ? (1ull << 63) : 0ull;
    float4 v;
    v.x = a;
    v.y = zy;
    memcpy(&v.z, &sb, 8);
    return v;
}
__host__ __device__ __forceinline__ void unpack_shard_part(const float4 &v, float &a, double &s, float &zy,
                                                           bool &holds) {
    unsigned long long sb;
    memcpy(&sb, &v.z, 8);
    holds = (sb >> 63) != 0ull;
    sb &= ~(1ull << 63);
    memcpy(&s, &sb, 8);
    a = v.x;
    zy = v.y;
}

// Per-row flags written by the loss kernels (workspace, one byte per row).
enum : uint8_t { kRowClipped = 1, kRowActive = 2 };

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init_cluster() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "r"(bytes)
        : "memory");
}

// Wait for the completion of the phase with the given parity (CTA-local producers).
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0u;
}

// Wait for the phase; a phase that never completes (a protocol bug) traps after ~2^26
// hardware-suspended retries (tens of seconds) instead of hanging the GPU.  Four probes per
// trip round the loop: a waiting warp issues ~2.5 instead of 6 instructions per probe (the
// K3c consumers' waits were ~10 % of the kernel's executed instructions).
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait(a, parity)) return;
    for (uint32_t spins = 0;; ++spins) {
        if (mbar_try_wait(a, parity) || mbar_try_wait(a, parity) || mbar_try_wait(a, parity) ||
            mbar_try_wait(a, parity))
            return;
        if (spins == (1u << 24)) __trap();
    }
}

// The same for a warp that has nothing else to do while it waits (the ring's producer, the
// epilogue warp): after each failed try_wait it sleeps `ns` nanoseconds, so its polling takes
// fewer issue slots from the consumer warps of its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t ns) {
    const uint32_t a = smem_u32(bar);
    uint32_t spins = 0;
    while (!mbar_try_wait(a, parity)) {
        __nanosleep(ns);
        if (++spins == (1u << 26)) __trap();  // see mbar_wait
    }
}

// Same, with cluster-scope acquire (the phase is completed by peer CTAs' st.async).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t spins = 0;
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
        if (ok) return;
        if (++spins == (1u << 26)) __trap();  // see mbar_wait
    }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Ask the TMA engine to bring [src, src + bytes) into L2 (bytes % 16 == 0).
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// 1-D bulk TMA global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 1-D bulk copy shared -> global (bytes % 16 == 0, both 16-byte aligned), in the issuing
// thread's bulk group, with an L2 eviction-priority policy
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(policy)
                 : "memory");
}

// arrive `count` times at once (release, CTA scope)
__device__ __forceinline__ void mbar_arrive_count(uint64_t *bar, uint32_t count) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
        "r"(count)
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}

__device__ __forceinline__ uint32_t ncluster_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

// Shared-memory address of the same variable in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

// 16-byte remote store that completes 16 bytes of transaction on the remote mbarrier.
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t rbar, float a, float b,
                                            float c, float d) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, "
        "[%5];" ::"r"(raddr),
        "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)),
        "r"(__float_as_uint(d)), "r"(rbar)
        : "memory");
}

// 8-byte remote store completing 8 bytes of transaction on the remote mbarrier.
__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint32_t rbar, float a, float b) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(
            raddr),
        "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(rbar)
        : "memory");
}

// A RowPart (16 bytes) stored into a peer CTA's shared memory, completing 16 bytes of
// transaction on its mbarrier.
__device__ __forceinline__ void st_async_part(uint32_t raddr, uint32_t rbar, float a, double s) {
    const unsigned long long sb = (unsigned long long)__double_as_longlong(s);
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, "
        "[%5];" ::"r"(raddr),
        "r"(__float_as_uint(a)), "r"(0u), "r"((uint32_t)sb), "r"((uint32_t)(sb >> 32)), "r"(rbar)
        : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 128-bit global load, L1 bypassed, with an L2 eviction-priority policy
// (evict_first for read-once streams, evict_last for a row re-read from L2).
__device__ __forceinline__ uint4 ldg_policy(const void *p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}

// Streaming 128-bit global store (written once, not re-read by this kernel).
__device__ __forceinline__ void stg_stream(void *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Two exp2 in one MUFU op on a packed bf16x2 argument (bf16 results).
__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
    uint32_t y;
    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

__device__ __forceinline__ uint32_t mul_bf16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ uint32_t bmax2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// Round-to-nearest-even pack of two floats into bf16x2 (lo in the low half).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}

__device__ __forceinline__ uint16_t f2bf(float x) {
    return static_cast<uint16_t>(pack_bf16x2(x, 0.0f) & 0xFFFFu);
}

__device__ __forceinline__ uint32_t word_of(const uint4 &x, int q) {
    return q == 0 ? x.x : (q == 1 ? x.y : (q == 2 ? x.z : x.w));
}

// Set the bf16 elements e >= valid of an 8-element vector to -inf (ragged row tail).
__device__ __forceinline__ uint4 mask_tail(uint4 x, int valid) {
    const uint32_t lo_inf = 0x0000FF80u, hi_inf = 0xFF800000u;
    x.x = (valid <= 0 ? (x.x & 0xFFFF0000u) | lo_inf : x.x);
    x.x = (valid <= 1 ? (x.x & 0x0000FFFFu) | hi_inf : x.x);
    x.y = (valid <= 2 ? (x.y & 0xFFFF0000u) | lo_inf : x.y);
    x.y = (valid <= 3 ? (x.y & 0x0000FFFFu) | hi_inf : x.y);
    x.z = (valid <= 4 ? (x.z & 0xFFFF0000u) | lo_inf : x.z);
    x.z = (valid <= 5 ? (x.z & 0x0000FFFFu) | hi_inf : x.z);
    x.w = (valid <= 6 ? (x.w & 0xFFFF0000u) | lo_inf : x.w);
    x.w = (valid <= 7 ? (x.w & 0x0000FFFFu) | hi_inf : x.w);
    return x;
}

// Store the first `valid` bf16 elements of an 8-element vector, one 2-byte store each.
__device__ __forceinline__ void store_tail(uint16_t *dst, const uint4 &d, int valid) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        if (e < valid) {
            const uint32_t w = word_of(d, e >> 1);
            dst[e] = (uint16_t)((e & 1) ? (w >> 16) : (w & 0xFFFFu));
        }
    }
}

// Softmax partials live in the log2 domain: a partial (a, s) stands for
// s * 2^a, i.e. a = a reference point in units of log2(e)*z and
// s = sum_v 2^(z_v*log2e - a).  A thread takes a = m*log2e rounded UP
// (__fmul_ru) so that every exponent z*log2e - a it feeds to ex2 is <= 0
// (no overflow for any finite logit) and the per-element exponent is one FFMA.
// The same reference is used when partials merge and when the backward
// recomputes p = 2^(z*log2e - lse2), so forward and backward agree exactly.
// The reference is also rounded up to an INTEGER, so that every rescale between two partials,
// 2^(a - b), is an exact power of two applied to the fp64 sum's exponent field (scale_pow2): no
// MUFU, no conversion, no rounding, and no lane-divergent fp64 multiply in the hot loop.  The
// row's largest element then has an exponent in (-1, 0], where fp32 still rounds it finely.
__device__ __forceinline__ float log2_ref(float m) {
    return m == -INFINITY ? -INFINITY : ceilf(__fmul_ru(m, kLog2e));
}

// s * 2^k for an integer-valued k <= 0 (a difference of two log2_ref references), exactly, by
// exponent arithmetic on the fp64 bits; 0 when the result would leave the normal range (or
// k = -inf, s = 0)
__device__ __forceinline__ double scale_pow2(double s, float k) {
    if (!(k > -2000.0f)) return 0.0;
    const long long b = __double_as_longlong(s);
    const int e = (int)((b >> 52) & 0x7FF);
    const int kk = (int)k;
    return e + kk > 0 ? __longlong_as_double(b + ((long long)kk << 52)) : 0.0;
}

// Merge (a, s) with (b, t).  Symmetric in its two arguments bit for bit, so
// butterfly reductions leave every lane with the identical result.
__device__ __forceinline__ void lse2_merge(float &a, float &s, float b, float t) {
    const float mn = fmaxf(a, b);
    if (mn == -INFINITY) {
        a = mn;
        s = 0.0f;
        return;
    }
    s = s * ex2(a - mn) + t * ex2(b - mn);
    a = mn;
}

__device__ __forceinline__ void warp_lse2_allreduce(float &a, float &s) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float b = __shfl_xor_sync(0xFFFFFFFFu, a, off);
        const float t = __shfl_xor_sync(0xFFFFFFFFu, s, off);
        lse2_merge(a, s, b, t);
    }
}

// Warp-wide (all lanes get the identical result: max and + are commutative,
// so both partners of every butterfly step compute the same bits).
__device__ __forceinline__ float warp_max_all(float x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x = fmaxf(x, __shfl_xor_sync(0xFFFFFFFFu, x, off));
    return x;
}
__device__ __forceinline__ float warp_sum_all(float x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, off);
    return x;
}
// Combine log2-domain partials (a, s) of the 32 lanes: one max reduction,
// one rescale per lane, one sum reduction.
__device__ __forceinline__ void warp_lse2_combine(float &a, float &s) {
    const float amax = warp_max_all(a);
    s = (amax == -INFINITY) ? 0.0f : s * ex2(a - amax);
    s = warp_sum_all(s);
    a = amax;
}

// The same with the sums held in fp64 (the row-wise kernels accumulate every thread's
// batch sums in fp64, so a row's sum carries no fp32 rounding beyond the 32-element
// batches).  The rescale factors 2^(a - amax) are exact powers of two
// (integer references, scale_pow2); the fp64 sums run in a fixed butterfly, so every lane
// holds identical bits.
__device__ __forceinline__ double warp_sum_all(double x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, off);
    return x;
}
__device__ __forceinline__ void warp_lse2_combine(float &a, double &s) {
    const float amax = warp_max_all(a);
    s = (amax == -INFINITY) ? 0.0 : scale_pow2(s, a - amax);
    s = warp_sum_all(s);
    a = amax;
}
// Merge (a, s) with (b, t), fp64 sums; symmetric in its arguments like lse2_merge.
__device__ __forceinline__ void lse2_merge(float &a, double &s, float b, double t) {
    const float mn = fmaxf(a, b);
    if (mn == -INFINITY) {
        a = mn;
        s = 0.0;
        return;
    }
    s = scale_pow2(s, a - mn) + scale_pow2(t, b - mn);
    a = mn;
}

// Per-row epilogue of eq:grpo_async / eq:ratio_async:
// r = exp(logp - logp_w), term = min(r A, clip(r) A), clipped iff the clip
// branch binds strictly, s = grad_scale * inv_norm * A * r * !clipped.
struct RowOut {
    double r, term;
    float s;
    float gy;  // the target's own gradient entry s (p_y - 1) = s expm1(logp), from fp64
    uint8_t flags;
};

// log2(e) = kLog2eHi + kLog2eLo to 1.7e-13: the high part has 16 significant bits, so
// fma(z, kLog2eLo, fma(z, kLog2eHi, -M)) is z*log2(e) - M rounded once at its own magnitude
// (the LM-head epilogue, whose fp32 logits have free issue slots, uses it)
constexpr float kLog2eHi = 1.44268798828125f;
constexpr float kLog2eLo = 7.0526075e-06f;

// log2 of a row's sum from the sum the row-wise kernels form with one FFMA per element,
//   S' = sum_v 2^(z_v*fl32(log2 e) - M),  fl32(log2 e) = log2(e) (1 - 1.34e-8):
// each term carries 2^(-z_v*(log2 e - fl32(log2 e))), i.e. S' = S * 2^(-(log2 e - fl32)*E_p[z])
// with S the exact sum.  The reference M = fl32(m*fl32(log2 e)) (m the row max, rounded up)
// carries the part E_p[z] ~ m of it, so
//   log2 S = log2 S' + M * (log2 e / fl32(log2 e) - 1)  (+ the residual 1.34e-8 * E_p[z - m]),
// which leaves logp an error of 1.34e-8 * |E_p[z - m]| (<= 1e-7 for any row whose
// probability mass lies within 7 nats of its max) instead of 1.34e-8 * |E_p[z]| -- 1.3e-4
// for logits near 1e4 (Z23).  fp64 throughout.
__device__ __forceinline__ double row_l2s(double s, float M) {
    const double kRatioM1 = 1.4426950408889634074 / (double)kLog2e - 1.0;
    return log2(s) + (double)M * kRatioM1;
}

// logp_t = z_y - lse from the row's log2-domain reference M and l2s = log2 of its sum
// S = sum_v 2^(z_v*log2e - M):
//   lse = (M + l2s) * ln2,  logp = z_y - lse,
// all in fp64 (a few DFMA per row) so that neither the fp32 rounding of lse nor that of
// M*ln2 reaches logp; the ratio r = exp(logp - logp_w) then carries only the error of S.
__device__ __forceinline__ double row_logp(float zy, float M, double l2s) {
    const double kLn2D = 0.69314718055994530942;
    return (double)zy - ((double)M + l2s) * kLn2D;
}

// eq:grpo_async / eq:ratio_async per token, in fp64 like the oracle (oracle_token_asym):
// the clip bounds are 1 -/+ the widened float eps, term = min(rA, clip(r)A) stays fp64 to
// the segmented sums, s = grad_scale * inv_norm * A * r is rounded to fp32 once.  A row
// with A == 0 or inv_norm == 0 (an all-equal group, a masked trajectory, a padding row
// outside cu_seqlens) gets s = 0 outright, and a row with A == 0 term = 0, so an infinite
// ratio there (logp_w = -inf on a padding row) cannot turn into 0 * inf = NaN.
__device__ __forceinline__ RowOut row_epilogue(double logp, const RowInfo &ri, float eps_lo,
                                               float eps_hi, float grad_scale) {
    RowOut o;
    const double r = exp(logp - (double)ri.logp_w);
    const double lo = 1.0 - (double)eps_lo, hi = 1.0 + (double)eps_hi;
    const double c = fmin(fmax(r, lo), hi);
    const double A = (double)ri.adv;
    const bool dead = ri.adv == 0.0f || ri.inv_norm == 0.0f;
    o.r = r;
    o.term = ri.adv == 0.0f ? 0.0 : fmin(r * A, c * A);  // a masked row keeps its term
    const bool clipped = (A > 0.0 && r > hi) || (A < 0.0 && r < lo);
    const double sd = (clipped || dead) ? 0.0 : (double)grad_scale * (double)ri.inv_norm * A * r;
    o.s = (float)sd;
    // p_y - 1 = expm1(logp) in fp64: a nearly certain target (p_y -> 1) keeps the relative
    // accuracy of logp instead of the fp32 resolution of 1 - ex2(z_y - lse2) (Z24)
    o.gy = (float)(sd * expm1(logp));
    o.flags = (clipped ? kRowClipped : 0) | ((!clipped && !dead) ? kRowActive : 0);
    return o;
}

// ------------------------------------------------------------ host launchers
// All return cudaGetLastError() of their launch; `launches` counts kernels.
struct LossArgs {
    const uint16_t *logits;
    uint16_t *dlogits;
    int64_t ld;
    int32_t V;
    int64_t row_begin;
    int64_t n_rows;
    const int64_t *target_ids;
    const float *logp_behav;
    const int64_t *cu_seqlens;
    int32_t N;
    const int32_t *traj_index;
    const float *adv;
    const float *inv_norm;
    float eps_lo, eps_hi;   // clip range [1 - eps_lo, 1 + eps_hi]
    float grad_scale;
    float *logp_out;
    float *lse_out;
    float *scale_out;
    double *traj_sum;
    double *stats;
    // workspace carve-up
    RowInfo *rowinfo;      // [n_rows]
    double *term_ws;       // [n_rows] (fp64: term_t reaches the segmented sums unrounded)
    float *logp_ws;        // [n_rows]
    uint8_t *flag_ws;      // [n_rows]
    double *part_ws;       // [N * 5]
};

cudaError_t launch_rowinfo(const LossArgs &a, cudaStream_t s, int *launches);
cudaError_t launch_group_partials(const float *rewards, const int32_t *group_ids, const int64_t *cu,
                                  int32_t N, int32_t P, const uint8_t *traj_mask, double *part,
                                  cudaStream_t s, int *launches);
cudaError_t launch_group_sq(const float *rewards, const int32_t *group_ids, int32_t N, int32_t P,
                            const double *glob, double *ss, cudaStream_t s, int *launches);
cudaError_t launch_advantage_from_stats(const float *rewards, const int32_t *group_ids, const int64_t *cu,
                                        int32_t N, int32_t P, float std_floor, int32_t norm,
                                        int32_t unbiased, const uint8_t *traj_mask, const double *glob,
                                        const double *ss, float *adv, float *inv_norm, cudaStream_t s,
                                        int *launches);
cudaError_t launch_fused_rowwise(const LossArgs &a, const grpo_tune_t *tune, cudaStream_t s,
                                 int *launches, grpo_plan_t *plan);
cudaError_t launch_segment_reduce(const LossArgs &a, cudaStream_t s, int *launches);
cudaError_t launch_fused_stream(const LossArgs &a, const grpo_tune_t *tune, cudaStream_t s, int *launches,
                                grpo_plan_t *plan, char *why, size_t why_len);
int32_t lmhead_n_split(int64_t n_rows, int32_t V);
cudaError_t launch_lmhead(int epi, const void *X, const void *W, int64_t n_rows, int32_t d, int32_t V,
                          const RowInfo *rowinfo, RowPart *part, float *zy, uint16_t *out, int64_t ld_out,
                          const int64_t *targets, const float *lse, const float *scale, float mult,
                          cudaStream_t s, int *launches, grpo_plan_t *plan, char *why, size_t why_len,
                          int cta_group, int32_t col_offset = 0);
cudaError_t launch_lmhead_rowpart(const RowPart *part, const float *zy, int32_t n_split, int64_t n_rows,
                                  const int64_t *targets, int32_t col_offset, int32_t Vs, float4 *out,
                                  cudaStream_t s, int *launches);
cudaError_t launch_lmhead_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W, int64_t n_rows, int32_t d,
                             int32_t Vs, int32_t world, int32_t rank, float *const *slots, cudaStream_t s,
                             int *launches, char *why, size_t why_len);
cudaError_t launch_lmhead_gemm_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W, int64_t n_rows,
                                  int32_t d, int32_t V, void *out, int out_bf16, cudaStream_t s, int *launches,
                                  char *why, size_t why_len);
cudaError_t launch_lmhead_gemm_dw(const uint16_t *dz, int64_t ld_dz, const uint16_t *X, int64_t n_rows,
                                  int32_t d, int32_t V, float *dW, cudaStream_t s, int *launches, char *why,
                                  size_t why_len);
cudaError_t launch_lmhead_dx_reduce(const float *own_slots, int32_t world, int64_t n_rows, int32_t d,
                                    int32_t rank, void *out, int out_bf16, cudaStream_t s, int *launches);
cudaError_t launch_lmhead_tp_combine(const float4 *parts, int32_t R, const LossArgs &a, cudaStream_t s,
                                     int *launches);
cudaError_t launch_lmhead_combine(const RowPart *part, const float *zy, int32_t n_split, const LossArgs &a,
                                  cudaStream_t s, int *launches);
cudaError_t launch_vp(const LossArgs &a, const grpo_vp_comm_t *comm, unsigned long long *row_ctr,
                      cudaStream_t s, int *launches,
                      grpo_plan_t *plan, char *why, size_t why_len);
cudaError_t launch_loss_bwd(const uint16_t *logits, int64_t n_rows, int32_t V, int64_t ld,
                            const int64_t *target_ids, const float *lse, const float *scale,
                            float mult, uint16_t *dlogits, cudaStream_t s, int *launches);
cudaError_t launch_validate(const int64_t *version_ids, const int64_t *cu, const int32_t *group_ids,
                            int32_t N, int64_t T, int32_t P, int32_t V, int32_t G, int32_t tbs,
                            int64_t v_theta, int32_t K, const int64_t *token_version,
                            const int64_t *targets, const float *logp_behav, const int64_t *tcu,
                            const int32_t *traj_index, int32_t n_tok_traj, int64_t T_tok,
                            uint32_t *flags, int32_t *group_count, int32_t *stale_hist,
                            grpo_validate_summary_t *summary, double *token_counts, cudaStream_t s,
                            int *launches);
cudaError_t launch_validate_combine(grpo_validate_summary_t *summary, const double *token_counts,
                                    cudaStream_t s, int *launches);
cudaError_t launch_combine_ranks(const double *gathered, int32_t world, int32_t n, double *out,
                                 cudaStream_t s, int *launches);
cudaError_t launch_advantage(const float *rewards, const int32_t *group_ids, const int64_t *cu,
                             int32_t N, int32_t P, float std_floor, int32_t norm,
                             int32_t unbiased, const uint8_t *traj_mask, float *adv,
                             float *inv_norm, int32_t *group_count, cudaStream_t s, int *launches);

}  // namespace grpo
