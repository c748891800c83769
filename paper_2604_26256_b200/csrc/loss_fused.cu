// loss_fused.cu -- the roofline kernel of the path: one pass over the bf16
// logits that computes, per row t, the vocab-wide log-softmax, the target
// log-prob, the clipped-ratio term of J_async and its gradient, and writes
// dlogits = s_t (softmax - onehot(y_t)) once.
//
//   PAPER.md P:32-33, P:136   log pi_theta(y_t | .) = z_{t,y} - logsumexp_v z_{t,v}
//   PAPER.md P:9-34, P:151    term = min(r A, clip_eps(r) A), r = exp(logp - logp_w)
//   DESIGN.md Z19             dlogits = d(-J)/dz = s_t (softmax - onehot)
//
// Design: a row of V bf16 logits (297 KiB at
// V = 152064) does not fit one SM, so a thread-block cluster of C CTAs owns a
// row: CTA c holds columns [c*slice, (c+1)*slice).  Thread 0 streams each
// CTA's slice of the next rows into a ring of S shared-memory stages with 1-D
// bulk TMA (cp.async.bulk + mbarrier transaction counts).  All warps copy the
// slice into registers, reduce (max, sum exp) over it, and warp 0 exchanges
// the 16-byte partial (m_c, s_c, z_y) with every CTA of the cluster through
// DSMEM (st.async completing on the peer's mbarrier).  Every CTA then holds
// the row's lse and writes its slice of dlogits straight from registers with
// 128-bit streaming stores.  HBM sees one read of the logits and one write
// of dlogits: 4V bytes per row.  Two CTAs per SM overlap one CTA's exchange
// latency with the other's arithmetic; the TMA ring keeps S rows in flight.
#include <cstdio>

#include "common.cuh"

namespace grpo {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kMaxCluster = 16;

struct FusedParams {
    const uint16_t *logits;
    uint16_t *dlogits;
    int64_t ld;
    int32_t V;
    int64_t n_rows;
    const RowInfo *rowinfo;
    float eps, grad_scale;
    float *logp_out, *lse_out, *scale_out, *term_ws, *logp_ws;
    uint8_t *flag_ws;
    int32_t n_vec_row;  // ceil(V / 8)
    int32_t slice_vec;  // vectors of 8 bf16 per CTA (last CTA may hold fewer)
    int32_t stages;
    uint32_t stage_bytes;
};

struct __align__(16) XMsg {
    float m, s, zy, pad;
};

__device__ __forceinline__ RowInfo load_rowinfo(const RowInfo *p) {
    const int4 q = __ldg(reinterpret_cast<const int4 *>(p));
    RowInfo r;
    r.target = q.x;
    r.logp_w = __int_as_float(q.y);
    r.adv = __int_as_float(q.z);
    r.inv_norm = __int_as_float(q.w);
    return r;
}

template <int VPT>
__global__ void __launch_bounds__(kThreads, 2)
    fused_cluster_kernel(const FusedParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int S = p.stages;
    uint8_t *stage_base = smem;
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
    uint64_t *xbar = full_bar + S;                                     // [2]
    XMsg *xch = reinterpret_cast<XMsg *>(                              // [2][kMaxCluster]
        smem + (size_t)S * p.stage_bytes + (((size_t)(S + 2) * 8 + 15) / 16) * 16);
    float2 *red = reinterpret_cast<float2 *>(xch + 2 * kMaxCluster);   // [kWarps]

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const uint32_t crank = cluster_ctarank();
    const uint32_t C = cluster_nctarank();
    const int64_t g = cluster_id_x();
    const int64_t n_cl = ncluster_x();

    const int32_t vec_begin = (int32_t)crank * p.slice_vec;
    const int32_t my_vecs = max(0, min(p.slice_vec, p.n_vec_row - vec_begin));
    const uint32_t my_bytes = (uint32_t)my_vecs * 16u;
    const int32_t col_begin = vec_begin * 8;
    // the row's last vector holds V % 8 valid columns (if nonzero)
    const int32_t tail_valid = p.V - (p.n_vec_row - 1) * 8;
    const int64_t my_rows = (g < p.n_rows) ? (p.n_rows - 1 - g) / n_cl + 1 : 0;
    uint64_t pol = 0;

    if (tid == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&full_bar[i], 1);
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        fence_mbar_init_cluster();
        mbar_arrive_expect_tx(&xbar[0], C * (uint32_t)sizeof(XMsg));  // arm row 0's exchange
        pol = policy_evict_first();
        for (int64_t it = 0; it < S && it < my_rows; ++it) {          // fill the ring
            mbar_arrive_expect_tx(&full_bar[it], my_bytes);
            if (my_bytes)
                bulk_g2s(stage_base + (size_t)it * p.stage_bytes,
                         p.logits + (g + it * n_cl) * p.ld + col_begin, my_bytes, &full_bar[it],
                         pol);
        }
    }
    cluster_sync_all();  // barriers of every CTA exist and are armed before any st.async

    RowInfo ri_next = my_rows > 0 ? load_rowinfo(p.rowinfo + g) : RowInfo{};
    for (int64_t it = 0; it < my_rows; ++it) {
        const int64_t row = g + it * n_cl;
        const int st = (int)(it % S);
        const uint32_t ph = (uint32_t)((it / S) & 1);
        const int xb = (int)(it & 1);
        const RowInfo ri = ri_next;
        if (it + 1 < my_rows) ri_next = load_rowinfo(p.rowinfo + row + n_cl);  // prefetch
        mbar_wait(&full_bar[st], ph);

        const uint32_t sbase = smem_u32(stage_base + (size_t)st * p.stage_bytes);
        uint4 v[VPT];
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            const int vi = tid + j * kThreads;
            if (vi < my_vecs) {
                v[j] = lds128(sbase + (uint32_t)vi * 16u);
                // mask columns >= V of the row's ragged last vector to -inf
                if (vec_begin + vi == p.n_vec_row - 1 && tail_valid < 8)
                    v[j] = mask_tail(v[j], tail_valid);
            } else {
                v[j] = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair,
                                  kBf16NegInfPair);
            }
        }
        // the CTA owning column y reads z_y from the stage
        const int32_t y = ri.target;
        const bool y_valid = (y >= 0) && (y < p.V);
        const int32_t y_owner = y_valid ? (y >> 3) / p.slice_vec : -1;
        float zy_local = 0.0f;
        if (tid == 0 && y_owner == (int32_t)crank) {
            const uint32_t a = sbase + (uint32_t)(y - col_begin) * 2u;
            uint16_t hv;
            asm volatile("ld.shared.u16 %0, [%1];" : "=h"(hv) : "r"(a) : "memory");
            zy_local = __uint_as_float(((uint32_t)hv) << 16);
        }

        // ---- thread-local max (packed bf16x2) then sum of exp
        uint32_t mx2 = kBf16NegInfPair;
#pragma unroll
        for (int j = 0; j < VPT; ++j)
            mx2 = bmax2(bmax2(mx2, bmax2(v[j].x, v[j].y)), bmax2(v[j].z, v[j].w));
        float a = log2_ref(fmaxf(bf_lo(mx2), bf_hi(mx2)));
        const float mL = (a == -INFINITY) ? 0.0f : a;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            s0 += ex2(fmaf(bf_lo(v[j].x), kLog2e, -mL)) + ex2(fmaf(bf_hi(v[j].x), kLog2e, -mL));
            s1 += ex2(fmaf(bf_lo(v[j].y), kLog2e, -mL)) + ex2(fmaf(bf_hi(v[j].y), kLog2e, -mL));
            s2 += ex2(fmaf(bf_lo(v[j].z), kLog2e, -mL)) + ex2(fmaf(bf_hi(v[j].z), kLog2e, -mL));
            s3 += ex2(fmaf(bf_lo(v[j].w), kLog2e, -mL)) + ex2(fmaf(bf_hi(v[j].w), kLog2e, -mL));
        }
        float s = (s0 + s1) + (s2 + s3);
        warp_lse2_allreduce(a, s);
        if (lane == 0) red[warp] = make_float2(a, s);
        __syncthreads();  // every warp has its slice in registers: stage st is free

        if (warp == 0) {
            if (lane == 0 && it + S < my_rows) {  // refill stage st with row it + S
                mbar_arrive_expect_tx(&full_bar[st], my_bytes);
                if (my_bytes)
                    bulk_g2s(stage_base + (size_t)st * p.stage_bytes,
                             p.logits + (row + S * n_cl) * p.ld + col_begin, my_bytes,
                             &full_bar[st], pol);
            }
            // combine the warps, arm the exchange for row it+1, send to every peer
            float cm = -INFINITY, cs = 0.0f;
            if (lane < kWarps) {
                const float2 r2 = red[lane];
                cm = r2.x;
                cs = r2.y;
            }
            warp_lse2_allreduce(cm, cs);
            const float zy = __shfl_sync(0xFFFFFFFFu, zy_local, 0);
            if (lane == 0 && it + 1 < my_rows)
                mbar_arrive_expect_tx(&xbar[xb ^ 1], C * (uint32_t)sizeof(XMsg));
            __syncwarp();
            if (lane < (int)C) {
                const uint32_t laddr = smem_u32(&xch[xb * kMaxCluster + crank]);
                const uint32_t lbar = smem_u32(&xbar[xb]);
                st_async_v4(mapa_shared(laddr, lane), mapa_shared(lbar, lane), cm, cs, zy, 0.0f);
            }
        }

        // ---- the row's lse from the C partials (identical in every warp and CTA)
        mbar_wait_cluster(&xbar[xb], (uint32_t)((it >> 1) & 1));
        float M = -INFINITY, Ssum = 0.0f, zsrc = 0.0f;
        if (lane < (int)C) {
            const XMsg msg = xch[xb * kMaxCluster + lane];
            M = msg.m;
            Ssum = msg.s;
            zsrc = msg.zy;
        }
        warp_lse2_allreduce(M, Ssum);
        const float zy = y_valid ? __shfl_sync(0xFFFFFFFFu, zsrc, max(y_owner, 0))
                                 : __int_as_float(0x7FC00000);
        const float l2s = log2f(Ssum);
        const float lse2 = M + l2s;           // log2-domain logsumexp of the row
        const float lse = lse2 * kLn2;
        const double logp_d = row_logp(zy, M, l2s);
        const float logp = (float)logp_d;
        const RowOut o = row_epilogue(logp_d, ri, p.eps, p.grad_scale);
        if (crank == 0 && tid == 0) {
            if (p.logp_out) p.logp_out[row] = logp;
            if (p.lse_out) p.lse_out[row] = lse;
            if (p.scale_out) p.scale_out[row] = o.s;
            p.term_ws[row] = o.term;
            p.logp_ws[row] = logp;
            p.flag_ws[row] = o.flags;
        }

        // ---- backward: dlogits = s (softmax - onehot), one write per element
        if (p.dlogits) {
            uint16_t *drow = p.dlogits + row * p.ld;
            const float off = lse2;
            const float sc = o.s;
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const int vi = tid + j * kThreads;
                if (vi >= my_vecs) continue;
                uint4 d;
                if (sc == 0.0f) {
                    d = make_uint4(0u, 0u, 0u, 0u);
                } else {
                    d.x = pack_bf16x2(sc * ex2(fmaf(bf_lo(v[j].x), kLog2e, -off)),
                                      sc * ex2(fmaf(bf_hi(v[j].x), kLog2e, -off)));
                    d.y = pack_bf16x2(sc * ex2(fmaf(bf_lo(v[j].y), kLog2e, -off)),
                                      sc * ex2(fmaf(bf_hi(v[j].y), kLog2e, -off)));
                    d.z = pack_bf16x2(sc * ex2(fmaf(bf_lo(v[j].z), kLog2e, -off)),
                                      sc * ex2(fmaf(bf_hi(v[j].z), kLog2e, -off)));
                    d.w = pack_bf16x2(sc * ex2(fmaf(bf_lo(v[j].w), kLog2e, -off)),
                                      sc * ex2(fmaf(bf_hi(v[j].w), kLog2e, -off)));
                }
                const int32_t col = (vec_begin + vi) * 8;
                if (vec_begin + vi == p.n_vec_row - 1 && tail_valid < 8)
                    store_tail(drow + col, d, tail_valid);
                else
                    stg_stream(drow + col, d);
                if (y_valid && (y >> 3) == vec_begin + vi) {
                    // target entry: s (p_y - 1), from the unrounded probability
                    const float py = ex2(fmaf(zy, kLog2e, -off));
                    drow[y] = f2bf(sc * (py - 1.0f));
                }
            }
        }
    }
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

// ------------------------------------------------------------------ host side
namespace {

int pick_cluster(int32_t n_vec_row) {
    // smallest power of two keeping a CTA slice <= 8 vectors (64 bf16) per thread
    int C = 1;
    while (C < kMaxCluster && (n_vec_row + C - 1) / C > 8 * kThreads) C *= 2;
    return C;
}

template <int VPT>
cudaError_t launch_vpt(const FusedParams &fp, int C, int ctas_per_sm, size_t smem,
                       cudaStream_t s, int64_t n_rows, char *why, size_t why_len) {
    auto kern = fused_cluster_kernel<VPT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (C > 8) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cfg.gridDim = dim3((unsigned)(C * ((n_sm * ctas_per_sm) / C)));
    int max_clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (max_clusters <= 0) {
        if (why) snprintf(why, why_len, "no cluster of %d CTAs (%zu B smem) fits", C, smem);
        return cudaErrorInvalidConfiguration;
    }
    int64_t n_cl = (int64_t)max_clusters;
    if (n_cl > n_rows) n_cl = n_rows;
    cfg.gridDim = dim3((unsigned)(n_cl * C));
    return cudaLaunchKernelEx(&cfg, kern, fp);
}

}  // namespace

cudaError_t launch_fused_cluster(const LossArgs &a, const grpo_tune_t *tune, cudaStream_t s,
                                 int *launches, char *why, size_t why_len) {
    if (a.n_rows == 0) return cudaSuccess;
    FusedParams fp;
    fp.logits = a.logits;
    fp.dlogits = a.dlogits;
    fp.ld = a.ld;
    fp.V = a.V;
    fp.n_rows = a.n_rows;
    fp.rowinfo = a.rowinfo;
    fp.eps = a.eps;
    fp.grad_scale = a.grad_scale;
    fp.logp_out = a.logp_out;
    fp.lse_out = a.lse_out;
    fp.scale_out = a.scale_out;
    fp.term_ws = a.term_ws;
    fp.logp_ws = a.logp_ws;
    fp.flag_ws = a.flag_ws;
    fp.n_vec_row = (a.V + 7) / 8;

    int C = (tune && tune->cluster_size > 0) ? tune->cluster_size : pick_cluster(fp.n_vec_row);
    int ctas_per_sm = (tune && tune->ctas_per_sm > 0) ? tune->ctas_per_sm : 2;
    fp.slice_vec = (fp.n_vec_row + C - 1) / C;
    const int vpt_needed = (fp.slice_vec + kThreads - 1) / kThreads;
    fp.stage_bytes = (uint32_t)(((size_t)fp.slice_vec * 16 + 127) / 128 * 128);
    const size_t fixed = 8 * 8 + 2 * 8 + 2 * kMaxCluster * sizeof(XMsg) + kWarps * 8 + 256;
    const size_t per_sm = 227 * 1024;
    int stages = (tune && tune->stages > 0) ? tune->stages : 0;
    if (stages == 0) {
        const size_t budget = per_sm / ctas_per_sm - 1024 - fixed;
        stages = (int)(budget / fp.stage_bytes);
        if (stages > 4) stages = 4;
        if (stages < 1) stages = 1;
    }
    fp.stages = stages;
    const size_t smem = (size_t)stages * fp.stage_bytes + (((size_t)(stages + 2) * 8 + 15) / 16) * 16 +
                        2 * kMaxCluster * sizeof(XMsg) + kWarps * sizeof(float2);
    if (C < 1 || C > kMaxCluster || (C & (C - 1)) != 0) {
        if (why) snprintf(why, why_len, "cluster_size %d not a power of two <= 16", C);
        return cudaErrorInvalidValue;
    }
    if (smem > per_sm) {
        if (why) snprintf(why, why_len, "fused kernel needs %zu B shared memory", smem);
        return cudaErrorInvalidConfiguration;
    }
    cudaError_t e;
    if (vpt_needed <= 2) e = launch_vpt<2>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else if (vpt_needed <= 4) e = launch_vpt<4>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else if (vpt_needed <= 6) e = launch_vpt<6>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else if (vpt_needed <= 8) e = launch_vpt<8>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else if (vpt_needed <= 10) e = launch_vpt<10>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else if (vpt_needed <= 12) e = launch_vpt<12>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else if (vpt_needed <= 16) e = launch_vpt<16>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len);
    else {
        if (why) snprintf(why, why_len, "slice of %d vectors too large for cluster %d", fp.slice_vec, C);
        return cudaErrorInvalidConfiguration;
    }
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace grpo
