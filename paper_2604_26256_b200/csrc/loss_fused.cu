// loss_fused.cu -- the roofline kernel of the path: one pass over the bf16
// logits that computes, per row t, the vocab-wide log-softmax, the target
// log-prob, the clipped-ratio term of J_async and its gradient, and writes
// dlogits = s_t (softmax - onehot(y_t)) once.
//
//   PAPER.md P:32-33, P:136   log pi_theta(y_t | .) = z_{t,y} - logsumexp_v z_{t,v}
//   PAPER.md P:9-34, P:151    term = min(r A, clip_eps(r) A), r = exp(logp - logp_w)
//   DESIGN.md Z19             dlogits = d(-J)/dz = s_t (softmax - onehot)
//
// Design.  A row of V bf16 logits (297 KiB at
// V = 152064) does not fit one SM, so a thread-block cluster of C CTAs owns a
// row: CTA c holds columns [c*slice, (c+1)*slice) of it in a ring of S
// shared-memory stages filled by 1-D bulk TMA (cp.async.bulk, mbarrier
// transaction counts).  HBM sees one read of the logits and one write of
// dlogits: 4V bytes per row.
//
// Warp specialisation, no CTA-wide barrier in the loop:
//   compute warps (kComp), per row k:
//     A(k): reduce the warp's share of the slice (stage k % S) to a
//           log2-domain partial (a, s) and st.async it (8 B) straight into
//           every CTA of the cluster (DSMEM, completing on the peer's xbar);
//     B(k - lag): when the row scalars of row k - lag are published, write
//           its dlogits from the stage; the last warp to finish a stage
//           refills it with row k - lag + S (bulk TMA).
//   control warp, per row r:  read z_y if this CTA owns the target column and
//     st.async (z_y, owner) to every CTA; E(r - lag + 1): once all C x kComp
//     partials of that row are in, form lse, logp, r, clip, term and the token
//     scale, publish them (smem + mbarrier), write the per-row outputs (cluster
//     rank 0), and re-arm the exchange slot.
// A peer's A(k) needs this CTA's partials of row k - S, and this CTA's A(j)
// comes after its B(j - lag - 1), i.e. after E(j - lag - 1); so with
// NX = S + lag + 1 exchange slots a slot is consumed and re-armed (in E(k))
// before any peer can write it for row k + NX.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace grpo {

constexpr int kComp = 7;                    // compute warps
constexpr int kWarps = kComp + 1;           // + the control warp
constexpr int kThreads = kWarps * 32;
constexpr int kCompThreads = kComp * 32;
constexpr int kMaxCluster = 16;
constexpr int kMaxStages = 8;
constexpr int kMaxSlots = kMaxStages + 3;   // exchange slots NX = S + lag + 1

struct FusedParams {
    const uint16_t *logits;
    uint16_t *dlogits;
    int64_t ld;
    int32_t V;
    int64_t n_rows;
    const RowInfo *rowinfo;
    float eps_lo, eps_hi, grad_scale;
    float *logp_out, *lse_out, *scale_out, *term_ws, *logp_ws;
    uint8_t *flag_ws;
    int32_t n_vec_row;  // ceil(V / 8)
    int32_t slice_vec;  // vectors of 8 bf16 per CTA (last CTA may hold fewer)
    int32_t stages;
    int32_t lag;        // B(k) runs `lag` rows after A(k)
    uint32_t piece;     // bytes per bulk-copy request (a slice is split into pieces)
    uint32_t stage_bytes;
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

// Shared-memory carve-up (host and device agree through this one function).
struct FusedSmem {
    size_t bars, cnt, part, zmsg, meta, rowsc, total;
};
__host__ __device__ __forceinline__ FusedSmem fused_smem_layout(int S, uint32_t stage_bytes) {
    FusedSmem L;
    L.bars = (size_t)S * stage_bytes;  // full[S], scal[kMaxSlots], xbar[kMaxSlots]
    L.cnt = L.bars + (size_t)(kMaxStages + 2 * kMaxSlots) * 8;                 // free counters
    L.part = L.cnt + (((size_t)kMaxStages * 4 + 15) / 16) * 16;
    L.zmsg = L.part + (size_t)kMaxSlots * kMaxCluster * kComp * sizeof(float2);
    L.meta = L.zmsg + (size_t)kMaxSlots * kMaxCluster * sizeof(float2);
    L.rowsc = L.meta + kMaxSlots * sizeof(RowInfo);
    L.total = L.rowsc + kMaxSlots * sizeof(float4);
    return L;
}

// One slice = bulk copies of at most `piece` bytes, all counted on one mbarrier.
__device__ __forceinline__ void load_slice(void *dst, const void *src, uint32_t bytes,
                                           uint32_t piece, uint64_t *bar, uint64_t pol) {
    for (uint32_t o = 0; o < bytes; o += piece)
        bulk_g2s(static_cast<uint8_t *>(dst) + o, static_cast<const uint8_t *>(src) + o,
                 min(piece, bytes - o), bar, pol);
}

template <int VPT>
__global__ void __launch_bounds__(kThreads, 2)
    fused_cluster_kernel(const FusedParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int S = p.stages;
    const int D = p.lag;
    const int NX = S + D + 1;
    const FusedSmem lay = fused_smem_layout(S, p.stage_bytes);
    uint8_t *stage_base = smem;
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + lay.bars);  // [S]
    uint64_t *scal_bar = full_bar + kMaxStages;                           // [NX]
    uint64_t *xbar = scal_bar + kMaxSlots;                                // [NX]
    int *free_cnt = reinterpret_cast<int *>(smem + lay.cnt);             // [S]
    float2 *part = reinterpret_cast<float2 *>(smem + lay.part);          // [NX][C][kComp]
    float2 *zmsg = reinterpret_cast<float2 *>(smem + lay.zmsg);          // [NX][C]
    RowInfo *meta = reinterpret_cast<RowInfo *>(smem + lay.meta);        // [NX]
    float4 *rowsc = reinterpret_cast<float4 *>(smem + lay.rowsc);        // [NX]

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
    const int32_t col_end = col_begin + my_vecs * 8;
    // the row's last vector holds V % 8 valid columns (if nonzero)
    const int32_t tail_valid = p.V - (p.n_vec_row - 1) * 8;
    const int32_t tail_vi = (tail_valid < 8) ? (p.n_vec_row - 1 - vec_begin) : -1;
    const int32_t my_rows = (g < p.n_rows) ? (int32_t)((p.n_rows - 1 - g) / n_cl + 1) : 0;
    const uint32_t xbytes = C * (uint32_t)((kComp + 1) * sizeof(float2));
    const int64_t row_stride = n_cl * p.ld;            // elements between my consecutive rows
    const uint16_t *src0 = p.logits + g * p.ld + col_begin;
    const bool control = (warp == kComp);

    if (control && lane == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_bar[i], 1);
            free_cnt[i] = 0;
        }
        for (int i = 0; i < NX; ++i) {
            mbar_init(&scal_bar[i], 1);
            mbar_init(&xbar[i], 1);
        }
        fence_mbar_init_cluster();
        for (int k = 0; k < NX && k < my_rows; ++k)   // every slot armed for its first row
            mbar_arrive_expect_tx(&xbar[k], xbytes);
        const uint64_t pol = policy_evict_first();
        for (int k = 0; k < S && k < my_rows; ++k) {   // fill the ring
            mbar_arrive_expect_tx(&full_bar[k], my_bytes);
            if (my_bytes)
                load_slice(stage_base + (size_t)k * p.stage_bytes, src0 + k * row_stride, my_bytes,
                           p.piece, &full_bar[k], pol);
        }
    }
    cluster_sync_all();  // barriers of every CTA exist and are armed before any st.async

    if (control) {
        // ================================================================ control warp
        int c_st = 0, z_slot = 0, e_slot = 0;
        uint32_t c_ph = 0, e_ph = 0;
        RowInfo ri0{}, ri1{};                           // lane 0: rows r and r + 1
        if (lane == 0 && my_rows > 0) ri0 = load_rowinfo(p.rowinfo + g);
        if (lane == 0 && my_rows > 1) ri1 = load_rowinfo(p.rowinfo + g + n_cl);
        for (int r = 0; r < my_rows + D; ++r) {
            if (r < my_rows) {
                // (a) the row's slice has landed: z_y if this CTA owns column y, to every CTA
                mbar_wait(&full_bar[c_st], c_ph);
                float zy = 0.0f, own = 0.0f;
                if (lane == 0) {
                    meta[z_slot] = ri0;
                    const int32_t y = ri0.target;
                    if (y >= col_begin && y < col_end && y < p.V) {
                        uint16_t hv;
                        asm volatile("ld.shared.u16 %0, [%1];"
                                     : "=h"(hv)
                                     : "r"(smem_u32(stage_base + (size_t)c_st * p.stage_bytes) +
                                           (uint32_t)(y - col_begin) * 2u)
                                     : "memory");
                        zy = __uint_as_float(((uint32_t)hv) << 16);
                        own = 1.0f;
                    }
                    ri0 = ri1;
                    if (r + 2 < my_rows) ri1 = load_rowinfo(p.rowinfo + g + (int64_t)(r + 2) * n_cl);
                }
                zy = __shfl_sync(0xFFFFFFFFu, zy, 0);
                own = __shfl_sync(0xFFFFFFFFu, own, 0);
                if (lane < (int)C)
                    st_async_v2(mapa_shared(smem_u32(&zmsg[z_slot * kMaxCluster + crank]), lane),
                                mapa_shared(smem_u32(&xbar[z_slot]), lane), zy, own);
                if (++c_st == S) { c_st = 0; c_ph ^= 1u; }
                if (++z_slot == NX) z_slot = 0;
            }
            // (b) E(r - D + 1): the row scalars, once every partial of the row is in
            const int ke = r - D + 1;
            if (ke >= 0 && ke < my_rows) {
                mbar_wait(&xbar[e_slot], e_ph);
                const int np = (int)C * kComp;
                const float2 *ps = part + (size_t)e_slot * kMaxCluster * kComp;
                float M = -INFINITY, Ssum = 0.0f;
                for (int q = lane; q < np; q += 32) {
                    const float2 v2 = ps[q];
                    lse2_merge(M, Ssum, v2.x, v2.y);
                }
                warp_lse2_combine(M, Ssum);
                float zsrc = 0.0f;
                bool own = false;
                if (lane < (int)C) {
                    const float2 zm = zmsg[e_slot * kMaxCluster + lane];
                    zsrc = zm.x;
                    own = zm.y != 0.0f;
                }
                const uint32_t own_mask = __ballot_sync(0xFFFFFFFFu, own);
                const float zsh = __shfl_sync(0xFFFFFFFFu, zsrc, own_mask ? __ffs(own_mask) - 1 : 0);
                if (lane == 0) {
                    const RowInfo ri = meta[e_slot];
                    const bool y_valid = own_mask != 0u;   // column y lies in [0, V)
                    const float zyv = y_valid ? zsh : __int_as_float(0x7FC00000);
                    const float l2s = log2f(Ssum);
                    const float lse2 = M + l2s;           // log2-domain logsumexp of the row
                    const double logp_d = row_logp(zyv, M, l2s);
                    const RowOut o = row_epilogue(logp_d, ri, p.eps_lo, p.eps_hi, p.grad_scale);
                    rowsc[e_slot] = make_float4(lse2, o.s, zyv,
                                                __int_as_float(y_valid ? ri.target : -1));
                    // slot consumed: re-arm it for row ke + NX before the compute warps
                    // can let any peer reach that row
                    if (ke + NX < my_rows) mbar_arrive_expect_tx(&xbar[e_slot], xbytes);
                    mbar_arrive(&scal_bar[e_slot]);
                    if (crank == 0) {
                        const int64_t row = g + (int64_t)ke * n_cl;
                        const float logp = (float)logp_d;
                        if (p.logp_out) p.logp_out[row] = logp;
                        if (p.lse_out) p.lse_out[row] = lse2 * kLn2;
                        if (p.scale_out) p.scale_out[row] = o.s;
                        p.term_ws[row] = o.term;
                        p.logp_ws[row] = logp;
                        p.flag_ws[row] = o.flags;
                    }
                }
                __syncwarp();
                if (++e_slot == NX) { e_slot = 0; e_ph ^= 1u; }
            }
        }
    } else {
        // ================================================================ compute warps
        const uint64_t pol = policy_evict_first();
        int a_st = 0, a_slot = 0, b_st = 0, b_slot = 0;
        uint32_t a_ph = 0, b_ph = 0;
        for (int it = 0; it < my_rows + D; ++it) {
            if (it < my_rows) {
                // ------------------------------------------------------------ A(it)
                mbar_wait(&full_bar[a_st], a_ph);
                const uint32_t sbase = smem_u32(stage_base + (size_t)a_st * p.stage_bytes);
                uint32_t mx2 = kBf16NegInfPair;
                uint4 v[VPT];
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    const int vi = tid + j * kCompThreads;
                    if (vi < my_vecs) {
                        v[j] = lds128(sbase + (uint32_t)vi * 16u);
                        // columns >= V of the row's ragged last vector count as -inf
                        if (vi == tail_vi) v[j] = mask_tail(v[j], tail_valid);
                    } else {
                        v[j] = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair,
                                          kBf16NegInfPair);
                    }
                    mx2 = bmax2(bmax2(mx2, bmax2(v[j].x, v[j].y)), bmax2(v[j].z, v[j].w));
                }
                float a = log2_ref(fmaxf(bf_lo(mx2), bf_hi(mx2)));
                const float aL = (a == -INFINITY) ? 0.0f : a;
                float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
                for (int j = 0; j < VPT; ++j) {
                    s0 += ex2(fmaf(bf_lo(v[j].x), kLog2e, -aL)) + ex2(fmaf(bf_hi(v[j].x), kLog2e, -aL));
                    s1 += ex2(fmaf(bf_lo(v[j].y), kLog2e, -aL)) + ex2(fmaf(bf_hi(v[j].y), kLog2e, -aL));
                    s2 += ex2(fmaf(bf_lo(v[j].z), kLog2e, -aL)) + ex2(fmaf(bf_hi(v[j].z), kLog2e, -aL));
                    s3 += ex2(fmaf(bf_lo(v[j].w), kLog2e, -aL)) + ex2(fmaf(bf_hi(v[j].w), kLog2e, -aL));
                }
                float s = (s0 + s1) + (s2 + s3);
                warp_lse2_combine(a, s);
                // the warp partial goes straight to every CTA of the cluster
                if (lane < (int)C)
                    st_async_v2(
                        mapa_shared(smem_u32(&part[((size_t)a_slot * kMaxCluster + crank) * kComp + warp]),
                                    lane),
                        mapa_shared(smem_u32(&xbar[a_slot]), lane), a, s);
                if (++a_st == S) { a_st = 0; a_ph ^= 1u; }
                if (++a_slot == NX) a_slot = 0;
            }
            if (it >= D) {
                // ------------------------------------------------------------ B(it - D)
                const int k = it - D;
                const int64_t row = g + (int64_t)k * n_cl;
                mbar_wait(&scal_bar[b_slot], b_ph);
                const float4 sc4 = rowsc[b_slot];
                const float lse2 = sc4.x, sc = sc4.y, zy = sc4.z;
                const int32_t y = __float_as_int(sc4.w);
                const uint32_t sbase = smem_u32(stage_base + (size_t)b_st * p.stage_bytes);
                if (p.dlogits) {
                    uint16_t *drow = p.dlogits + row * p.ld + col_begin;
                    const int32_t yv = (y >= col_begin && y < col_end) ? ((y - col_begin) >> 3) : -1;
#pragma unroll
                    for (int j = 0; j < VPT; ++j) {
                        const int vi = tid + j * kCompThreads;
                        if (vi >= my_vecs) continue;
                        uint4 d = make_uint4(0u, 0u, 0u, 0u);
                        if (sc != 0.0f) {
                            const uint4 x = lds128(sbase + (uint32_t)vi * 16u);
                            d.x = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.x), kLog2e, -lse2)),
                                              sc * ex2(fmaf(bf_hi(x.x), kLog2e, -lse2)));
                            d.y = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.y), kLog2e, -lse2)),
                                              sc * ex2(fmaf(bf_hi(x.y), kLog2e, -lse2)));
                            d.z = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.z), kLog2e, -lse2)),
                                              sc * ex2(fmaf(bf_hi(x.z), kLog2e, -lse2)));
                            d.w = pack_bf16x2(sc * ex2(fmaf(bf_lo(x.w), kLog2e, -lse2)),
                                              sc * ex2(fmaf(bf_hi(x.w), kLog2e, -lse2)));
                        }
                        if (vi == tail_vi)
                            store_tail(drow + vi * 8, d, tail_valid);
                        else
                            stg_stream(drow + vi * 8, d);
                        if (vi == yv) {
                            // target entry: s (p_y - 1), from the unrounded probability
                            const float py = ex2(fmaf(zy, kLog2e, -lse2));
                            drow[y - col_begin] = f2bf(sc * (py - 1.0f));
                        }
                    }
                }
                // the last warp done with this stage refills it with row k + S
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    if (atomicAdd(&free_cnt[b_st], 1) == kComp - 1) {
                        free_cnt[b_st] = 0;
                        __threadfence_block();
                        if (k + S < my_rows) {
                            mbar_arrive_expect_tx(&full_bar[b_st], my_bytes);
                            if (my_bytes)
                                load_slice(stage_base + (size_t)b_st * p.stage_bytes,
                                           src0 + (int64_t)(k + S) * row_stride, my_bytes, p.piece,
                                           &full_bar[b_st], pol);
                        }
                    }
                }
                if (++b_st == S) b_st = 0;
                if (++b_slot == NX) { b_slot = 0; b_ph ^= 1u; }
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
    while (C < kMaxCluster && (n_vec_row + C - 1) / C > 8 * kCompThreads) C *= 2;
    return C;
}

template <int VPT>
cudaError_t launch_vpt(const FusedParams &fp, int C, int ctas_per_sm, size_t smem,
                       cudaStream_t s, int64_t n_rows, char *why, size_t why_len,
                       grpo_plan_t *plan) {
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
    if (plan) {
        plan->kernel = 1;
        plan->cluster_size = C;
        plan->ctas_per_sm = ctas_per_sm;
        plan->stages = fp.stages;
        plan->lag = fp.lag;
        plan->vec_per_thread = VPT;
        plan->grid = (int32_t)(n_cl * C);
        plan->max_clusters = max_clusters;
        plan->smem_bytes = (int32_t)smem;
    }
    return cudaLaunchKernelEx(&cfg, kern, fp);
}

}  // namespace

cudaError_t launch_fused_cluster(const LossArgs &a, const grpo_tune_t *tune, cudaStream_t s,
                                 int *launches, char *why, size_t why_len, grpo_plan_t *plan) {
    if (a.n_rows == 0) return cudaSuccess;
    FusedParams fp;
    fp.logits = a.logits;
    fp.dlogits = a.dlogits;
    fp.ld = a.ld;
    fp.V = a.V;
    fp.n_rows = a.n_rows;
    fp.rowinfo = a.rowinfo;
    fp.eps_lo = a.eps_lo;
    fp.eps_hi = a.eps_hi;
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
    const int vpt_needed = (fp.slice_vec + kCompThreads - 1) / kCompThreads;
    fp.stage_bytes = (uint32_t)(((size_t)fp.slice_vec * 16 + 127) / 128 * 128);
    const bool auto_lag = !(tune && tune->lag > 0);
    int lag = auto_lag ? 2 : tune->lag;
    if (lag > 2) {
        if (why) snprintf(why, why_len, "lag %d > 2", lag);
        return cudaErrorInvalidValue;
    }
    const size_t per_sm = 227 * 1024;
    int stages = (tune && tune->stages > 0) ? tune->stages : 0;
    if (stages == 0) {
        const size_t fixed = fused_smem_layout(0, fp.stage_bytes).total + 8 * 8;
        const size_t budget = per_sm / ctas_per_sm - 1024 - fixed;
        stages = (int)(budget / fp.stage_bytes);
        if (stages > kMaxStages) stages = kMaxStages;
    }
    if (auto_lag && stages < lag + 2) lag = stages - 2 >= 1 ? stages - 2 : 1;
    fp.lag = lag;
    fp.piece = fp.stage_bytes;  // one bulk copy per slice
    if (stages > kMaxStages) {
        if (why) snprintf(why, why_len, "stages %d > %d", stages, kMaxStages);
        return cudaErrorInvalidValue;
    }
    if (stages < lag + 2) {
        if (why) snprintf(why, why_len, "%d stages < lag + 2 = %d (slice %u B)", stages, lag + 2,
                          fp.stage_bytes);
        return cudaErrorInvalidConfiguration;
    }
    fp.stages = stages;
    const size_t smem = fused_smem_layout(stages, fp.stage_bytes).total;
    if (C < 1 || C > kMaxCluster || (C & (C - 1)) != 0) {
        if (why) snprintf(why, why_len, "cluster_size %d not a power of two <= 16", C);
        return cudaErrorInvalidValue;
    }
    if (smem > per_sm) {
        if (why) snprintf(why, why_len, "fused kernel needs %zu B shared memory", smem);
        return cudaErrorInvalidConfiguration;
    }
    cudaError_t e;
    if (vpt_needed <= 2) e = launch_vpt<2>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else if (vpt_needed <= 4) e = launch_vpt<4>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else if (vpt_needed <= 6) e = launch_vpt<6>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else if (vpt_needed <= 8) e = launch_vpt<8>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else if (vpt_needed <= 10) e = launch_vpt<10>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else if (vpt_needed <= 12) e = launch_vpt<12>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else if (vpt_needed <= 16) e = launch_vpt<16>(fp, C, ctas_per_sm, smem, s, a.n_rows, why, why_len, plan);
    else {
        if (why) snprintf(why, why_len, "slice of %d vectors too large for cluster %d", fp.slice_vec, C);
        return cudaErrorInvalidConfiguration;
    }
    if (e == cudaSuccess) *launches += 1;
    return e;
}

}  // namespace grpo
