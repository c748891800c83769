// loss_aux.cu -- the smaller kernels around the fused loss:
//   rowinfo_kernel      row -> trajectory lookup (binary search over cu_seqlens) and
//                       the per-row metadata the fused kernel streams (16 B per row)
//   rowwise_kernel      a simple fused fwd+bwd variant: one CTA per row, two
//                       passes over the row (the second re-reads from L2)
//   segsum_kernel       deterministic per-trajectory segmented sums of term_t
//                       (eq:grpo_async's sum_t) and per-chunk counters
//   stats_kernel        fixed-order reduction of the trajectory partials into
//                       J's chunk contribution  sum_i inv_norm_i * sum_t term_t
//   bwd_kernel          unfused backward: dlogits = s (exp(z - lse) - onehot)
#include "common.cuh"
#include "rowwise.cuh"

namespace grpo {

// ------------------------------------------------------------------ row info
__global__ void rowinfo_kernel(int64_t row_begin, int64_t n_rows, const int64_t *__restrict__ cu,
                               int32_t N, const int32_t *__restrict__ traj_index,
                               const int64_t *__restrict__ targets,
                               const float *__restrict__ logp_behav,
                               const float *__restrict__ adv,
                               const float *__restrict__ inv_norm, RowInfo *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_rows;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = row_begin + k;
        RowInfo ri;
        const int64_t y = targets[k];
        ri.target = (y >= 0 && y < 0x7FFFFFFF) ? (int32_t)y : -1;
        ri.logp_w = logp_behav[k];
        ri.adv = 0.0f;
        ri.inv_norm = 0.0f;
        if (t >= cu[0] && t < cu[N]) {
            // largest i with cu[i] <= t  (then cu[i+1] > t)
            int32_t lo = 0, hi = N;
            while (hi - lo > 1) {
                const int32_t mid = (lo + hi) >> 1;
                if (cu[mid] <= t) lo = mid;
                else hi = mid;
            }
            const int32_t ti = traj_index ? traj_index[lo] : lo;
            ri.adv = adv[ti];
            ri.inv_norm = inv_norm[ti];
        }
        out[k] = ri;
    }
}

cudaError_t launch_rowinfo(const LossArgs &a, cudaStream_t s, int *launches) {
    if (a.n_rows == 0) return cudaSuccess;
    int64_t blocks = (a.n_rows + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    rowinfo_kernel<<<(unsigned)blocks, 256, 0, s>>>(a.row_begin, a.n_rows, a.cu_seqlens, a.N,
                                                    a.traj_index, a.target_ids, a.logp_behav,
                                                    a.adv, a.inv_norm, a.rowinfo);
    *launches += 1;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ row-wise fused variant
struct RowwiseParams {
    const uint16_t *logits;
    uint16_t *dlogits;
    int64_t ld;
    int32_t V;
    int64_t n_rows;
    const RowInfo *rowinfo;
    float eps_lo, eps_hi, grad_scale;
    float *logp_out, *lse_out, *scale_out;
    double *term_ws;
    float *logp_ws;
    uint8_t *flag_ws;
    int32_t prefetch;
    int32_t flags;  // bit 0: pass 2 in reverse batch order; bit 1: pass-1 policy evict_normal
    int32_t cache_vecs;  // leading vectors per thread kept in shared memory for pass 2
};


// Row-wise two-pass kernel.  A row (or, with C > 1, a 1/C slice of it held by one
// CTA of a C-CTA cluster) is processed by one CTA at a time; the grid is
// persistent and strides over rows.  Pass 1 streams the slice from HBM in
// batches of U vectors per thread (U x 16 B in flight per thread, L2
// evict_last) and reduces it to a log2-domain (max, sum) pair; the first
// cache_vecs vectors of every thread are also kept in shared memory.  With
// C > 1 the CTAs of the cluster swap their 16-byte partials through DSMEM
// around one cluster barrier.  Pass 2 writes dlogits with streaming 128-bit
// stores: the vectors not in shared memory are re-read newest-first (the end of
// the slice is the part most likely still in L2), the cached head comes from
// shared memory.  Full batches run without bounds checks; only the slice's
// last batch carries them and the ragged-tail masking.
template <int NT, int U, int C>
__global__ void __launch_bounds__(NT, (NT >= 1024 ? 1 : 1024 / NT)) rowwise_kernel(const RowwiseParams p) {
    using B = RowwiseBatch<NT, U>;
    constexpr int NW = NT / 32;
    constexpr int BV = NT * U;  // vectors per batch
    __shared__ RowPart red[NW];
    __shared__ float row_scalars[4];          // lse2 (log2 domain), s, g_y = s (p_y - 1), y
    __shared__ float4 xpart[2][C];            // cluster exchange, double-buffered by row parity
    extern __shared__ uint4 row_cache[];      // [cache_vecs][NT]
    const uint32_t crank = C > 1 ? cluster_ctarank() : 0;
    const int64_t grp = C > 1 ? (int64_t)cluster_id_x() : (int64_t)blockIdx.x;
    const int64_t n_grp = C > 1 ? (int64_t)ncluster_x() : (int64_t)gridDim.x;
    const int n_vec_row = (p.V + 7) / 8;
    const int slice = (n_vec_row + C - 1) / C;
    const int vec_lo = min((int)crank * slice, n_vec_row);
    const int n_vec = min(slice, n_vec_row - vec_lo);       // vectors of this CTA's slice
    const int tail_valid = p.V - (n_vec_row - 1) * 8;
    const int tail_vi = (tail_valid < 8 && n_vec_row - 1 >= vec_lo && n_vec_row - 1 < vec_lo + n_vec)
                            ? n_vec_row - 1 - vec_lo : -1;  // slice-local index of the ragged vector
    const int n_batch = (n_vec + BV - 1) / BV;
    // full batches run unchecked; the batch holding the ragged tail vector (if any) and a
    // short last batch take the checked path
    const int n_full = tail_vi >= 0 ? tail_vi / BV : n_vec / BV;
    const int cache_vecs = min(p.cache_vecs, n_batch * U);  // per thread
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    const uint4 neg_inf = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair,
                                     kBf16NegInfPair);
    int parity = 0;
    for (int64_t row = grp; row < p.n_rows; row += n_grp, parity ^= 1) {
        const uint16_t *zrow = p.logits + row * p.ld + (int64_t)vec_lo * 8;
        // the epilogue's dependent global reads (row info, then z_y), issued before pass 1
        // so that they do not stall the CTA at its end
        RowInfo ri_pre;
        uint16_t zy_pre = 0;
        if (warp == 0) {
            ri_pre = p.rowinfo[row];
            const int y_loc = ri_pre.target - vec_lo * 8;
            if (ri_pre.target >= 0 && ri_pre.target < p.V && y_loc >= 0 && y_loc < n_vec * 8)
                zy_pre = zrow[y_loc];
        }
        // ---- pass 1
        float a = -INFINITY;
        double s = 0.0;
        for (int bi = 0; bi < n_full; ++bi) {
            const uint4 *src = reinterpret_cast<const uint4 *>(zrow) + bi * BV + threadIdx.x;
            uint4 x[U];
#pragma unroll
            for (int j = 0; j < U; ++j)
                // vectors kept in shared memory are not re-read: let L2 evict them first
                x[j] = ldg_policy(src + j * NT, bi * U + j < cache_vecs ? pol_stream : pol_keep);
#pragma unroll
            for (int j = 0; j < U; ++j)
                if (bi * U + j < cache_vecs) row_cache[(bi * U + j) * NT + threadIdx.x] = x[j];
            B::reduce(x, a, s);
        }
        for (int bi = n_full; bi < n_batch; ++bi) {  // the checked last batch
            uint4 x[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int vi = bi * BV + j * NT + threadIdx.x;
                x[j] = vi < n_vec ? ldg_policy(zrow + (int64_t)vi * 8,
                                               bi * U + j < cache_vecs ? pol_stream : pol_keep)
                                  : neg_inf;
                if (vi == tail_vi) x[j] = mask_tail(x[j], tail_valid);
            }
#pragma unroll
            for (int j = 0; j < U; ++j)
                if (bi * U + j < cache_vecs) row_cache[(bi * U + j) * NT + threadIdx.x] = x[j];
            B::reduce(x, a, s);
        }
        warp_lse2_combine(a, s);
        if (lane == 0) red[warp] = RowPart{a, 0.0f, s};
        __syncthreads();
        if (warp == 0) {
            float cm = -INFINITY;
            double cs = 0.0;
            if (lane < NW) {
                cm = red[lane].a;
                cs = red[lane].s;
            }
            warp_lse2_combine(cm, cs);
            const RowInfo ri = ri_pre;
            const bool y_valid = ri.target >= 0 && ri.target < p.V;
            const int y_loc = ri.target - vec_lo * 8;
            const bool mine = y_valid && y_loc >= 0 && y_loc < n_vec * 8;
            float zy = mine ? __uint_as_float(((uint32_t)zy_pre) << 16) : 0.0f;
            if (C > 1) {
                // every CTA of the cluster gets this CTA's partial (and z_y if it owns y)
                if (lane < C) {
                    // (a, z_y, s fp64 with the holds-y bit in its sign)
                    const uint64_t sb = (uint64_t)__double_as_longlong(cs) | (mine ? (1ull << 63) : 0ull);
                    const uint32_t raddr = mapa_shared(smem_u32(&xpart[parity][crank]), lane);
                    asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(raddr),
                                 "r"(__float_as_uint(cm)), "r"(__float_as_uint(zy)), "r"((uint32_t)sb),
                                 "r"((uint32_t)(sb >> 32))
                                 : "memory");
                }
            }
            if (C == 1 && lane == 0) {
                const double l2s = row_l2s(cs, cm);
                const float lse2 = cm + (float)l2s;
                const float zyv = y_valid ? zy : __int_as_float(0x7FC00000);
                const double logp_d = row_logp(zyv, cm, l2s);
                const RowOut o = row_epilogue(logp_d, ri, p.eps_lo, p.eps_hi, p.grad_scale);
                const float logp = (float)logp_d;
                if (p.logp_out) p.logp_out[row] = logp;
                if (p.lse_out) p.lse_out[row] = lse2 * kLn2;
                if (p.scale_out) p.scale_out[row] = o.s;
                p.term_ws[row] = o.term;
                p.logp_ws[row] = logp;
                p.flag_ws[row] = o.flags;
                row_scalars[0] = lse2;
                row_scalars[1] = o.s;
                row_scalars[2] = o.gy;
                row_scalars[3] = __int_as_float(y_valid ? ri.target : -1);
            }
        }
        if (C > 1) {
            cluster_sync_all();  // the partials of every CTA of the cluster have landed
            if (warp == 0) {
                float M = -INFINITY, zsrc = 0.0f;
                double S = 0.0;
                bool own = false;
                if (lane < C) {
                    const uint4 m4 = reinterpret_cast<const uint4 &>(xpart[parity][lane]);
                    const uint64_t sb = ((uint64_t)m4.w << 32) | m4.z;
                    M = __uint_as_float(m4.x);
                    zsrc = __uint_as_float(m4.y);
                    S = __longlong_as_double((long long)(sb & ~(1ull << 63)));
                    own = (sb >> 63) != 0ull;
                }
                warp_lse2_combine(M, S);    // identical bits in every CTA of the cluster
                const uint32_t own_mask = __ballot_sync(0xFFFFFFFFu, own);
                const float zsh = __shfl_sync(0xFFFFFFFFu, zsrc, own_mask ? __ffs(own_mask) - 1 : 0);
                if (lane == 0) {
                    const RowInfo ri = p.rowinfo[row];
                    const bool y_valid = own_mask != 0u;
                    const float zyv = y_valid ? zsh : __int_as_float(0x7FC00000);
                    const double l2s = row_l2s(S, M);
                    const float lse2 = M + (float)l2s;
                    const double logp_d = row_logp(zyv, M, l2s);
                    const RowOut o = row_epilogue(logp_d, ri, p.eps_lo, p.eps_hi, p.grad_scale);
                    if (crank == 0) {
                        const float logp = (float)logp_d;
                        if (p.logp_out) p.logp_out[row] = logp;
                        if (p.lse_out) p.lse_out[row] = lse2 * kLn2;
                        if (p.scale_out) p.scale_out[row] = o.s;
                        p.term_ws[row] = o.term;
                        p.logp_ws[row] = logp;
                        p.flag_ws[row] = o.flags;
                    }
                    row_scalars[0] = lse2;
                    row_scalars[1] = o.s;
                    row_scalars[2] = o.gy;
                    row_scalars[3] = __int_as_float(y_valid ? ri.target : -1);
                }
            }
        }
        __syncthreads();
        // ---- pass 2: dlogits = s (softmax - onehot), written once
        if (p.dlogits) {
            const float lse2 = row_scalars[0], sc = row_scalars[1], gy = row_scalars[2];
            const auto gref = B::grad_ref(sc, lse2);
            const int32_t y = __float_as_int(row_scalars[3]);
            const int y_loc = y >= 0 ? y - vec_lo * 8 : -1;
            const int yv = (y_loc >= 0 && y_loc < n_vec * 8) ? (y_loc >> 3) : -1;
            uint16_t *drow = p.dlogits + row * p.ld + (int64_t)vec_lo * 8;
            uint4 *dst4 = reinterpret_cast<uint4 *>(drow);
            if (sc == 0.0f) {
                // clipped token or zero advantage: the row of dlogits is exactly zero
                const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
                for (int vi = threadIdx.x; vi < n_vec; vi += NT) {
                    if (vi == tail_vi) store_tail(drow + (int64_t)vi * 8, z4, tail_valid);
                    else stg_stream(dst4 + vi, z4);
                }
            } else {
                // batches newest first: the end of the slice is the part most likely still in
                // L2; the head of the slice comes from shared memory (cache_vecs per thread)
                for (int q = 0; q < n_batch; ++q) {
                    const int bi = n_batch - 1 - q;
                    const int v0 = bi * BV + threadIdx.x;
                    uint4 x[U];
                    if (bi < n_full) {
                        const uint4 *src = reinterpret_cast<const uint4 *>(zrow) + v0;
#pragma unroll
                        for (int j = 0; j < U; ++j)
                            x[j] = (bi * U + j < cache_vecs) ? row_cache[(bi * U + j) * NT + threadIdx.x]
                                                             : ldg_policy(src + j * NT, pol_stream);
#pragma unroll
                        for (int j = 0; j < U; ++j) stg_stream(dst4 + v0 + j * NT, B::grad_scaled(x[j], gref));
                    } else {
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            const int vi = v0 + j * NT;
                            x[j] = (bi * U + j < cache_vecs) ? row_cache[(bi * U + j) * NT + threadIdx.x]
                                   : (vi < n_vec ? ldg_policy(zrow + (int64_t)vi * 8, pol_stream) : neg_inf);
                        }
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            const int vi = v0 + j * NT;
                            if (vi >= n_vec) break;
                            const uint4 d = B::grad_scaled(x[j], gref);
                            if (vi == tail_vi) store_tail(drow + (int64_t)vi * 8, d, tail_valid);
                            else stg_stream(dst4 + vi, d);
                        }
                    }
                }
                // the target entry: s (p_y - 1) from the epilogue (fp64 expm1), by the thread
                // whose vector store covered it (program order keeps this store last)
                if (yv >= 0 && (yv % NT) == (int)threadIdx.x) {
                    drow[y_loc] = f2bf(gy);
                }
            }
        }
        __syncthreads();  // row_scalars / red / row_cache reused by the next row
    }
    if (C > 1) cluster_sync_all();  // no CTA leaves while a peer may still address its smem
}

cudaError_t launch_fused_rowwise(const LossArgs &a, const grpo_tune_t *tune, cudaStream_t s,
                                 int *launches, grpo_plan_t *plan) {
    if (a.n_rows == 0) return cudaSuccess;
    RowwiseParams p;
    p.logits = a.logits;
    p.dlogits = a.dlogits;
    p.ld = a.ld;
    p.V = a.V;
    p.n_rows = a.n_rows;
    p.rowinfo = a.rowinfo;
    p.eps_lo = a.eps_lo;
    p.eps_hi = a.eps_hi;
    p.grad_scale = a.grad_scale;
    p.logp_out = a.logp_out;
    p.lse_out = a.lse_out;
    p.scale_out = a.scale_out;
    p.term_ws = a.term_ws;
    p.logp_ws = a.logp_ws;
    p.flag_ws = a.flag_ws;
    p.prefetch = (tune && (tune->prefetch & 1)) ? 1 : 0;
    p.flags = 1;  // pass 2 newest-first (measured +2% over forward order, K3b)
    const int n_vec = (a.V + 7) / 8;
    // auto residency by row length (measured on B200): long rows
    // want 2 x 512-thread CTAs with 80 KB of row cache each; mid rows (V ~ 48k-112k, e.g.
    // the vocabulary shards of the tensor-parallel head) 4 x 256 threads; short rows 8.
    const int cps = (tune && tune->ctas_per_sm > 0) ? tune->ctas_per_sm
                                                    : (n_vec >= 14000 ? 2 : (n_vec >= 6000 ? 4 : 8));
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = 0;
    const int U = (tune && tune->stages > 0) ? tune->stages : (cps <= 4 ? 8 : 4);
    int nt = 0;
#define GRPO_RW(NT_, U_, C_)                                                               \
    if (nt == 0 && cps_nt == NT_ && U == U_ && Cl == C_) {                                 \
        nt = NT_;                                                                          \
        const size_t vec_bytes = (size_t)NT_ * 16;                                         \
        const size_t avail = (size_t)(227 * 1024) / cps - 4096;                            \
        const int rc = tune ? tune->row_cache : 0;                                         \
        /* auto: 160 KB of cache per SM; the rest of the 256 KB L1/smem stays L1, which  \
           stages the in-flight loads (more cache starves them: measured cliff)  */       \
        const size_t auto_bytes = (size_t)(160 * 1024) / cps;                              \
        int cv = rc > 0 ? rc : (rc == 0 ? (int)(auto_bytes / vec_bytes) : 0);             \
        const int nv = ((n_vec + C_ - 1) / C_ + NT_ - 1) / NT_;                            \
        if (cv > nv) cv = nv;                                                              \
        if ((size_t)cv * vec_bytes > avail) return cudaErrorInvalidConfiguration;          \
        p.cache_vecs = cv;                                                                 \
        smem = (size_t)cv * vec_bytes;                                                     \
        auto kern = rowwise_kernel<NT_, U_, C_>;                                           \
        cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                              (int)smem);                                  \
        if (ea != cudaSuccess) return ea;                                                  \
        cudaLaunchConfig_t cfg = {};                                                       \
        cudaLaunchAttribute attr[1];                                                       \
        attr[0].id = cudaLaunchAttributeClusterDimension;                                  \
        attr[0].val.clusterDim.x = C_;                                                     \
        attr[0].val.clusterDim.y = 1;                                                      \
        attr[0].val.clusterDim.z = 1;                                                      \
        cfg.blockDim = dim3(NT_);                                                          \
        cfg.dynamicSmemBytes = smem;                                                       \
        cfg.stream = s;                                                                    \
        cfg.attrs = attr;                                                                  \
        cfg.numAttrs = 1;                                                                  \
        int64_t groups = (int64_t)n_sm * cps / C_;                                         \
        if (groups > a.n_rows) groups = a.n_rows;                                          \
        blocks = groups * C_;                                                              \
        cfg.gridDim = dim3((unsigned)blocks);                                              \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT_, smem);              \
        ea = cudaLaunchKernelEx(&cfg, kern, p);                                            \
        if (ea != cudaSuccess) return ea;                                                  \
    }
    size_t smem = 0;
    int occ = 0;
    const int cps_nt = cps == 1 ? 1024 : (cps == 2 ? 512 : (cps == 3 ? 384 : 256));
    const int Cl = (tune && tune->cluster_size > 0) ? tune->cluster_size : 1;
    GRPO_RW(1024, 2, 1) GRPO_RW(1024, 4, 1) GRPO_RW(1024, 8, 1)
    GRPO_RW(512, 2, 1) GRPO_RW(512, 4, 1) GRPO_RW(512, 8, 1)
    GRPO_RW(384, 4, 1) GRPO_RW(384, 8, 1)
    GRPO_RW(256, 4, 1) GRPO_RW(256, 8, 1)
    GRPO_RW(1024, 4, 2) GRPO_RW(512, 8, 2) GRPO_RW(512, 4, 2) GRPO_RW(384, 8, 2)
    GRPO_RW(256, 8, 2) GRPO_RW(512, 8, 4) GRPO_RW(512, 4, 4) GRPO_RW(256, 8, 4)
#undef GRPO_RW
    if (nt == 0) return cudaErrorInvalidValue;
    if (plan) {
        *plan = grpo_plan_t{};
        plan->kernel = 2;
        plan->ctas_per_sm = cps;
        plan->cluster_size = Cl;
        plan->grid = (int32_t)blocks;
        plan->vec_per_thread = nt;
        plan->stages = p.cache_vecs;
        plan->max_clusters = occ;  // kernel 2: resident CTAs per SM the occupancy query allows
        plan->smem_bytes = (int32_t)smem;
    }
    *launches += 1;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ segmented reduce
// One CTA per trajectory i: its rows inside this chunk, summed in fp64 in a
// fixed order (thread-strided sequential sums, an xor butterfly per warp, then
// the warps in index order), so the result does not depend on scheduling.
// part[i*5 + {0..4}] = {inv_norm*sum term, inv_norm*sum |term|, sum logp,
// #clipped, #active}; traj_sum[i] += sum term when the chunk holds rows of i.
constexpr int kSegThreads = 256;

__global__ void __launch_bounds__(kSegThreads)
    segsum_kernel(int64_t row_begin, int64_t n_rows, const int64_t *__restrict__ cu, int32_t N,
                  const int32_t *__restrict__ traj_index, const float *__restrict__ inv_norm,
                  const double *__restrict__ term, const float *__restrict__ logp,
                  const uint8_t *__restrict__ flags, double *__restrict__ traj_sum,
                  double *__restrict__ part) {
    __shared__ double sh[5][kSegThreads / 32];
    const int64_t i = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t row_end = row_begin + n_rows;
    const int64_t b = max(cu[i], row_begin), e = min(cu[i + 1], row_end);
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t t = b + threadIdx.x; t < e; t += kSegThreads) {
        const int64_t k = t - row_begin;
        const double x = term[k];
        acc[0] += x;
        acc[1] += fabs(x);
        acc[2] += (double)logp[k];
        const uint8_t f = flags[k];
        acc[3] += (f & kRowClipped) ? 1.0 : 0.0;
        acc[4] += (f & kRowActive) ? 1.0 : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xFFFFFFFFu, acc[q], off);
        if (lane == 0) sh[q][warp] = acc[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot[5];
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            tot[q] = 0.0;
            for (int w = 0; w < kSegThreads / 32; ++w) tot[q] += sh[q][w];
        }
        const double wgt = (double)inv_norm[traj_index ? traj_index[i] : i];
        if (e > b) traj_sum[i] += tot[0];
        part[i * 5 + 0] = wgt * tot[0];
        part[i * 5 + 1] = wgt * tot[1];
        part[i * 5 + 2] = tot[2];
        part[i * 5 + 3] = tot[3];
        part[i * 5 + 4] = tot[4];
    }
}

// One CTA: fixed-order sums of the N partials into stats[] (deterministic).
__global__ void __launch_bounds__(1024) stats_kernel(int32_t N, int64_t n_rows,
                                                     const double *__restrict__ part,
                                                     double *__restrict__ stats) {
    __shared__ double sh[5][1024];
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t i = threadIdx.x; i < N; i += 1024)
#pragma unroll
        for (int q = 0; q < 5; ++q) acc[q] += part[i * 5 + q];
#pragma unroll
    for (int q = 0; q < 5; ++q) sh[q][threadIdx.x] = acc[q];
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
#pragma unroll
            for (int q = 0; q < 5; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        stats[GRPO_STAT_J] += sh[0][0];
        stats[GRPO_STAT_ABS] += sh[1][0];
        stats[GRPO_STAT_LOGP] += sh[2][0];
        stats[GRPO_STAT_CLIPPED] += sh[3][0];
        stats[GRPO_STAT_ACTIVE] += sh[4][0];
        stats[GRPO_STAT_ROWS] += (double)n_rows;
    }
}

cudaError_t launch_segment_reduce(const LossArgs &a, cudaStream_t s, int *launches) {
    segsum_kernel<<<(unsigned)a.N, kSegThreads, 0, s>>>(
        a.row_begin, a.n_rows, a.cu_seqlens, a.N, a.traj_index, a.inv_norm, a.term_ws, a.logp_ws,
        a.flag_ws, a.traj_sum, a.part_ws);
    stats_kernel<<<1, 1024, 0, s>>>(a.N, a.n_rows, a.part_ws, a.stats);
    *launches += 2;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ unfused backward
constexpr int kBwdVecPerThread = 4;

__global__ void __launch_bounds__(256)
    bwd_kernel(const uint16_t *__restrict__ logits, int64_t n_rows, int32_t V, int64_t ld,
               const int64_t *__restrict__ targets, const float *__restrict__ lse,
               const float *__restrict__ scale, float mult, uint16_t *dlogits,
               int32_t tiles_per_row) {
    const int n_vec = (V + 7) / 8;
    const int tail_valid = V - (n_vec - 1) * 8;
    const int64_t n_items = n_rows * tiles_per_row;
    const uint64_t pol_stream = policy_evict_first();
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t row = item / tiles_per_row;
        const int tile = (int)(item - row * tiles_per_row);
        const float sc = scale[row] * mult;
        const float off = lse[row] * kLog2e;
        const int64_t y = targets[row];
        const uint16_t *zrow = logits + row * ld;
        uint16_t *drow = dlogits + row * ld;
        const int v0 = tile * 256 * kBwdVecPerThread + threadIdx.x;
        // z_y is read before any store of this thread (dlogits may alias logits)
        const int yv = (y >= 0 && y < V) ? (int)(y >> 3) : -1;
        const bool y_mine = yv >= v0 && (yv - v0) % 256 == 0 && (yv - v0) / 256 < kBwdVecPerThread;
        const float zy = y_mine ? __uint_as_float(((uint32_t)zrow[y]) << 16) : 0.0f;
        uint4 x[kBwdVecPerThread];
#pragma unroll
        for (int j = 0; j < kBwdVecPerThread; ++j) {
            const int vi = v0 + j * 256;
            x[j] = (vi < n_vec && sc != 0.0f) ? ldg_policy(zrow + (int64_t)vi * 8, pol_stream)
                                              : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int j = 0; j < kBwdVecPerThread; ++j) {
            const int vi = v0 + j * 256;
            if (vi >= n_vec) break;
            uint4 d = make_uint4(0u, 0u, 0u, 0u);
            if (sc != 0.0f) {
                d.x = pack_bf16x2(sc * ex2(fmaf(bf_lo(x[j].x), kLog2e, -off)),
                                  sc * ex2(fmaf(bf_hi(x[j].x), kLog2e, -off)));
                d.y = pack_bf16x2(sc * ex2(fmaf(bf_lo(x[j].y), kLog2e, -off)),
                                  sc * ex2(fmaf(bf_hi(x[j].y), kLog2e, -off)));
                d.z = pack_bf16x2(sc * ex2(fmaf(bf_lo(x[j].z), kLog2e, -off)),
                                  sc * ex2(fmaf(bf_hi(x[j].z), kLog2e, -off)));
                d.w = pack_bf16x2(sc * ex2(fmaf(bf_lo(x[j].w), kLog2e, -off)),
                                  sc * ex2(fmaf(bf_hi(x[j].w), kLog2e, -off)));
            }
            if (vi == n_vec - 1 && tail_valid < 8) {
                store_tail(drow + (int64_t)vi * 8, d, tail_valid);
            } else {
                stg_stream(drow + (int64_t)vi * 8, d);
            }
            if (y_mine && yv == vi && sc != 0.0f) drow[y] = f2bf(sc * (ex2(fmaf(zy, kLog2e, -off)) - 1.0f));
        }
    }
}

cudaError_t launch_loss_bwd(const uint16_t *logits, int64_t n_rows, int32_t V, int64_t ld,
                            const int64_t *target_ids, const float *lse, const float *scale,
                            float mult, uint16_t *dlogits, cudaStream_t s, int *launches) {
    if (n_rows == 0) return cudaSuccess;
    const int n_vec = (V + 7) / 8;
    const int tiles = (n_vec + 256 * kBwdVecPerThread - 1) / (256 * kBwdVecPerThread);
    int64_t items = n_rows * tiles;
    int64_t blocks = items < 148 * 8 ? items : 148 * 8;
    bwd_kernel<<<(unsigned)blocks, 256, 0, s>>>(logits, n_rows, V, ld, target_ids, lse, scale,
                                                mult, dlogits, tiles);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace grpo
