// loss_vp.cu -- SURVEY NEXT(3): the fused loss for vocabulary-parallel logits, the
// way the paper's trainer (Megatron-LM) shards the LM head: rank q
// of a tensor-parallel group of R GPUs holds columns [q*Vs, (q+1)*Vs) of every
// row.  log pi_theta(y_t) needs the row's logsumexp over all R
// shards, so every row has one exchange of 16 bytes per rank; it is fused into the
// loss kernel over NVLink peer memory instead of a separate all-reduce:
//
//   pass 1 over the local shard (as rowwise_kernel) -> (a, s, z_y?) -> warp 0 stores
//   the 16-byte partial into row t's slot of EVERY rank's exchange buffer (peer
//   pointers) and, after a system-scope fence, adds 1 to that rank's arrival
//   counter for row t -> waits until its own counter for row t shows all R
//   partials (acquire, system scope) -> combines them in rank order (bit-identical
//   on every rank) -> epilogue -> pass 2 (dlogits of the local shard).
//
// Each rank's CTA g walks the same row sequence, so a row's partials are produced
// at about the same time on all ranks; a CTA waits on its peers for at most one row.
// Call e uses half e % 2 of the buffers and each rank re-zeroes its own counter of a
// row once it has read the row's partials (the protocol argument is at the re-arm).
// With fewer GPUs than ranks, one launch runs several ranks (n_local > 1) as a
// cooperative grid over one GPU's memory -- the protocol is identical.
#include <cstdio>

#include "common.cuh"
#include "rowwise.cuh"

namespace grpo {

struct VpParams {
    int32_t world, rank_begin, n_local, shard_cols;
    const uint16_t *logits[GRPO_VP_MAX_RANKS];
    uint16_t *dlogits[GRPO_VP_MAX_RANKS];
    float4 *xbuf[GRPO_VP_MAX_RANKS];
    uint32_t *flags[GRPO_VP_MAX_RANKS];
    int64_t half;     // (epoch % 2) * slots: the half of xbuf / flags this call uses
    int64_t ld;
    int32_t V;
    int64_t n_rows;
    const RowInfo *rowinfo;
    float eps_lo, eps_hi, grad_scale;
    float *logp_out, *lse_out, *scale_out, *term_ws, *logp_ws;
    uint8_t *flag_ws;
    int32_t cache_vecs;
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float4 ld_relaxed_sys_v4(const float4 *p) {
    float4 v;
    asm volatile("ld.relaxed.sys.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

template <int NT, int U>
__global__ void __launch_bounds__(NT, (NT >= 1024 ? 1 : 1024 / NT)) vp_kernel(const VpParams p) {
    using B = RowwiseBatch<NT, U>;
    constexpr int NW = NT / 32;
    constexpr int BV = NT * U;
    __shared__ float2 red[NW];
    __shared__ float row_scalars[4];
    extern __shared__ uint4 row_cache[];
    const int g_per = gridDim.x / p.n_local;
    const int lr = blockIdx.x / g_per;          // local rank of this CTA
    const int g = blockIdx.x - lr * g_per;
    const int rank = p.rank_begin + lr;
    const int32_t c0 = rank * p.shard_cols;     // first vocabulary column of this shard
    const int32_t vc = max(0, min(p.shard_cols, p.V - c0));
    const int n_vec = (vc + 7) / 8;
    const int tail_valid = vc - (n_vec - 1) * 8;
    const int tail_vi = (n_vec > 0 && tail_valid < 8) ? n_vec - 1 : -1;
    const int n_batch = (n_vec + BV - 1) / BV;
    const int n_full = tail_vi >= 0 ? tail_vi / BV : n_vec / BV;
    const int cache_vecs = min(p.cache_vecs, n_batch * U);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    const uint4 neg_inf = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair,
                                     kBf16NegInfPair);
    const uint16_t *shard = p.logits[lr];
    uint16_t *dshard = p.dlogits[lr];
    for (int64_t row = g; row < p.n_rows; row += g_per) {
        const uint16_t *zrow = shard + row * p.ld;
        // ---- pass 1 over the local shard
        float a = -INFINITY, s = 0.0f;
        for (int bi = 0; bi < n_full; ++bi) {
            const uint4 *src = reinterpret_cast<const uint4 *>(zrow) + bi * BV + threadIdx.x;
            uint4 x[U];
#pragma unroll
            for (int j = 0; j < U; ++j)
                x[j] = ldg_policy(src + j * NT, bi * U + j < cache_vecs ? pol_stream : pol_keep);
#pragma unroll
            for (int j = 0; j < U; ++j)
                if (bi * U + j < cache_vecs) row_cache[(bi * U + j) * NT + threadIdx.x] = x[j];
            B::reduce(x, a, s);
        }
        for (int bi = n_full; bi < n_batch; ++bi) {
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
        if (lane == 0) red[warp] = make_float2(a, s);
        __syncthreads();
        if (warp == 0) {
            float cm = -INFINITY, cs = 0.0f;
            if (lane < NW) {
                cm = red[lane].x;
                cs = red[lane].y;
            }
            warp_lse2_combine(cm, cs);
            const RowInfo ri = p.rowinfo[row];
            const int y_loc = ri.target - c0;
            const bool mine = ri.target >= 0 && ri.target < p.V && y_loc >= 0 && y_loc < vc;
            const float zy = mine ? __uint_as_float(((uint32_t)zrow[y_loc]) << 16) : 0.0f;
            // ---- the exchange: this rank's partial into row `row` of every rank's buffer
            const int64_t slot = p.half + row;
            if (lane < p.world) {
                float4 *dst = p.xbuf[lane] + slot * p.world + rank;
                asm volatile("st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst),
                             "f"(cm), "f"(cs), "f"(zy), "f"(mine ? 1.0f : 0.0f)
                             : "memory");
                __threadfence_system();
                atomicAdd_system(p.flags[lane] + slot, 1u);
                // wait for all world partials of this row in this rank's buffer
                const uint32_t *f = p.flags[rank] + slot;
                long long spins = 0;
                while (ld_acquire_sys(f) < (uint32_t)p.world) {
                    __nanosleep(64);
                    if (++spins > (1ll << 27)) __trap();  // a peer never arrived: fail, don't hang
                }
            }
            __syncwarp();
            float M = -INFINITY, S = 0.0f, zsrc = 0.0f;
            bool own = false;
            if (lane < p.world) {
                const float4 m4 = ld_relaxed_sys_v4(p.xbuf[rank] + slot * p.world + lane);
                M = m4.x;
                S = m4.y;
                zsrc = m4.z;
                own = m4.w != 0.0f;
            }
            __syncwarp();
            // re-arm this rank's counter.  The next arrival on this slot belongs to call
            // e+2, which a peer can only start after seeing this rank's partial of call
            // e+1 -- released (fence.sc.sys) after this store in program order.
            if (lane == 0)
                asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p.flags[rank] + slot), "r"(0u)
                             : "memory");
            warp_lse2_combine(M, S);  // same inputs in the same lanes on every rank
            const uint32_t own_mask = __ballot_sync(0xFFFFFFFFu, own);
            const float zsh = __shfl_sync(0xFFFFFFFFu, zsrc, own_mask ? __ffs(own_mask) - 1 : 0);
            if (lane == 0) {
                const bool y_valid = own_mask != 0u;
                const float zyv = y_valid ? zsh : __int_as_float(0x7FC00000);
                const float l2s = log2f(S);
                const float lse2 = M + l2s;
                const double logp_d = row_logp(zyv, M, l2s);
                const RowOut o = row_epilogue(logp_d, ri, p.eps_lo, p.eps_hi, p.grad_scale);
                if (lr == 0) {  // per-row outputs: identical on every rank, written once per call
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
                row_scalars[2] = zyv;
                row_scalars[3] = __int_as_float(mine ? y_loc : -1);
            }
        }
        __syncthreads();
        // ---- pass 2: dlogits of the local shard
        if (dshard) {
            const float lse2 = row_scalars[0], sc = row_scalars[1], zy = row_scalars[2];
            const int32_t y_loc = __float_as_int(row_scalars[3]);
            const int yv = y_loc >= 0 ? (y_loc >> 3) : -1;
            uint16_t *drow = dshard + row * p.ld;
            uint4 *dst4 = reinterpret_cast<uint4 *>(drow);
            if (sc == 0.0f) {
                const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
                for (int vi = threadIdx.x; vi < n_vec; vi += NT) {
                    if (vi == tail_vi) store_tail(drow + (int64_t)vi * 8, z4, tail_valid);
                    else stg_stream(dst4 + vi, z4);
                }
            } else {
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
                        for (int j = 0; j < U; ++j) stg_stream(dst4 + v0 + j * NT, B::grad(x[j], sc, lse2));
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
                            const uint4 d = B::grad(x[j], sc, lse2);
                            if (vi == tail_vi) store_tail(drow + (int64_t)vi * 8, d, tail_valid);
                            else stg_stream(dst4 + vi, d);
                        }
                    }
                }
                if (yv >= 0 && (yv % NT) == (int)threadIdx.x) {
                    const float py = ex2(fmaf(zy, kLog2e, -lse2));
                    drow[y_loc] = f2bf(sc * (py - 1.0f));
                }
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_vp(const LossArgs &a, const grpo_vp_comm_t *comm, cudaStream_t s, int *launches,
                      grpo_plan_t *plan, char *why, size_t why_len) {
    if (a.n_rows == 0) return cudaSuccess;
    constexpr int NT = 512, U = 8, CPS = 2;
    VpParams p = {};
    p.world = comm->world;
    p.rank_begin = comm->rank_begin;
    p.n_local = comm->n_local;
    p.shard_cols = comm->shard_cols;
    for (int q = 0; q < comm->n_local; ++q) {
        p.logits[q] = comm->logits[q];
        p.dlogits[q] = comm->dlogits[q];
    }
    for (int q = 0; q < comm->world; ++q) {
        p.xbuf[q] = static_cast<float4 *>(comm->xbuf[q]);
        p.flags[q] = comm->flags[q];
    }
    p.half = (int64_t)(comm->epoch & 1u) * comm->slots;
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
    const int n_vec = (comm->shard_cols + 7) / 8;
    int cv = (int)((size_t)(160 * 1024) / CPS / ((size_t)NT * 16));
    const int nv = (n_vec + NT - 1) / NT;
    if (cv > nv) cv = nv;
    p.cache_vecs = cv;
    const size_t smem = (size_t)cv * NT * 16;
    auto kern = vp_kernel<NT, U>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, n_sm = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    // every CTA must be resident (a CTA may wait for a peer rank's CTA of the same index)
    int64_t g_per = (int64_t)n_sm * (occ < CPS ? occ : CPS) / comm->n_local;
    if (g_per > a.n_rows) g_per = a.n_rows;
    if (g_per < 1) {
        if (why) snprintf(why, why_len, "vp kernel: no resident CTA per local rank");
        return cudaErrorInvalidConfiguration;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)(g_per * comm->n_local));
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p);
    if (e != cudaSuccess) return e;
    if (plan) {
        *plan = grpo_plan_t{};
        plan->kernel = 3;
        plan->ctas_per_sm = CPS;
        plan->grid = (int32_t)(g_per * comm->n_local);
        plan->vec_per_thread = NT;
        plan->stages = cv;
        plan->max_clusters = occ;
        plan->smem_bytes = (int32_t)smem;
    }
    *launches += 1;
    return cudaSuccess;
}

}  // namespace grpo
