// loss_vp.cu -- SURVEY NEXT(3): the fused loss for vocabulary-parallel logits, the
// way the paper's trainer (Megatron-LM) shards the LM head: rank q
// of a tensor-parallel group of R GPUs holds columns [q*Vs, (q+1)*Vs) of every
// row.  log pi_theta(y_t) needs the row's logsumexp over all R
// shards, so every row has one exchange of 16 bytes per rank; it is fused into the
// loss kernel over NVLink peer memory instead of a separate all-reduce:
//
//   pass 1 over the local shard (as rowwise_kernel) -> (a, s, z_y?) -> warp 0 stores
//   the 32-byte tagged partial into row t's slot of EVERY rank's exchange buffer
//   (peer pointers) -> waits until its own buffer holds all R partials of row t with
//   this call's tag -> combines them in rank order (bit-identical on every rank) ->
//   epilogue -> pass 2 (dlogits of the local shard).
//
// Each rank's CTA g walks the same row sequence, so a row's partials are produced
// at about the same time on all ranks; a CTA waits on its peers for at most one row.
// Call e uses half e % 2 of the buffers with tag e + 1.  A peer can only write call
// e+2's partial of row t (the same half) after completing call e+1, which needs this
// rank's call-e+1 partial of row t, which this rank posts after it has finished
// reading call e: a slot is never overwritten before it is read.
// With fewer GPUs than ranks, one launch runs several ranks (n_local > 1) as a
// cooperative grid over one GPU's memory -- the protocol is identical.
#include <cstdio>

#include "common.cuh"
#include "rowwise.cuh"
#include "tc.cuh"

namespace grpo {

struct VpParams {
    int32_t world, rank_begin, n_local, shard_cols;
    const uint16_t *logits[GRPO_VP_MAX_RANKS];
    uint16_t *dlogits[GRPO_VP_MAX_RANKS];
    ulonglong2 *xbuf[GRPO_VP_MAX_RANKS];
    int64_t half;     // (epoch % 2) * slots: the half of xbuf this call uses
    uint32_t tag;     // epoch + 1: marks this call's words (0 = never written)
    unsigned long long *row_ctr;  // [n_local] next row to take (zeroed before the launch)
    int dynamic;      // 1: CTAs take rows from row_ctr; 0: CTA g takes g, g + g_per, ...
    int64_t ld;
    int32_t V;
    int64_t n_rows;
    const RowInfo *rowinfo;
    float eps_lo, eps_hi, grad_scale;
    float *logp_out, *lse_out, *scale_out;
    double *term_ws;
    float *logp_ws;
    uint8_t *flag_ws;
    int32_t cache_vecs;
};

__device__ __forceinline__ void st_relaxed_sys_v2(ulonglong2 *p, uint64_t a, uint64_t b) {
    asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ ulonglong2 ld_relaxed_sys_v2(const ulonglong2 *p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}

// LAG = 1 defers the wait: the partial of row k is posted right after its pass 1,
// and the CTA waits for the peers' partials of row k-1 only after pass 1 of row k --
// a whole pass of slack for the peer skew and the NVLink latency.  The row cache is
// split into two halves (rows alternate) so that row k-1's head is still there for
// its pass 2.
template <int NT, int U, int LAG>
__global__ void __launch_bounds__(NT, (NT >= 1024 ? 1 : 1024 / NT)) vp_kernel(const VpParams p) {
    using B = RowwiseBatch<NT, U>;
    constexpr int NW = NT / 32;
    constexpr int BV = NT * U;
    __shared__ RowPart red[NW];
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
    const int half_vecs = LAG ? p.cache_vecs / 2 : p.cache_vecs;  // per thread, per row
    const int cache_vecs = min(half_vecs, n_batch * U);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
    const uint4 neg_inf = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair,
                                     kBf16NegInfPair);
    const uint16_t *shard = p.logits[lr];
    uint16_t *dshard = p.dlogits[lr];

    // pass 1 of `row` into `cache`, then warp 0 posts the row's partial to every rank
    auto pass1 = [&](int64_t row, uint4 *cache) {
        const uint16_t *zrow = shard + row * p.ld;
        float a = -INFINITY;
        double s = 0.0;
        for (int bi = 0; bi < n_full; ++bi) {
            const uint4 *src = reinterpret_cast<const uint4 *>(zrow) + bi * BV + threadIdx.x;
            uint4 x[U];
#pragma unroll
            for (int j = 0; j < U; ++j)
                x[j] = ldg_policy(src + j * NT, bi * U + j < cache_vecs ? pol_stream : pol_keep);
#pragma unroll
            for (int j = 0; j < U; ++j)
                if (bi * U + j < cache_vecs) cache[(bi * U + j) * NT + threadIdx.x] = x[j];
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
                if (bi * U + j < cache_vecs) cache[(bi * U + j) * NT + threadIdx.x] = x[j];
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
            const int32_t y = p.rowinfo[row].target;
            const int y_loc = y - c0;
            const bool mine = y >= 0 && y < p.V && y_loc >= 0 && y_loc < vc;
            const float zy = mine ? __uint_as_float(((uint32_t)zrow[y_loc]) << 16) : 0.0f;
            // ---- the exchange: this rank's partial into row `row` of every rank's buffer.
            // Each 64-bit word carries the call's tag next to its payload, and 64-bit
            // accesses are single-copy atomic: a reader that sees the tag in all four
            // words has the whole message -- no fence, no counter, no flag to re-arm.
            if (lane < p.world) {
                const uint64_t hi = (uint64_t)p.tag << 32;
                ulonglong2 *dst = p.xbuf[lane] + ((p.half + row) * p.world + rank) * 2;
                const uint64_t sb = (uint64_t)__double_as_longlong(cs) | (mine ? (1ull << 63) : 0ull);
                st_relaxed_sys_v2(dst, hi | __float_as_uint(cm), hi | (uint32_t)sb);
                st_relaxed_sys_v2(dst + 1, hi | (uint32_t)(sb >> 32), hi | __float_as_uint(zy));
            }
        }
    };

    // wait for all partials of `row`, combine, epilogue, pass 2 from `cache`
    auto finish = [&](int64_t row, const uint4 *cache) {
        const uint16_t *zrow = shard + row * p.ld;
        if (warp == 0) {
            float M = -INFINITY, zsrc = 0.0f;
            double S = 0.0;
            bool own = false;
            if (lane < p.world) {
                const ulonglong2 *src = p.xbuf[rank] + ((p.half + row) * p.world + lane) * 2;
                ulonglong2 w0, w1;
                long long spins = 0;
                for (;;) {
                    w0 = ld_relaxed_sys_v2(src);
                    w1 = ld_relaxed_sys_v2(src + 1);
                    if ((uint32_t)(w0.x >> 32) == p.tag && (uint32_t)(w0.y >> 32) == p.tag &&
                        (uint32_t)(w1.x >> 32) == p.tag && (uint32_t)(w1.y >> 32) == p.tag)
                        break;
                    __nanosleep(32);
                    if (++spins > (1ll << 27)) __trap();  // a peer never arrived: fail, don't hang
                }
                // (a, s fp64 with the holds-y bit in its sign, z_y)
                const uint64_t sb = ((w1.x & 0xFFFFFFFFull) << 32) | (w0.y & 0xFFFFFFFFull);
                M = __uint_as_float((uint32_t)w0.x);
                S = __longlong_as_double((long long)(sb & ~(1ull << 63)));
                own = (sb >> 63) != 0ull;
                zsrc = __uint_as_float((uint32_t)w1.y);
            }
            warp_lse2_combine(M, S);  // same inputs in the same lanes on every rank
            const uint32_t own_mask = __ballot_sync(0xFFFFFFFFu, own);
            const float zsh = __shfl_sync(0xFFFFFFFFu, zsrc, own_mask ? __ffs(own_mask) - 1 : 0);
            if (lane == 0) {
                const RowInfo ri = p.rowinfo[row];
                const int y_loc = ri.target - c0;
                const bool mine = ri.target >= 0 && ri.target < p.V && y_loc >= 0 && y_loc < vc;
                const bool y_valid = own_mask != 0u;
                const float zyv = y_valid ? zsh : __int_as_float(0x7FC00000);
                const double l2s = row_l2s(S, M);
                const float lse2 = M + (float)l2s;
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
                row_scalars[2] = o.gy;
                row_scalars[3] = __int_as_float(mine ? y_loc : -1);
            }
        }
        __syncthreads();
        // ---- pass 2: dlogits of the local shard
        if (dshard) {
            const float lse2 = row_scalars[0], sc = row_scalars[1], gy = row_scalars[2];
            const auto gref = B::grad_ref(sc, lse2);
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
                            x[j] = (bi * U + j < cache_vecs) ? cache[(bi * U + j) * NT + threadIdx.x]
                                                             : ldg_policy(src + j * NT, pol_stream);
#pragma unroll
                        for (int j = 0; j < U; ++j) stg_stream(dst4 + v0 + j * NT, B::grad_scaled(x[j], gref));
                    } else {
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            const int vi = v0 + j * NT;
                            x[j] = (bi * U + j < cache_vecs) ? cache[(bi * U + j) * NT + threadIdx.x]
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
                if (yv >= 0 && (yv % NT) == (int)threadIdx.x) {
                    drow[y_loc] = f2bf(gy);
                }
            }
        }
        __syncthreads();
    };

    // rows: static (CTA g takes g, g + g_per, ...) or dynamic (in the order CTAs ask for
    // them; every rank hands out rows in increasing order and posts a row's partial
    // before it waits for anything, so a waited-for row is always eventually posted)
    __shared__ int64_t next_row[2];
    auto take = [&](int64_t cur, int slot) {
        if (threadIdx.x == 0)
            next_row[slot] = p.dynamic ? (int64_t)atomicAdd(p.row_ctr + lr, 1ull) : cur + g_per;
    };
    if (threadIdx.x == 0) next_row[0] = p.dynamic ? (int64_t)atomicAdd(p.row_ctr + lr, 1ull) : g;
    __syncthreads();
    int k = 0;
    int64_t row = next_row[0];
    if (LAG == 0) {
        while (row < p.n_rows) {
            take(row, (k + 1) & 1);
            pass1(row, row_cache);
            finish(row, row_cache);  // ends with __syncthreads: next_row is visible
            row = next_row[(++k) & 1];
        }
    } else {
        const int half_stride = half_vecs * NT;
        int64_t prev = -1;
        while (row < p.n_rows) {
            take(row, (k + 1) & 1);
            pass1(row, row_cache + (k & 1) * half_stride);
            if (prev >= 0) finish(prev, row_cache + ((k - 1) & 1) * half_stride);
            else __syncthreads();
            prev = row;
            row = next_row[(++k) & 1];
        }
        if (prev >= 0) finish(prev, row_cache + ((k - 1) & 1) * half_stride);
    }
}

// The same exchange inside the streamed ring kernel (K3c, loss_stream.cu), with K3c's three
// roles: one producer thread per CTA moves the local shard's rows with bulk copies into a
// FIFO ring of NS slots (pass-1 chunks of row k, the first LA chunks of row k+1, the
// re-loads of row k); the consumers run pass 1, publish their warp partials on an mbarrier,
// stream row k+1's first LA chunks and then run pass 2 of row k; the epilogue warp combines
// the warp partials, posts the row's partial to every rank, polls its own buffer for the
// group's partials (sleeping between polls), combines them in rank order, runs the fp64
// epilogue and hands (lse2, s, g_y, y) to pass 2.  The wait for the peers thus sits in the
// epilogue warp, overlapped with the look-ahead, instead of stopping the consumers after
// every row's pass 1.  Static rows only (CTA g of every rank takes rows g, g + g_per, ...);
// lag and dynamic_rows select the row-wise kernel.
template <int NT, int MINB, int CHUNK_VECS>
__global__ void __launch_bounds__(NT + 64, MINB) vp_stream_kernel(const VpParams p, const int ns,
                                                                   const int pf, const int la) {
    constexpr int CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr int U = CHUNK_VECS / NT;
    constexpr int NW = NT / 32;
    using B = RowwiseBatch<NT, U>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint4 *ring = reinterpret_cast<uint4 *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)ns * CHUNK_BYTES);
    uint64_t *empty = full + ns;
    __shared__ RowPart red[2][NW];
    __shared__ float4 scal[2];
    __shared__ __align__(8) uint64_t part_bar[2];
    __shared__ __align__(8) uint64_t scal_bar[2];
    const int g_per = gridDim.x / p.n_local;
    const int lr = blockIdx.x / g_per;  // local rank of this CTA
    const int g = blockIdx.x - lr * g_per;
    const int rank = p.rank_begin + lr;
    const int32_t c0 = rank * p.shard_cols;  // first vocabulary column of this shard
    const int32_t vc = max(0, min(p.shard_cols, p.V - c0));
    const int n_vec = (vc + 7) / 8;
    const int n = (n_vec + CHUNK_VECS - 1) / CHUNK_VECS;  // chunks per row
    const uint16_t *shard = p.logits[lr];
    uint16_t *dshard = p.dlogits[lr];
    const bool two_pass = dshard != nullptr;
    const int R = two_pass ? min(n, max(0, ns - pf)) : 0;  // chunks resident after pass 1
    const int LA = two_pass ? max(0, min(la, min(ns - R, n - R))) : 0;
    const int tail_valid = vc - (n_vec - 1) * 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int q = 0; q < ns; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, NW);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(part_bar + b, NW);
            mbar_init(scal_bar + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {
        // ------------------------------------------------------------ producer
        if (lane == 0 && n > 0) {
            const uint64_t pol_keep = policy_evict_last(), pol_once = policy_evict_first();
            const int64_t row_bytes = (int64_t)n_vec * 16;
            int slot = 0;
            uint32_t par = 0;
            auto load = [&](int64_t row, int c, bool reload) {
                const uint8_t *src = reinterpret_cast<const uint8_t *>(shard + row * p.ld);
                mbar_wait_sleep(empty + slot, par ^ 1u, 64);
                const int64_t off = (int64_t)c * CHUNK_BYTES;
                const uint32_t bytes = (uint32_t)(row_bytes - off < CHUNK_BYTES ? row_bytes - off : CHUNK_BYTES);
                const uint64_t pol = (!reload && c < n - R && two_pass) ? pol_keep : pol_once;
                mbar_arrive_expect_tx(full + slot, bytes);
                bulk_g2s(ring + (size_t)slot * CHUNK_VECS, src + off, bytes, full + slot, pol);
                if (++slot == ns) {
                    slot = 0;
                    par ^= 1u;
                }
            };
            for (int64_t row = g; row < p.n_rows; row += g_per) {
                for (int c = (row == g ? 0 : LA); c < n; ++c) load(row, c, false);
                if (row + g_per < p.n_rows)
                    for (int c = 0; c < LA; ++c) load(row + g_per, c, false);
                if (two_pass)
                    for (int c = 0; c < n - R; ++c) load(row, c, true);
            }
        }
        return;
    }

    if (warp == NW + 1) {
        // ------------------------------------------------------------ epilogue warp
        uint32_t rowk = 0;
        for (int64_t row = g; row < p.n_rows; row += g_per, ++rowk) {
            const int b = rowk & 1;
            const uint32_t ph = (rowk >> 1) & 1u;
            RowInfo ri;
            uint16_t zy_bits = 0;
            int32_t y_loc = -1;
            bool mine = false;
            if (lane == 0) {
                ri = p.rowinfo[row];
                y_loc = ri.target - c0;
                mine = ri.target >= 0 && ri.target < p.V && y_loc >= 0 && y_loc < vc;
                if (mine) zy_bits = shard[row * p.ld + y_loc];
            }
            if (n > 0) mbar_wait_sleep(part_bar + b, ph, 128);
            float cm = (n > 0 && lane < NW) ? red[b][lane].a : -INFINITY;
            double cs = (n > 0 && lane < NW) ? red[b][lane].s : 0.0;
            warp_lse2_combine(cm, cs);
            const bool own_y = __shfl_sync(0xFFFFFFFFu, mine, 0);
            const float zy = own_y ? __uint_as_float(((uint32_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)zy_bits, 0)) << 16)
                                   : 0.0f;
            // ---- the exchange (tagged 64-bit words, see vp_kernel)
            if (lane < p.world) {
                const uint64_t hi = (uint64_t)p.tag << 32;
                ulonglong2 *dst = p.xbuf[lane] + ((p.half + row) * p.world + rank) * 2;
                const uint64_t sb = (uint64_t)__double_as_longlong(cs) | (own_y ? (1ull << 63) : 0ull);
                st_relaxed_sys_v2(dst, hi | __float_as_uint(cm), hi | (uint32_t)sb);
                st_relaxed_sys_v2(dst + 1, hi | (uint32_t)(sb >> 32), hi | __float_as_uint(zy));
            }
            float M = -INFINITY, zsrc = 0.0f;
            double S = 0.0;
            bool own = false;
            if (lane < p.world) {
                const ulonglong2 *src = p.xbuf[rank] + ((p.half + row) * p.world + lane) * 2;
                ulonglong2 w0, w1;
                long long spins = 0;
                for (;;) {
                    w0 = ld_relaxed_sys_v2(src);
                    w1 = ld_relaxed_sys_v2(src + 1);
                    if ((uint32_t)(w0.x >> 32) == p.tag && (uint32_t)(w0.y >> 32) == p.tag &&
                        (uint32_t)(w1.x >> 32) == p.tag && (uint32_t)(w1.y >> 32) == p.tag)
                        break;
                    __nanosleep(32);
                    if (++spins > (1ll << 27)) __trap();  // a peer never arrived: fail, don't hang
                }
                // (a, s fp64 with the holds-y bit in its sign, z_y)
                const uint64_t sb = ((w1.x & 0xFFFFFFFFull) << 32) | (w0.y & 0xFFFFFFFFull);
                M = __uint_as_float((uint32_t)w0.x);
                S = __longlong_as_double((long long)(sb & ~(1ull << 63)));
                own = (sb >> 63) != 0ull;
                zsrc = __uint_as_float((uint32_t)w1.y);
            }
            warp_lse2_combine(M, S);  // same inputs in the same lanes on every rank
            const uint32_t own_mask = __ballot_sync(0xFFFFFFFFu, own);
            const float zsh = __shfl_sync(0xFFFFFFFFu, zsrc, own_mask ? __ffs(own_mask) - 1 : 0);
            if (lane == 0) {
                const float zyv = own_mask != 0u ? zsh : __int_as_float(0x7FC00000);
                const double l2s = row_l2s(S, M);
                const float lse2 = M + (float)l2s;
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
                scal[b] = make_float4(lse2, o.s, o.gy, __int_as_float(mine ? y_loc : -1));
                mbar_arrive(scal_bar + b);
            }
            __syncwarp();
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const uint4 neg_inf = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair);
    int slot = 0;
    uint32_t par = 0;
    auto pass1_chunk = [&](int c, bool last, float &a, double &s) {
        const int sl = slot;
        mbar_wait(full + sl, par);
        if (++slot == ns) {
            slot = 0;
            par ^= 1u;
        }
        const uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;
        uint4 x[U];
#pragma unroll
        for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
        if (last) {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int vi = c * CHUNK_VECS + j * NT + threadIdx.x;
                if (vi >= n_vec) x[j] = neg_inf;
                else if (vi == n_vec - 1 && tail_valid < 8) x[j] = mask_tail(x[j], tail_valid);
            }
        }
        B::reduce(x, a, s);
        if (c < n - R) {
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + sl);
        }
    };
    float a = -INFINITY;
    double s = 0.0;
    if (g < p.n_rows)
        for (int c = 0; c < LA; ++c) pass1_chunk(c, c == n - 1, a, s);
    uint32_t rowk = 0;
    for (int64_t row = g; row < p.n_rows; row += g_per, ++rowk) {
        const int b = rowk & 1;
        const int res_base = slot;  // slot of this row's chunk LA (chunks LA..n-1 are contiguous loads)
#pragma unroll 1
        for (int c = LA; c < n - 1; ++c) pass1_chunk(c, false, a, s);
        if (n - 1 >= LA && n > 0) pass1_chunk(n - 1, true, a, s);
        warp_lse2_combine(a, s);
        if (!two_pass && rowk >= 2) mbar_wait(scal_bar + b, ((rowk - 2) >> 1) & 1u);
        if (lane == 0 && n > 0) {
            red[b][warp] = RowPart{a, 0.0f, s};
            mbar_arrive(part_bar + b);
        }
        a = -INFINITY;
        s = 0.0;
        if (row + g_per < p.n_rows)
            for (int c = 0; c < LA; ++c) pass1_chunk(c, c == n - 1, a, s);
        if (!two_pass) continue;
        // ---- pass 2: resident chunks n-R..n-1, then the re-loads
        mbar_wait(scal_bar + b, (rowk >> 1) & 1u);
        const float4 sc4 = scal[b];
        const float lse2 = sc4.x, sc = sc4.y, gy = sc4.z;
        const auto gref = B::grad_ref(sc, lse2);
        const int32_t y = __float_as_int(sc4.w);
        const int y_chunk = y >= 0 ? (y >> 3) / CHUNK_VECS : -1;
        uint16_t *drow = dshard + row * p.ld;
        uint4 *dst4 = reinterpret_cast<uint4 *>(drow);
        for (int i = 0; i < n; ++i) {
            const bool resident = i < R;
            const int c = resident ? n - R + i : i - R;
            int sl;
            if (resident) {
                sl = (res_base + (c - LA)) % ns;
            } else {
                sl = slot;
                mbar_wait(full + sl, par);
                if (++slot == ns) {
                    slot = 0;
                    par ^= 1u;
                }
            }
            const uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;
            const int v0 = c * CHUNK_VECS + threadIdx.x;
            if (c != n - 1) {
                if (sc == 0.0f) {
#pragma unroll
                    for (int j = 0; j < U; ++j) stg_stream(dst4 + v0 + j * NT, make_uint4(0u, 0u, 0u, 0u));
                } else {
                    uint4 x[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
#pragma unroll
                    for (int j = 0; j < U; ++j) stg_stream(dst4 + v0 + j * NT, B::grad_scaled(x[j], gref));
                }
            } else {
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int vi = v0 + j * NT;
                    if (vi >= n_vec) break;
                    const uint4 d = sc == 0.0f ? make_uint4(0u, 0u, 0u, 0u)
                                               : B::grad_scaled(chunk[j * NT + threadIdx.x], gref);
                    if (vi == n_vec - 1 && tail_valid < 8) store_tail(drow + (int64_t)vi * 8, d, tail_valid);
                    else stg_stream(dst4 + vi, d);
                }
            }
            if (y_chunk == c && sc != 0.0f && ((y >> 3) - c * CHUNK_VECS) % NT == (int)threadIdx.x) {
                drow[y] = f2bf(gy);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + sl);
        }
    }
}

// The ring kernel with the pass 2 of every row DELAYED by D rows (grpo_vp_comm_t.lag = D + 1,
// D = 1..3): the consumers run pass 1 of row k, post its warp partials and then pass 2 of row
// k - D, so the exchange of a row -- posting its partial, waiting for the slowest peer rank --
// runs in the epilogue warp under D rows of streaming instead of under a look-ahead of one
// chunk.  No chunk stays resident: pass 1 streams row k with L2 evict_last and pass 2
// re-loads row k - D (evict_first), which (D + 1) x 74 KB x 296 CTAs (R = 4 at V = 152064;
// 44 MB at D = 1) keeps in L2.  The producer's order is P1(0) .. P1(D-1), then P1(k), RL(k-D)
// for k >= D, then the last D re-loads; the row partials, token scales and their mbarriers
// are rings of NB = D + 1 (row k uses buffer k mod NB; the consumers' pass 2 of row k-D
// precedes their partial of row k+1, and the epilogue warp handles rows in order, so a
// buffer is free again when it is rewritten).  Same combine order: bit-identical outputs.
template <int NT, int MINB, int CHUNK_VECS>
__global__ void __launch_bounds__(NT + 96, MINB) vp_delay_kernel(const VpParams p, const int ns, const int D) {
    constexpr int CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr int U = CHUNK_VECS / NT;
    constexpr int NW = NT / 32;
    constexpr int NBMAX = 4;
    using B = RowwiseBatch<NT, U>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint4 *ring = reinterpret_cast<uint4 *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)ns * CHUNK_BYTES);
    uint64_t *empty = full + ns;
    uint64_t *wrote = empty + ns;  // pass-2 uses: NW warp arrivals, the slot holds dlogits
    __shared__ RowPart red[NBMAX][NW];
    __shared__ float4 scal[NBMAX];
    __shared__ __align__(8) uint64_t part_bar[NBMAX];
    __shared__ __align__(8) uint64_t scal_bar[NBMAX];
    const int NB = D + 1;
    const int g_per = gridDim.x / p.n_local;
    const int lr = blockIdx.x / g_per;  // local rank of this CTA
    const int g = blockIdx.x - lr * g_per;
    const int rank = p.rank_begin + lr;
    const int32_t c0 = rank * p.shard_cols;  // first vocabulary column of this shard
    const int32_t vc = max(0, min(p.shard_cols, p.V - c0));
    const int n_vec = (vc + 7) / 8;
    const int n = (n_vec + CHUNK_VECS - 1) / CHUNK_VECS;  // chunks per row
    const uint16_t *shard = p.logits[lr];
    uint16_t *dshard = p.dlogits[lr];
    const bool two_pass = dshard != nullptr;
    const int tail_valid = vc - (n_vec - 1) * 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t n_mine = g < p.n_rows ? (p.n_rows - g + g_per - 1) / g_per : 0;  // rows of this CTA
    auto row_of = [&](int64_t k) { return (int64_t)g + k * g_per; };

    if (threadIdx.x == 0) {
        for (int q = 0; q < ns; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, NW);
            mbar_init(wrote + q, NW);
        }
        for (int b = 0; b < NB; ++b) {
            mbar_init(part_bar + b, NW);
            mbar_init(scal_bar + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NW) {
        // ------------------------------------------------------------ producer
        if (lane == 0 && n > 0) {
            const uint64_t pol_keep = policy_evict_last(), pol_once = policy_evict_first();
            const int64_t row_bytes = (int64_t)n_vec * 16;
            int slot = 0;
            uint32_t par = 0;
            auto load_row = [&](int64_t row, uint64_t pol) {
                const uint8_t *src = reinterpret_cast<const uint8_t *>(shard + row * p.ld);
                for (int c = 0; c < n; ++c) {
                    mbar_wait_sleep(empty + slot, par ^ 1u, 64);
                    const int64_t off = (int64_t)c * CHUNK_BYTES;
                    const uint32_t bytes = (uint32_t)(row_bytes - off < CHUNK_BYTES ? row_bytes - off : CHUNK_BYTES);
                    mbar_arrive_expect_tx(full + slot, bytes);
                    bulk_g2s(ring + (size_t)slot * CHUNK_VECS, src + off, bytes, full + slot, pol);
                    if (++slot == ns) {
                        slot = 0;
                        par ^= 1u;
                    }
                }
            };
            for (int64_t k = 0; k < n_mine; ++k) {
                load_row(row_of(k), two_pass ? pol_keep : pol_once);
                if (two_pass && k >= D) load_row(row_of(k - D), pol_once);
            }
            if (two_pass)
                for (int64_t k = (n_mine > D ? n_mine - D : (int64_t)0); k < n_mine; ++k) load_row(row_of(k), pol_once);
        }
        return;
    }

    if (warp == NW + 2) {
        // ------------------------------------------------------------ store warp
        // as in K3c (loss_stream.cu): pass 2 writes each chunk's dlogits over its re-loaded
        // logits in the slot; one thread copies the slot to the dlogits row (bulk shared ->
        // global) and frees it once read, walking the producer's load order (P1(k), then the
        // re-loads of row k - D); the partial last vector is stored by its consumer thread
        if (lane == 0 && two_pass && n > 0) {
            const uint64_t pol = policy_evict_first();
            const int64_t full_bytes = (int64_t)(tail_valid < 8 ? n_vec - 1 : n_vec) * 16;
            int slot = 0;
            uint32_t wpar = 0u;  // per slot: parity of its next pass-2 use
            auto skip_row = [&]() {
                slot += n;
                while (slot >= ns) slot -= ns;
            };
            auto store_row = [&](int64_t row) {
                for (int c = 0; c < n; ++c) {
                    const int sl = slot;
                    if (++slot == ns) slot = 0;
                    mbar_wait_sleep(wrote + sl, (wpar >> sl) & 1u, 32);
                    wpar ^= 1u << sl;
                    const int64_t off = (int64_t)c * CHUNK_BYTES;
                    const int64_t end = off + CHUNK_BYTES < full_bytes ? off + CHUNK_BYTES : full_bytes;
                    if (end > off) {
                        bulk_s2g(reinterpret_cast<uint8_t *>(dshard + row * p.ld) + off,
                                 ring + (size_t)sl * CHUNK_VECS, (uint32_t)(end - off), pol);
                        tc::bulk_commit();
                        tc::bulk_wait_read<0>();
                    }
                    mbar_arrive_count(empty + sl, NW);
                }
            };
            for (int64_t k = 0; k < n_mine; ++k) {
                skip_row();  // pass 1 of row k: freed by the consumers
                if (k >= D) store_row(row_of(k - D));
            }
            for (int64_t k = (n_mine > D ? n_mine - D : (int64_t)0); k < n_mine; ++k) store_row(row_of(k));
            tc::bulk_wait_all();
        }
        return;
    }

    if (warp == NW + 1) {
        // ------------------------------------------------------------ epilogue warp
        for (int64_t k = 0; k < n_mine; ++k) {
            const int64_t row = row_of(k);
            const int b = (int)(k % NB);
            const uint32_t ph = (uint32_t)(k / NB) & 1u;
            RowInfo ri;
            uint16_t zy_bits = 0;
            int32_t y_loc = -1;
            bool mine = false;
            if (lane == 0) {
                ri = p.rowinfo[row];
                y_loc = ri.target - c0;
                mine = ri.target >= 0 && ri.target < p.V && y_loc >= 0 && y_loc < vc;
                if (mine) zy_bits = shard[row * p.ld + y_loc];
            }
            if (n > 0) mbar_wait_sleep(part_bar + b, ph, 128);
            float cm = (n > 0 && lane < NW) ? red[b][lane].a : -INFINITY;
            double cs = (n > 0 && lane < NW) ? red[b][lane].s : 0.0;
            warp_lse2_combine(cm, cs);
            const bool own_y = __shfl_sync(0xFFFFFFFFu, mine, 0);
            const float zy = own_y ? __uint_as_float(((uint32_t)__shfl_sync(0xFFFFFFFFu, (uint32_t)zy_bits, 0)) << 16)
                                   : 0.0f;
            // ---- the exchange (tagged 64-bit words, see vp_kernel)
            if (lane < p.world) {
                const uint64_t hi = (uint64_t)p.tag << 32;
                ulonglong2 *dst = p.xbuf[lane] + ((p.half + row) * p.world + rank) * 2;
                const uint64_t sb = (uint64_t)__double_as_longlong(cs) | (own_y ? (1ull << 63) : 0ull);
                st_relaxed_sys_v2(dst, hi | __float_as_uint(cm), hi | (uint32_t)sb);
                st_relaxed_sys_v2(dst + 1, hi | (uint32_t)(sb >> 32), hi | __float_as_uint(zy));
            }
            float M = -INFINITY, zsrc = 0.0f;
            double S = 0.0;
            bool own = false;
            if (lane < p.world) {
                const ulonglong2 *src = p.xbuf[rank] + ((p.half + row) * p.world + lane) * 2;
                ulonglong2 w0, w1;
                long long spins = 0;
                for (;;) {
                    w0 = ld_relaxed_sys_v2(src);
                    w1 = ld_relaxed_sys_v2(src + 1);
                    if ((uint32_t)(w0.x >> 32) == p.tag && (uint32_t)(w0.y >> 32) == p.tag &&
                        (uint32_t)(w1.x >> 32) == p.tag && (uint32_t)(w1.y >> 32) == p.tag)
                        break;
                    __nanosleep(32);
                    if (++spins > (1ll << 27)) __trap();  // a peer never arrived: fail, don't hang
                }
                const uint64_t sb = ((w1.x & 0xFFFFFFFFull) << 32) | (w0.y & 0xFFFFFFFFull);
                M = __uint_as_float((uint32_t)w0.x);
                S = __longlong_as_double((long long)(sb & ~(1ull << 63)));
                own = (sb >> 63) != 0ull;
                zsrc = __uint_as_float((uint32_t)w1.y);
            }
            warp_lse2_combine(M, S);  // same inputs in the same lanes on every rank
            const uint32_t own_mask = __ballot_sync(0xFFFFFFFFu, own);
            const float zsh = __shfl_sync(0xFFFFFFFFu, zsrc, own_mask ? __ffs(own_mask) - 1 : 0);
            if (lane == 0) {
                const float zyv = own_mask != 0u ? zsh : __int_as_float(0x7FC00000);
                const double l2s = row_l2s(S, M);
                const float lse2 = M + (float)l2s;
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
                scal[b] = make_float4(lse2, o.s, o.gy, __int_as_float(mine ? y_loc : -1));
                mbar_arrive(scal_bar + b);
            }
            __syncwarp();
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const uint4 neg_inf = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair);
    int slot = 0;
    uint32_t par = 0;
    auto take = [&]() {
        const int sl = slot;
        mbar_wait(full + sl, par);
        if (++slot == ns) {
            slot = 0;
            par ^= 1u;
        }
        return sl;
    };
    auto release = [&](int sl) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + sl);
    };
    auto pass1 = [&](int64_t k) {
        float a = -INFINITY;
        double s = 0.0;
        for (int c = 0; c < n; ++c) {
            const int sl = take();
            const uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;
            uint4 x[U];
#pragma unroll
            for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
            if (c == n - 1) {
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int vi = c * CHUNK_VECS + j * NT + threadIdx.x;
                    if (vi >= n_vec) x[j] = neg_inf;
                    else if (vi == n_vec - 1 && tail_valid < 8) x[j] = mask_tail(x[j], tail_valid);
                }
                B::reduce_first(x, (n_vec - c * CHUNK_VECS + NT - 1) / NT, a, s);
            } else {
                B::reduce(x, a, s);
            }
            release(sl);
        }
        warp_lse2_combine(a, s);
        const int b = (int)(k % NB);
        // the epilogue warp has read red[b] for row k - NB (pass 2 of row k - NB waited for
        // it when two_pass; forward-only waits here)
        if (!two_pass && k >= NB) mbar_wait(scal_bar + b, (uint32_t)((k - NB) / NB) & 1u);
        if (lane == 0 && n > 0) {
            red[b][warp] = RowPart{a, 0.0f, s};
            mbar_arrive(part_bar + b);
        }
    };
    auto pass2 = [&](int64_t k) {
        const int64_t row = row_of(k);
        const int b = (int)(k % NB);
        mbar_wait(scal_bar + b, (uint32_t)(k / NB) & 1u);
        const float4 sc4 = scal[b];
        const float lse2 = sc4.x, sc = sc4.y, gy = sc4.z;
        const auto gref = B::grad_ref(sc, lse2);
        const int32_t y = __float_as_int(sc4.w);
        const int y_chunk = y >= 0 ? (y >> 3) / CHUNK_VECS : -1;
        uint16_t *drow = dshard + row * p.ld;
        for (int c = 0; c < n; ++c) {
            const int sl = take();
            uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;  // dlogits go over the logits here
            const int v0 = c * CHUNK_VECS + threadIdx.x;
            bool tail_here = false;
            if (c != n - 1) {
                if (sc == 0.0f) {
#pragma unroll
                    for (int j = 0; j < U; ++j) chunk[j * NT + threadIdx.x] = make_uint4(0u, 0u, 0u, 0u);
                } else {
                    uint4 x[U];
#pragma unroll
                    for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
#pragma unroll
                    for (int j = 0; j < U; ++j) chunk[j * NT + threadIdx.x] = B::grad_scaled(x[j], gref);
                }
            } else {
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int vi = v0 + j * NT;
                    if (vi >= n_vec) break;
                    const uint4 d = sc == 0.0f ? make_uint4(0u, 0u, 0u, 0u)
                                               : B::grad_scaled(chunk[j * NT + threadIdx.x], gref);
                    if (vi == n_vec - 1 && tail_valid < 8) {
                        store_tail(drow + (int64_t)vi * 8, d, tail_valid);
                        tail_here = true;
                    } else {
                        chunk[j * NT + threadIdx.x] = d;
                    }
                }
            }
            if (y_chunk == c && sc != 0.0f && ((y >> 3) - c * CHUNK_VECS) % NT == (int)threadIdx.x) {
                if (tail_here && (y >> 3) == n_vec - 1) drow[y] = f2bf(gy);
                else reinterpret_cast<uint16_t *>(chunk)[y - c * CHUNK_VECS * 8] = f2bf(gy);
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(wrote + sl);
        }
    };
    for (int64_t k = 0; k < n_mine; ++k) {
        pass1(k);
        if (two_pass && k >= D) pass2(k - D);
    }
    if (two_pass)
        for (int64_t k = (n_mine > D ? n_mine - D : (int64_t)0); k < n_mine; ++k) pass2(k);
}

template <int NT, int MINB, int CV>
static cudaError_t launch_vp_delay(VpParams p, const grpo_vp_comm_t *comm, int ns, int D, int64_t n_rows,
                                   cudaStream_t s, int *launches, grpo_plan_t *plan, char *why,
                                   size_t why_len) {
    const size_t smem = (size_t)ns * CV * 16 + 3 * (size_t)ns * 8;
    auto kern = vp_delay_kernel<NT, MINB, CV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, n_sm = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT + 96, smem);
    if (e != cudaSuccess) return e;
    // every CTA must be resident (a CTA may wait for a peer rank's CTA of the same index)
    int64_t g_per = (int64_t)n_sm * (occ < MINB ? occ : MINB) / comm->n_local;
    if (g_per > n_rows) g_per = n_rows;
    if (g_per < 1) {
        if (why) snprintf(why, why_len, "vp delay kernel: no resident CTA per local rank");
        return cudaErrorInvalidConfiguration;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)(g_per * comm->n_local));
    cfg.blockDim = dim3(NT + 96);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, p, ns, D);
    if (e != cudaSuccess) return e;
    if (plan) {
        *plan = grpo_plan_t{};
        plan->kernel = 9;
        plan->ctas_per_sm = MINB;
        plan->grid = (int32_t)(g_per * comm->n_local);
        plan->vec_per_thread = NT;
        plan->stages = ns;
        plan->max_clusters = occ;
        plan->smem_bytes = (int32_t)smem;
        plan->lag = D + 1;
    }
    *launches += 1;
    return cudaSuccess;
}

template <int NT, int MINB, int CV>
static cudaError_t launch_vp_stream(VpParams p, const grpo_vp_comm_t *comm, int ns, int pf,
                                    int64_t n_rows, cudaStream_t s, int *launches, grpo_plan_t *plan,
                                    char *why, size_t why_len) {
    const size_t smem = (size_t)ns * CV * 16 + 2 * (size_t)ns * 8;
    auto kern = vp_stream_kernel<NT, MINB, CV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, n_sm = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT + 64, smem);
    if (e != cudaSuccess) return e;
    // every CTA must be resident (a CTA may wait for a peer rank's CTA of the same index)
    int64_t g_per = (int64_t)n_sm * (occ < MINB ? occ : MINB) / comm->n_local;
    if (g_per > n_rows) g_per = n_rows;
    if (g_per < 1) {
        if (why) snprintf(why, why_len, "vp stream kernel: no resident CTA per local rank");
        return cudaErrorInvalidConfiguration;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)(g_per * comm->n_local));
    cfg.blockDim = dim3(NT + 64);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int la = 1;  // look-ahead chunks (K3c's default)
    e = cudaLaunchKernelEx(&cfg, kern, p, ns, pf, la);
    if (e != cudaSuccess) return e;
    if (plan) {
        *plan = grpo_plan_t{};
        plan->kernel = 8;
        plan->ctas_per_sm = MINB;
        plan->grid = (int32_t)(g_per * comm->n_local);
        plan->vec_per_thread = NT;
        plan->stages = ns;
        plan->max_clusters = occ;
        plan->smem_bytes = (int32_t)smem;
        plan->lag = pf;
    }
    *launches += 1;
    return cudaSuccess;
}

template <int NT, int U, int CPS>
static cudaError_t launch_vp_plan(VpParams p, const grpo_vp_comm_t *comm, int lag, int64_t n_rows,
                                  cudaStream_t s, int *launches, grpo_plan_t *plan, char *why,
                                  size_t why_len) {
    const int n_vec = (comm->shard_cols + 7) / 8;
    int cv = (int)((size_t)(160 * 1024) / CPS / ((size_t)NT * 16));
    const int nv = (n_vec + NT - 1) / NT * (lag ? 2 : 1);
    if (lag) cv &= ~1;
    if (cv > nv) cv = nv;
    p.cache_vecs = cv;
    const size_t smem = (size_t)cv * NT * 16;
    auto kern = lag ? vp_kernel<NT, U, 1> : vp_kernel<NT, U, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, n_sm = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    // every CTA must be resident (a CTA may wait for a peer rank's CTA of the same index)
    int64_t g_per = (int64_t)n_sm * (occ < CPS ? occ : CPS) / comm->n_local;
    if (g_per > n_rows) g_per = n_rows;
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
        plan->kernel = 7;
        plan->ctas_per_sm = CPS;
        plan->grid = (int32_t)(g_per * comm->n_local);
        plan->vec_per_thread = NT;
        plan->stages = cv;
        plan->max_clusters = occ;
        plan->smem_bytes = (int32_t)smem;
        plan->lag = lag;
    }
    *launches += 1;
    return cudaSuccess;
}

cudaError_t launch_vp(const LossArgs &a, const grpo_vp_comm_t *comm, unsigned long long *row_ctr,
                      cudaStream_t s, int *launches,
                      grpo_plan_t *plan, char *why, size_t why_len) {
    if (a.n_rows == 0) return cudaSuccess;
    const int lag = comm->lag ? 1 : 0;  // (lag >= 2: the ring kernel with pass 2 delayed by lag - 1 rows)
    VpParams p = {};
    p.world = comm->world;
    p.rank_begin = comm->rank_begin;
    p.n_local = comm->n_local;
    p.shard_cols = comm->shard_cols;
    for (int q = 0; q < comm->n_local; ++q) {
        p.logits[q] = comm->logits[q];
        p.dlogits[q] = comm->dlogits[q];
    }
    for (int q = 0; q < comm->world; ++q) p.xbuf[q] = static_cast<ulonglong2 *>(comm->xbuf[q]);
    p.tag = comm->epoch + 1u;
    p.row_ctr = row_ctr;
    p.dynamic = comm->dynamic_rows ? 1 : 0;
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
    if (comm->lag >= 2) {  // pass 2 delayed by lag - 1 rows (vp_delay_kernel), ring geometry by row length
        const int D = comm->lag - 1;
        if (n_vec >= 7500)  // one CTA per SM: (D + 1) rows x 148 CTAs stay in L2 for rows >= 120 KB
            return launch_vp_delay<512, 1, 2048>(p, comm, 6, D, a.n_rows, s, launches, plan, why, why_len);
        return launch_vp_delay<256, 2, 1024>(p, comm, 6, D, a.n_rows, s, launches, plan, why, why_len);
    }
    // long shards (>= 90000 columns), default schedule: the streamed ring kernel with the
    // loss_fwd auto plan's geometry for that row length (api.cu); two such rows per SM would
    // not stay in L2 for a delayed pass 2
    if (!lag && !comm->dynamic_rows && n_vec >= 11250)
        return launch_vp_stream<512, 1, 2048>(p, comm, 6, 3, a.n_rows, s, launches, plan, why, why_len);
    // shards of 16384 .. 89999 columns (R = 2, 4, 8 at V = 152064): the ring kernel with pass 2
    // delayed by one row, the row re-read from L2 -- on B200s, 65536 rows, max over ranks:
    // R = 2 x 76032 (one 512-thread CTA per SM) 3.38 ms vs 3.83 for the look-ahead ring, 1.00x
    // the single-GPU kernel on one shard; R = 4 x 38016 (two 256-thread CTAs) 1.78 ms vs 2.18
    // for the row-wise kernel, 1.04x one shard; delays of 2 / 3 rows are slower (the re-read
    // rows no longer stay in L2), and so is the two-CTA geometry on the R = 2 rows (4.60 ms:
    // 2 rows x 148 KB x 296 CTAs = 88 MB), DESIGN.md section 9.1
    if (!lag && !comm->dynamic_rows && n_vec >= 7500)
        return launch_vp_delay<512, 1, 2048>(p, comm, 6, 1, a.n_rows, s, launches, plan, why, why_len);
    if (!lag && !comm->dynamic_rows && n_vec >= 2048)
        return launch_vp_delay<256, 2, 1024>(p, comm, 6, 1, a.n_rows, s, launches, plan, why, why_len);
    // the row-wise kernel's residency rule on the shard's row length (loss_aux.cu)
    if (n_vec >= 14000) return launch_vp_plan<512, 8, 2>(p, comm, lag, a.n_rows, s, launches, plan, why, why_len);
    if (n_vec >= 6000) return launch_vp_plan<256, 8, 4>(p, comm, lag, a.n_rows, s, launches, plan, why, why_len);
    return launch_vp_plan<256, 4, 8>(p, comm, lag, a.n_rows, s, launches, plan, why, why_len);
}

}  // namespace grpo
