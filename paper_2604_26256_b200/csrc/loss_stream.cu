// loss_stream.cu -- K3c: the fused loss as one row per SM streamed through a TMA ring.
//
// K3b (loss_aux.cu) keeps the head of each row in shared memory and re-reads the rest
// from L2 in pass 2; with two 304 KB rows in flight per SM about 10 % of the re-reads
// miss L2.  K3c gives each SM one row at a time and moves it with the bulk-copy engine
// (cp.async.bulk global -> shared, completion on mbarriers) into a FIFO ring of NS
// slots, so the loads need neither registers nor L1 staging and almost the whole
// shared memory holds row data.  Four roles:
//
//   producer (one thread)   loads, per row k, the pass-1 chunks of row k, then the first
//                           LA (= 1) chunks of row k+1 (the look-ahead), then the re-loads of
//                           row k's chunks 0..n-R-1 (the part that did not stay resident)
//                           for pass 2, slot j % NS for the j-th load;
//   consumers (NT threads)  pass 1 of row k (log2-domain max / sum; the first LA chunks
//                           were consumed in the previous row's look-ahead), publish the
//                           warps' partials, pass 1 of row k+1's first LA chunks, then pass
//                           2 of row k (the R resident chunks, then the re-loads), writing
//                           each chunk's dlogits over its logits in the slot;
//   store warp (one thread) copies every pass-2 slot to the dlogits row (bulk shared ->
//                           global) and frees it once the copy has read it;
//   epilogue warp           per row: waits for the 16 warp partials, combines them (and,
//                           with SPLIT = 2, exchanges them with the partner CTA), runs the
//                           fp64 per-row epilogue (logp, ratio, clip, term, token scale)
//                           and hands (ref = lse2 - log2|s|, s, g_y = s (p_y - 1), y) to the
//                           consumers' pass 2 (the log2 once per row, not once per thread).
//
// The epilogue and the block combine thus run while the consumers stream the next row's
// first chunks: no per-row barrier among the consumers and no serial section on their
// path (the per-row reduce -> epilogue -> barrier chain took ~3 % of the step in the
// previous single-role design).  Consumption order equals load order,
// so the ring is strictly FIFO: load j waits for the release of load j - NS.  The R
// resident chunks of row k are its last ones, consumed first in its pass 2; LA <= NS - R
// and LA <= n - R keep every slot a load waits for released before the consumer needs it.
#include <cstdio>

#include "common.cuh"
#include "rowwise.cuh"
#include "tc.cuh"

namespace grpo {
namespace k3c {


struct Params {
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
    int32_t ns;  // ring slots
    int32_t pf;  // slots kept free at the end of pass 1
    int32_t la;  // look-ahead chunks of the next row before a row's pass 2
};

struct Geometry {
    int n_vec;       // 8-element vectors per row (ceil(V / 8))
    int n;           // chunks per row
    int R;           // chunks resident after pass 1 (re-consumed without a load)
    int LA;          // look-ahead chunks (first chunks of the next row before pass 2)
    int tail_valid;  // valid elements of the last vector
};

template <int CHUNK_VECS>
__device__ __forceinline__ Geometry geometry(const Params &p, int V, bool two_pass) {
    Geometry g;
    g.n_vec = (V + 7) / 8;
    g.n = (g.n_vec + CHUNK_VECS - 1) / CHUNK_VECS;
    g.R = two_pass ? min(g.n, max(0, p.ns - p.pf)) : 0;
    g.LA = two_pass ? max(0, min(p.la, min(p.ns - g.R, g.n - g.R))) : 0;
    g.tail_valid = V - (g.n_vec - 1) * 8;
    return g;
}

// SPLIT = 2: a cluster of two CTAs (two SMs) shares each row, CTA r streaming vectors
// [r*h, ...) of it (h = ceil(ceil(V/8)/2)); the epilogue warps of the two CTAs exchange
// their (max, sum) partials through distributed shared memory (st.async onto the
// partner's mbarrier, one buffer per row parity) and merge them in rank order, so both
// hold identical row scalars.  Halving the row halves the time between a chunk's pass-1
// load and its pass-2 re-load, so at V = 262144 (512 KB rows) the re-loads stay in L2;
// the pair's wait for each other sits in the epilogue warps, off the consumers' path.
// BULK: pass 2's dlogits leave through the ring slots by a store warp's bulk copies (one CTA
// per SM); otherwise every consumer thread stores its vectors (the two-CTA plan).
template <int NT, int MINB, int CHUNK_VECS, int SPLIT, bool BULK = (MINB == 1)>
__global__ void __launch_bounds__(NT + (BULK ? 96 : 64), MINB) stream_kernel(const Params p) {
    constexpr int CHUNK_BYTES = CHUNK_VECS * 16;
    constexpr int U = CHUNK_VECS / NT;  // vectors per consumer thread per chunk
    constexpr int NW = NT / 32;
    extern __shared__ __align__(128) uint8_t smem[];
    uint4 *ring = reinterpret_cast<uint4 *>(smem);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)p.ns * CHUNK_BYTES);
    uint64_t *empty = full + p.ns;
    uint64_t *wrote = empty + p.ns;  // pass-2 uses: NW warp arrivals, the slot holds dlogits
    __shared__ RowPart red[2][NW];                 // warp partials, by row parity
    __shared__ float4 scal[2];                     // (ref, s, g_y, y) for pass 2, by row parity
    __shared__ __align__(8) uint64_t part_bar[2];  // NW warp arrivals: red[b] complete
    __shared__ __align__(8) uint64_t scal_bar[2];  // 1 arrival: scal[b] written
    __shared__ RowPart xbuf[2];
    __shared__ __align__(8) uint64_t xbar[2];
    const bool two_pass = p.dlogits != nullptr;
    const uint32_t crank = SPLIT == 2 ? cluster_ctarank() : 0u;
    const int hv = ((p.V + 7) / 8 + 1) / 2;
    const int col0 = SPLIT == 2 ? (int)crank * hv * 8 : 0;              // first column of the slice
    const int Vloc = SPLIT == 2 ? (crank == 0 ? hv * 8 : p.V - hv * 8) : p.V;  // its width
    const Geometry g = geometry<CHUNK_VECS>(p, Vloc, two_pass);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.ns; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NW);
            mbar_init(wrote + s, NW);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(part_bar + b, NW);
            mbar_init(scal_bar + b, 1);
            mbar_init(xbar + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (SPLIT == 2) cluster_sync_all();  // the partner's barriers exist before any st.async
    else __syncthreads();

    const int64_t row0 = SPLIT == 2 ? (int64_t)cluster_id_x() : (int64_t)blockIdx.x;
    const int64_t rstep = SPLIT == 2 ? (int64_t)ncluster_x() : (int64_t)gridDim.x;
    if (warp == NW) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol_keep = policy_evict_last(), pol_once = policy_evict_first();
            const int64_t row_bytes = (int64_t)g.n_vec * 16;
            int slot = 0;
            uint32_t par = 0;  // parity of the slot's current use
            auto load = [&](int64_t row, int c, bool reload) {
                const uint8_t *src = reinterpret_cast<const uint8_t *>(p.logits + row * p.ld + col0);
                mbar_wait_sleep(empty + slot, par ^ 1u, 64);
                const int64_t off = (int64_t)c * CHUNK_BYTES;
                const uint32_t bytes = (uint32_t)(row_bytes - off < CHUNK_BYTES ? row_bytes - off : CHUNK_BYTES);
                // chunks read again from L2 in pass 2 stay; the rest streams through
                const uint64_t pol = (!reload && c < g.n - g.R && two_pass) ? pol_keep : pol_once;
                mbar_arrive_expect_tx(full + slot, bytes);
                bulk_g2s(ring + (size_t)slot * CHUNK_VECS, src + off, bytes, full + slot, pol);
                if (++slot == p.ns) {
                    slot = 0;
                    par ^= 1u;
                }
            };
            for (int64_t row = row0; row < p.n_rows; row += rstep) {
                for (int c = (row == row0 ? 0 : g.LA); c < g.n; ++c) load(row, c, false);
                if (row + rstep < p.n_rows)
                    for (int c = 0; c < g.LA; ++c) load(row + rstep, c, false);
                if (two_pass)
                    for (int c = 0; c < g.n - g.R; ++c) load(row, c, true);
            }
        }
        return;
    }

    if (BULK && warp == NW + 2) {
        // ------------------------------------------------------------ store warp
        // Pass 2 writes each chunk's dlogits over its logits in the ring slot; one thread here
        // copies the slot to the dlogits row with a bulk copy (shared -> global) and frees the
        // slot once the copy has read it.  It walks the producer's load order (= the
        // consumers' order) and acts on the pass-2 uses only: the resident chunks of row k and
        // its re-loads; a pass-1-only use is freed by the consumers themselves.  The partial
        // last vector of a row (V % 8 != 0) is stored by its consumer thread instead: a bulk
        // copy would write the padding columns behind V.
        if (lane == 0 && two_pass) {
            const uint64_t pol = policy_evict_first();
            const int64_t full_bytes = (int64_t)(g.tail_valid < 8 ? g.n_vec - 1 : g.n_vec) * 16;
            int slot = 0;
            uint32_t wpar = 0u;  // per slot: parity of its next pass-2 use
            auto use = [&](int64_t row, int c, bool pass2) {
                const int sl = slot;
                if (++slot == p.ns) slot = 0;
                if (!pass2) return;
                mbar_wait_sleep(wrote + sl, (wpar >> sl) & 1u, 32);
                wpar ^= 1u << sl;
                const int64_t off = (int64_t)c * CHUNK_BYTES;
                const int64_t end = off + CHUNK_BYTES < full_bytes ? off + CHUNK_BYTES : full_bytes;
                if (end > off) {
                    bulk_s2g(reinterpret_cast<uint8_t *>(p.dlogits + row * p.ld + col0) + off,
                             ring + (size_t)sl * CHUNK_VECS, (uint32_t)(end - off), pol);
                    tc::bulk_commit();
                    tc::bulk_wait_read<0>();
                }
                mbar_arrive_count(empty + sl, NW);
            };
            for (int64_t row = row0; row < p.n_rows; row += rstep) {
                for (int c = (row == row0 ? 0 : g.LA); c < g.n; ++c) use(row, c, c >= g.n - g.R);
                if (row + rstep < p.n_rows)
                    for (int c = 0; c < g.LA; ++c) use(row + rstep, c, false);
                for (int c = 0; c < g.n - g.R; ++c) use(row, c, true);
            }
            tc::bulk_wait_all();
        }
        return;
    }

    if (warp == NW + 1) {
        // ------------------------------------------------------------ epilogue warp
        uint32_t rowk = 0;
        for (int64_t row = row0; row < p.n_rows; row += rstep, ++rowk) {
            const int b = rowk & 1;
            const uint32_t ph = (rowk >> 1) & 1u;
            // the epilogue's dependent global reads, issued before the wait
            RowInfo ri;
            uint16_t zy_bits = 0;
            if (lane == 0) {
                ri = p.rowinfo[row];
                if (ri.target >= 0 && ri.target < p.V) zy_bits = p.logits[row * p.ld + ri.target];
            }
            mbar_wait_sleep(part_bar + b, ph, 256);  // a row's pass 1 takes ~7 us
            float cm = lane < NW ? red[b][lane].a : -INFINITY;
            double cs = lane < NW ? red[b][lane].s : 0.0;
            warp_lse2_combine(cm, cs);
            if (lane == 0) {
                if (SPLIT == 2) {
                    mbar_arrive_expect_tx(xbar + b, 16);
                    st_async_part(mapa_shared(smem_u32(xbuf + b), crank ^ 1u),
                                  mapa_shared(smem_u32(xbar + b), crank ^ 1u), cm, cs);
                    mbar_wait_cluster(xbar + b, ph);
                    const RowPart o = xbuf[b];
                    // rank order on both CTAs: bit-identical row scalars
                    float m0 = crank == 0 ? cm : o.a;
                    double s0 = crank == 0 ? cs : o.s;
                    lse2_merge(m0, s0, crank == 0 ? o.a : cm, crank == 0 ? o.s : cs);
                    cm = m0;
                    cs = s0;
                }
                const bool y_valid = ri.target >= 0 && ri.target < p.V;
                const float zy = y_valid ? __uint_as_float(((uint32_t)zy_bits) << 16) : __int_as_float(0x7FC00000);
                const double l2s = row_l2s(cs, cm);
                const float lse2 = cm + (float)l2s;
                const double logp_d = row_logp(zy, cm, l2s);
                const RowOut o = row_epilogue(logp_d, ri, p.eps_lo, p.eps_hi, p.grad_scale);
                const float logp = (float)logp_d;
                if (crank == 0) {
                    if (p.logp_out) p.logp_out[row] = logp;
                    if (p.lse_out) p.lse_out[row] = lse2 * kLn2;
                    if (p.scale_out) p.scale_out[row] = o.s;
                    p.term_ws[row] = o.term;
                    p.logp_ws[row] = logp;
                    p.flag_ws[row] = o.flags;
                }
                scal[b] = make_float4(RowwiseBatch<NT, U>::grad_ref(o.s, lse2).ref, o.s, o.gy,
                                      __int_as_float(y_valid ? ri.target : -1));
                mbar_arrive(scal_bar + b);
            }
            __syncwarp();
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const uint4 neg_inf = make_uint4(kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair, kBf16NegInfPair);
    int slot = 0;      // slot of the next load this CTA consumes
    uint32_t par = 0;  // and the parity of that slot's use
    // one pass-1 chunk c of a row into (a, s); `last` = the ragged last chunk
    auto pass1_chunk = [&](int c, bool last, float &a, double &s) {
        const int sl = slot;
        mbar_wait(full + sl, par);
        if (++slot == p.ns) {
            slot = 0;
            par ^= 1u;
        }
        const uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;
        uint4 x[U];
        if (!last) {
#pragma unroll
            for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
            RowwiseBatch<NT, U>::reduce(x, a, s);  // running max reference, fp64 sum (rowwise.cuh)
        } else {
            // the ragged last chunk: only its first jb = ceil(valid / NT) vector batches hold
            // row data (prod: 573 of 2048 vectors, 2 of 4 batches), so the exponentials of
            // the empty batches are not computed at all
            const int jb = (g.n_vec - c * CHUNK_VECS + NT - 1) / NT;
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int vi = c * CHUNK_VECS + j * NT + threadIdx.x;
                x[j] = j < jb ? chunk[j * NT + threadIdx.x] : neg_inf;
                if (vi >= g.n_vec) x[j] = neg_inf;
                else if (vi == g.n_vec - 1 && g.tail_valid < 8) x[j] = mask_tail(x[j], g.tail_valid);
            }
            RowwiseBatch<NT, U>::reduce_first(x, jb, a, s);
        }
        if (c < g.n - g.R) {  // not resident: release now
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + sl);
        }
    };
    float a = -INFINITY;  // the current row's partial (its first LA chunks come from the look-ahead)
    double s = 0.0;
    if (row0 < p.n_rows)
        for (int c = 0; c < g.LA; ++c) pass1_chunk(c, c == g.n - 1, a, s);
    uint32_t rowk = 0;
    for (int64_t row = row0; row < p.n_rows; row += rstep, ++rowk) {
        const int b = rowk & 1;
        // ---- pass 1 (rest): the full chunks without masking, the ragged last one after them
        int res_base = slot;  // slot of this row's chunk LA: chunks LA..n-1 are contiguous loads
#pragma unroll 1
        for (int c = g.LA; c < g.n - 1; ++c) pass1_chunk(c, false, a, s);
        if (g.n - 1 >= g.LA) pass1_chunk(g.n - 1, true, a, s);
        // ---- publish the warp's partial; before reusing red[b], the epilogue of row k-2
        // (same buffer) must have read it -- in two-pass mode pass 2 of row k-2 waited for it
        warp_lse2_combine(a, s);
        if (!two_pass && rowk >= 2) mbar_wait(scal_bar + b, ((rowk - 2) >> 1) & 1u);
        if (lane == 0) {
            red[b][warp] = RowPart{a, 0.0f, s};
            mbar_arrive(part_bar + b);
        }
        // ---- look-ahead: the next row's first chunks while the epilogue warp finishes this row
        a = -INFINITY;
        s = 0.0;
        if (row + rstep < p.n_rows)
            for (int c = 0; c < g.LA; ++c) pass1_chunk(c, c == g.n - 1, a, s);
        if (!two_pass) continue;
        // ---- pass 2: resident chunks n-R..n-1 (loads res_base + (c - LA)), then the re-loads
        mbar_wait(scal_bar + b, (rowk >> 1) & 1u);
        const float4 sc4 = scal[b];
        const float sc = sc4.y, gy = sc4.z;
        const typename RowwiseBatch<NT, U>::GradRef gref{sc4.x, sc < 0.0f ? 0x80008000u : 0u};
        const int32_t yfull = __float_as_int(sc4.w);
        const int32_t y = (yfull >= col0 && yfull < col0 + Vloc) ? yfull - col0 : -1;  // in this slice
        const int y_chunk = y >= 0 ? (y >> 3) / CHUNK_VECS : -1;
        const int res_sl = g.R > 0 ? (res_base + (g.n - g.R - g.LA)) % p.ns : 0;  // slot of chunk n-R
        uint16_t *drow = p.dlogits + row * p.ld + col0;
        for (int i = 0; i < g.n; ++i) {
            const bool resident = i < g.R;
            const int c = resident ? g.n - g.R + i : i - g.R;
            int sl;
            if (resident) {
                sl = res_sl + i;  // the pass-1 load of chunk c, still in its slot
                if (sl >= p.ns) sl -= p.ns;
            } else {
                sl = slot;
                mbar_wait(full + sl, par);
                if (++slot == p.ns) {
                    slot = 0;
                    par ^= 1u;
                }
            }
            if constexpr (BULK) {
                // the chunk's dlogits go over its logits in the slot (each thread rewrites the
                // vectors it read); the store warp copies the slot out (bulk shared -> global)
                uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;
                const int v0 = c * CHUNK_VECS + threadIdx.x;
                bool tail_here = false;  // this thread stored the row's partial last vector itself
                if (c != g.n - 1) {  // full chunk: no checks
                    if (sc == 0.0f) {
    #pragma unroll
                        for (int j = 0; j < U; ++j) chunk[j * NT + threadIdx.x] = make_uint4(0u, 0u, 0u, 0u);
                    } else {
                        uint4 x[U];
    #pragma unroll
                        for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
                        if (gref.sign == 0u) {  // s > 0: no sign flip on the packed pairs
                            const typename RowwiseBatch<NT, U>::GradRef gp{gref.ref, 0u};
    #pragma unroll
                            for (int j = 0; j < U; ++j)
                                chunk[j * NT + threadIdx.x] = RowwiseBatch<NT, U>::grad_scaled(x[j], gp);
                        } else {
    #pragma unroll
                            for (int j = 0; j < U; ++j)
                                chunk[j * NT + threadIdx.x] = RowwiseBatch<NT, U>::grad_scaled(x[j], gref);
                        }
                    }
                } else {
    #pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const int vi = v0 + j * NT;
                        if (vi >= g.n_vec) break;
                        const uint4 d = sc == 0.0f ? make_uint4(0u, 0u, 0u, 0u)
                                                   : RowwiseBatch<NT, U>::grad_scaled(chunk[j * NT + threadIdx.x], gref);
                        if (vi == g.n_vec - 1 && g.tail_valid < 8) {
                            store_tail(drow + (int64_t)vi * 8, d, g.tail_valid);
                            tail_here = true;
                        } else {
                            chunk[j * NT + threadIdx.x] = d;
                        }
                    }
                }
                // the target's own column (g_y from the fp64 epilogue), rewritten by the thread that
                // wrote its vector: in the slot, or in global memory behind the partial last vector
                if (y_chunk == c && sc != 0.0f && ((y >> 3) - c * CHUNK_VECS) % NT == (int)threadIdx.x) {
                    if (tail_here && (y >> 3) == g.n_vec - 1) drow[y] = f2bf(gy);
                    else reinterpret_cast<uint16_t *>(chunk)[y - c * CHUNK_VECS * 8] = f2bf(gy);
                }
                tc::fence_proxy_async_smem();  // the generic-proxy writes, visible to the bulk copy
                __syncwarp();
                if (lane == 0) mbar_arrive(wrote + sl);
            } else {
                // direct stores (the two-CTA plan: its 16 KB slots and 2 x 352 threads lost 3 % at
                // V = 50688 with the store warp, t67)
                const uint4 *chunk = ring + (size_t)sl * CHUNK_VECS;
                uint4 *dst4 = reinterpret_cast<uint4 *>(drow);
                const int v0 = c * CHUNK_VECS + threadIdx.x;
                if (c != g.n - 1) {
                    if (sc == 0.0f) {
    #pragma unroll
                        for (int j = 0; j < U; ++j) stg_stream(dst4 + v0 + j * NT, make_uint4(0u, 0u, 0u, 0u));
                    } else {
                        uint4 x[U];
    #pragma unroll
                        for (int j = 0; j < U; ++j) x[j] = chunk[j * NT + threadIdx.x];
                        if (gref.sign == 0u) {
                            const typename RowwiseBatch<NT, U>::GradRef gp{gref.ref, 0u};
    #pragma unroll
                            for (int j = 0; j < U; ++j)
                                stg_stream(dst4 + v0 + j * NT, RowwiseBatch<NT, U>::grad_scaled(x[j], gp));
                        } else {
    #pragma unroll
                            for (int j = 0; j < U; ++j)
                                stg_stream(dst4 + v0 + j * NT, RowwiseBatch<NT, U>::grad_scaled(x[j], gref));
                        }
                    }
                } else {
    #pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const int vi = v0 + j * NT;
                        if (vi >= g.n_vec) break;
                        const uint4 d = sc == 0.0f ? make_uint4(0u, 0u, 0u, 0u)
                                                   : RowwiseBatch<NT, U>::grad_scaled(chunk[j * NT + threadIdx.x], gref);
                        if (vi == g.n_vec - 1 && g.tail_valid < 8) store_tail(drow + (int64_t)vi * 8, d, g.tail_valid);
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
}

}  // namespace k3c

cudaError_t launch_fused_stream(const LossArgs &a, const grpo_tune_t *tune, cudaStream_t s, int *launches,
                                grpo_plan_t *plan, char *why, size_t why_len) {
    using namespace k3c;
    if (a.n_rows == 0) return cudaSuccess;
    Params p{};
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
    p.ns = (tune && tune->stages > 0) ? tune->stages : 0;
    p.pf = (tune && tune->lag > 0) ? tune->lag : 3;
    // look-ahead chunks of the next row before a row's pass 2 (tune->prefetch; 0 = 1, -1 = none).
    // A look-ahead chunk is loaded a whole row before its pass-2 re-load, so each one costs
    // L2 hits: DRAM reads 1.008x / 1.04x / 1.13x the logits for 0 / 1 / 2 chunks (ncu, 131072
    // rows of prod), launch 12.86 / 12.72 / 12.92 ms: one chunk hides the epilogue warp's work
    p.la = (tune && tune->prefetch != 0) ? (tune->prefetch < 0 ? 0 : tune->prefetch) : 1;
    // consumer threads (ctas_per_sm 256 / 512), CTAs per SM (row_cache 1 / 2), slot size
    const int nt = (tune && tune->ctas_per_sm == 256) ? 256 : 512;
    const int cps = (tune && tune->row_cache == 2) ? 2 : 1;
    const int ckb = (tune && (tune->chunk_kb == 24 || tune->chunk_kb == 32 || tune->chunk_kb == 48 ||
                              tune->chunk_kb == 64)) ? tune->chunk_kb : 16;
    // cluster_size 2: two SMs per row (SPLIT = 2; one 512-thread CTA per SM, 16 or 32 KB slots)
    const int split = (tune && tune->cluster_size == 2) ? 2 : 1;
    if (split == 2 && (cps != 1 || nt != 512 || (ckb != 16 && ckb != 32) || a.V < 16384)) {
        if (why) snprintf(why, why_len, "stream kernel: cluster_size 2 needs 512 threads, 1 CTA per SM, "
                          "16 or 32 KB slots and V >= 16384");
        return cudaErrorInvalidValue;
    }
    const int max_ns = (cps == 2 ? 96 : 224) / ckb;  // 7 x 32 KB + barriers + static < 227 KB
    if (!(tune && tune->stages > 0)) p.ns = (cps == 2 ? 96 : 208) / ckb;
    if (p.ns < 2 || p.ns > max_ns || p.pf >= p.ns) {
        if (why) snprintf(why, why_len, "stream kernel: stages %d (2..%d), lag %d (< stages)", p.ns,
                          max_ns, p.pf);
        return cudaErrorInvalidValue;
    }
    const size_t smem = (size_t)p.ns * ckb * 1024 + 3 * (size_t)p.ns * 8;  // ring + full / empty / wrote
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    int grid = (int)std::min<int64_t>(a.n_rows, (int64_t)n_sm * cps);
    cudaError_t e;
    if (split == 2) {
        // one cluster per row in flight: as many clusters as can be co-resident (an SM pair
        // must sit in one GPC, so this can be below n_sm / 2)
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(512 + 96);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        auto kfn = ckb == 32 ? stream_kernel<512, 1, 2048, 2> : stream_kernel<512, 1, 1024, 2>;
        e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int max_clusters = 0;
        cfg.gridDim = dim3(n_sm);
        e = cudaOccupancyMaxActiveClusters(&max_clusters, kfn, &cfg);
        if (e != cudaSuccess) return e;
        if (max_clusters < 1) max_clusters = 1;
        grid = 2 * (int)std::min<int64_t>(a.n_rows, (int64_t)max_clusters);
        cfg.gridDim = dim3(grid);
        e = cudaLaunchKernelEx(&cfg, kfn, p);
        if (e != cudaSuccess) return e;
    } else {
#define GRPO_K3C(NT_, MB_, CV_)                                                                         \
    do {                                                                                               \
        e = cudaFuncSetAttribute(stream_kernel<NT_, MB_, CV_, 1>,                                         \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
        if (e != cudaSuccess) return e;                                                                \
        stream_kernel<NT_, MB_, CV_, 1><<<grid, NT_ + (MB_ == 1 ? 96 : 64), smem, s>>>(p);                                  \
    } while (0)
    if (ckb == 64) {
        GRPO_K3C(512, 1, 4096);
    } else if (ckb == 48) {
        GRPO_K3C(512, 1, 3072);
    } else if (ckb == 24) {
        GRPO_K3C(512, 1, 1536);
    } else if (ckb == 32) {
        if (nt == 512 && cps == 1) GRPO_K3C(512, 1, 2048);
        else if (nt == 512) GRPO_K3C(512, 2, 2048);
        else if (cps == 1) GRPO_K3C(256, 1, 2048);
        else GRPO_K3C(256, 2, 2048);
    } else {
        if (nt == 512 && cps == 1) GRPO_K3C(512, 1, 1024);
        else if (nt == 512) GRPO_K3C(512, 2, 1024);
        else if (cps == 1) GRPO_K3C(256, 1, 1024);
        else GRPO_K3C(256, 2, 1024);
    }
#undef GRPO_K3C
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *launches += 1;
    if (plan) {
        *plan = grpo_plan_t{};
        plan->kernel = 3;
        plan->ctas_per_sm = cps;
        plan->cluster_size = split;
        plan->stages = p.ns;
        plan->lag = p.pf;
        plan->vec_per_thread = nt;
        plan->grid = grid;
        plan->smem_bytes = (int32_t)smem;
    }
    return cudaSuccess;
}

}  // namespace grpo
