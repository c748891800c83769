// lmhead.cu -- SURVEY NEXT(2): the loss fused with the LM head that produces the
// logits.  z = X W^T (X: hidden states [n, d], W: LM-head weight [V, d], both bf16)
// runs on the 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM,
// operands staged by TMA in 128-byte-swizzled shared memory) and the epilogue
// consumes each 128 x 256 accumulator tile straight out of TMEM:
//
//   EPI_STATS  per-row log2-domain softmax partials (max, sum 2^(t - max)) and z_y
//              -> lmhead_combine_kernel -> log pi_theta(y_t) and the
//              per-token epilogue of eq:grpo_async -- the logits never reach HBM;
//   EPI_DZ     the logits gradient dJ/dz = s_t (softmax(z) - onehot(y_t)) of the same
//              tile (recomputed in the backward, as Cut-Cross-Entropy does) -> bf16;
//   EPI_LOGITS the bf16 logits themselves (the unfused producer; also the GEMM check).
//
// One CTA per SM, persistent, warp-specialised: warp 0 issues TMA, warp 1 issues
// tcgen05.mma (one thread) into one of two 256-column TMEM accumulators, warps 2-5
// drain the other accumulator (each thread owns one row = one TMEM lane).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sched.cuh"
#include "tc.cuh"

namespace grpo {
namespace lm {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
__device__ int32_t g_units[sched::N_COUNTERS];  // unit counters of the launches (sched.cuh)
constexpr int A_BYTES = BM * BK * 2;
constexpr int NUM_THREADS = 192;
constexpr uint32_t TMEM_COLS = 2 * BN;

enum { EPI_STATS = 0, EPI_DZ = 1, EPI_LOGITS = 2 };

struct Params {
    int32_t n_rows, V, d;
    int32_t m_tiles, n_vt, vt_per_unit, n_units, group_m;
    int32_t col_offset;  // first vocabulary id of this W shard (tensor-parallel head), else 0
    int32_t pol_x, pol_w;  // L2 policies of the X / W loads: 0 normal, 1 evict_first, 2 evict_last
    int32_t *counter;      // the launch's unit counter, 0 at launch (sched.cuh)
    // EPI_STATS
    const RowInfo *rowinfo;
    RowPart *part;  // [n_split][n_rows] log2-domain (max, sum fp64)
    float *zy;     // [n_rows]
    // EPI_DZ / EPI_LOGITS
    uint16_t *out;  // [n_rows][ld_out] bf16
    int64_t ld_out;
    const int64_t *targets;
    const float *lse;    // natural-log lse per row (from the forward)
    const float *scale;  // s_t per row
    float mult;          // extra factor on s_t (EPI_DZ)
};

// Units are rastered in groups of GROUP_M row tiles: the CTAs running at the same
// time cover ~GROUP_M row tiles x ~grid/GROUP_M vocabulary tiles, so the X and W tiles
// they stream (re-read once per tile of the other operand) stay resident in L2.
__device__ __forceinline__ void decode(const Params &p, int unit, int &m_tile, int &split) {
    const int GROUP_M = p.group_m;
    const int n_split = (p.n_vt + p.vt_per_unit - 1) / p.vt_per_unit;
    const int per_group = GROUP_M * n_split;
    const int grp = unit / per_group;
    const int rem = unit - grp * per_group;
    const int gm = min(GROUP_M, p.m_tiles - grp * GROUP_M);  // row tiles in this group
    split = rem / gm;
    m_tile = grp * GROUP_M + (rem - split * gm);
}

// CG = CTAs per MMA: 1 (one SM, M = 128 per tile) or 2 (a CTA pair on one TPC issuing
// tcgen05.mma.cta_group::2, M = 256: each CTA stages its own 128 rows of X and half of the
// 256 vocabulary rows of W, so a pair moves 2 x 32 KB per k-block instead of 2 x 48 KB).
template <int CG>
struct Geo {
    static constexpr int B_ROWS = BN / CG;                 // W rows staged per CTA
    static constexpr int B_BYTES_CG = B_ROWS * BK * 2;
    static constexpr int STAGE = A_BYTES + B_BYTES_CG;
    static constexpr int NSTAGE = CG == 1 ? STAGES : 6;
    static constexpr int SMEM = NSTAGE * STAGE + 1024 + 256;
    // + the store epilogues' staging (EPI_DZ / EPI_LOGITS): 4 warps x 2 boxes of 32 x 128 B
    static constexpr int STAGING = 4 * 2 * 4096;
    static constexpr int SMEM_STORE = SMEM + STAGING;
};

template <int EPI, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    lmhead_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                  const __grid_constant__ CUtensorMap tmO, const Params p) {
    using GG = Geo<CG>;
    constexpr int NS = GG::NSTAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem;                             // NS x A_BYTES
    uint8_t *sB = smem + NS * A_BYTES;              // NS x B_BYTES_CG
    // the store epilogues' staging boxes sit between the stages and the barriers
    uint8_t *staging = smem + NS * GG::STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NS * GG::STAGE + (EPI == EPI_STATS ? 0 : GG::STAGING));
    uint64_t *full = bars, *empty = bars + NS, *tfull = bars + 2 * NS, *tempty = bars + 2 * NS + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NS + 4);
    sched::Queue *uq = reinterpret_cast<sched::Queue *>(bars + 2 * NS + 6);  // dynamic units (sched.cuh)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = p.d / BK;
    const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;        // 0 = the pair's leader

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 128 * CG);  // every epilogue thread of the pair
        }
        sched::init<CG>(uq);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tc::prefetch_tmap(&tmX);
        tc::prefetch_tmap(&tmW);
        if (EPI != EPI_STATS) tc::prefetch_tmap(&tmO);
    }
    if (warp == 1) {
        if (CG == 2) tc::tmem_alloc2(tmem_slot, TMEM_COLS);
        else tc::tmem_alloc(tmem_slot, TMEM_COLS);
    }
    tc::fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();  // the peer's barriers are initialised before use
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            auto mkpol = [](int c) {
                return c == 1 ? policy_evict_first() : c == 2 ? policy_evict_last() : policy_evict_normal();
            };
            const uint64_t pol_a = mkpol(p.pol_x), pol_b = mkpol(p.pol_w);
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0;; ++i) {
                const int unit = crank == 0 ? sched::fetch<CG>(uq, i, p.counter, p.n_units)
                                            : sched::next<CG>(uq, i, crank);
                if (unit < 0) break;
                int m_tile, split;
                decode(p, unit, m_tile, split);
                const int vt0 = split * p.vt_per_unit, vt1 = min(vt0 + p.vt_per_unit, p.n_vt);
                const int a_row = m_tile * (BM * CG) + (int)crank * BM;
                for (int vt = vt0; vt < vt1; ++vt)
                    for (int kb = 0; kb < nk; ++kb) {
                        mbar_wait(empty + stage, phase ^ 1u);
                        const int b_row = vt * BN + (int)crank * GG::B_ROWS;
                        if (CG == 1) {
                            mbar_arrive_expect_tx(full + stage, GG::STAGE);
                            tc::tma_load_2d(sA + stage * A_BYTES, &tmX, kb * BK, a_row, full + stage, pol_a);
                            tc::tma_load_2d(sB + stage * GG::B_BYTES_CG, &tmW, kb * BK, b_row, full + stage, pol_b);
                        } else {
                            // the leader's full barrier counts both CTAs' bytes
                            if (crank == 0) mbar_arrive_expect_tx(full + stage, 2 * GG::STAGE);
                            tc::tma_load_2d_pair(sA + stage * A_BYTES, &tmX, kb * BK, a_row, full + stage, pol_a);
                            tc::tma_load_2d_pair(sB + stage * GG::B_BYTES_CG, &tmW, kb * BK, b_row, full + stage,
                                                 pol_b);
                        }
                        if (++stage == NS) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0 && crank == 0) {  // one thread of the pair's leader issues every MMA
            constexpr uint32_t idesc = tc::idesc_bf16_f32(BM * CG, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int i = 0;; ++i) {
                const int unit = sched::next<CG>(uq, i, 0u);
                if (unit < 0) break;
                int m_tile, split;
                decode(p, unit, m_tile, split);
                const int vt0 = split * p.vt_per_unit, vt1 = min(vt0 + p.vt_per_unit, p.n_vt);
                for (int vt = vt0; vt < vt1; ++vt) {
                    mbar_wait(tempty + acc, acc_phase ^ 1u);
                    tc::fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
                    for (int kb = 0; kb < nk; ++kb) {
                        mbar_wait(full + stage, phase);
                        tc::fence_after();
                        const uint64_t ad = tc::desc_k_sw128(sA + stage * A_BYTES);
                        const uint64_t bd = tc::desc_k_sw128(sB + stage * GG::B_BYTES_CG);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {  // +32 B along K inside the swizzle atom
                            if (CG == 1) tc::mma_bf16(d_tmem, ad + 2u * k, bd + 2u * k, idesc, (kb | k) != 0);
                            else tc::mma2_bf16(d_tmem, ad + 2u * k, bd + 2u * k, idesc, (kb | k) != 0);
                        }
                        if (CG == 1) tc::commit(empty + stage);
                        else tc::commit2_multicast(empty + stage, 0x3);  // frees the stage in both CTAs
                        if (++stage == NS) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    if (CG == 1) tc::commit(tfull + acc);
                    else tc::commit2_multicast(tfull + acc, 0x3);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1u;
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 2-5)
        const int q = warp & 3;                 // TMEM lane quarter this warp may access
        const int r_in_tile = q * 32 + lane;
        uint8_t *wbuf = staging + q * 8192;     // store epilogues: this warp's two boxes
        int n_boxes = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            int unit = 0;
            if (lane == 0) unit = sched::next<CG>(uq, i, crank);
            unit = __shfl_sync(0xffffffffu, unit, 0);
            if (unit < 0) break;
            int m_tile, split;
            decode(p, unit, m_tile, split);
            const int vt0 = split * p.vt_per_unit, vt1 = min(vt0 + p.vt_per_unit, p.n_vt);
            const int row = m_tile * (BM * CG) + (int)crank * BM + r_in_tile;
            const bool valid = row < p.n_rows;
            int32_t y = -1;
            float lse2 = 0.0f, sc = 0.0f;
            if (EPI == EPI_STATS) {
                // the target's column in this W shard (-1: another shard holds it)
                const int64_t t = !valid ? -1 : (p.rowinfo ? (int64_t)p.rowinfo[row].target : p.targets[row]);
                y = (t >= p.col_offset && t - p.col_offset < p.V) ? (int32_t)(t - p.col_offset) : -1;
            } else if (EPI == EPI_DZ && valid) {
                const int64_t t = p.targets[row];
                y = (t >= p.col_offset && t - p.col_offset < p.V) ? (int32_t)(t - p.col_offset) : -1;
                lse2 = p.lse[row] * kLog2e;
                sc = p.scale[row] * p.mult;
            }
            float M = -INFINITY, zy = 0.0f;
            double S = 0.0;
            bool have_y = false;
            for (int vt = vt0; vt < vt1; ++vt) {
                mbar_wait(tfull + acc, acc_phase);
                tc::fence_after();
                const int v0 = vt * BN;
                const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
                if (EPI == EPI_STATS) {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tc::tmem_ld32(t_row + (uint32_t)(c * 32), r);
                    tc::tmem_wait_ld();
                    const int cb = v0 + c * 32;          // first vocabulary column of the chunk
                    const int nvalid = min(32, p.V - cb);  // > 0 except in a ragged last tile
                    {
                        // exponents z*log2(e) - M with the exact log2 e (two FMAs, common.cuh
                        // kLog2eHi/Lo), the chunk's 32 terms summed in fp32, the row's sum in fp64
                        float zt[32];
                        float zm = -INFINITY;
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            zt[j] = j < nvalid ? __uint_as_float(r[j]) : -INFINITY;
                            zm = fmaxf(zm, zt[j]);
                        }
                        const float cm = log2_ref(zm);
                        if (cm > M) {
                            S = (M == -INFINITY) ? 0.0 : scale_pow2(S, M - cm);
                            M = cm;
                        }
                        if (M != -INFINITY) {
                            float cs = 0.0f;
#pragma unroll
                            for (int j = 0; j < 32; ++j) cs += ex2(fmaf(zt[j], kLog2eLo, fmaf(zt[j], kLog2eHi, -M)));
                            S += (double)cs;
                        }
                        if (y >= cb && y < cb + 32) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (cb + j == y) zy = __uint_as_float(r[j]);
                            have_y = true;
                        }
                    }
                }
                } else {
                    // 64 columns per box: 32 rows x 128 B staged with the 128-byte swizzle, then a TMA
                    // tile store (rows >= n_rows and columns >= V clipped by the tensor map, so the
                    // padding columns of dz stay untouched) -- coalesced 128-byte rows
#pragma unroll 1
                    for (int c = 0; c < BN / 32; c += 2) {
                        const int cb = v0 + c * 32;
                        if (cb >= p.V) break;  // warp-uniform: the rest of a ragged last tile
                        uint32_t r[32], r2[32];
                        tc::tmem_ld32(t_row + (uint32_t)(c * 32), r);
                        tc::tmem_ld32(t_row + (uint32_t)(c * 32 + 32), r2);
                        tc::tmem_wait_ld();
                        // a box that straddles V (the ragged last tile) is stored element by
                        // element: a TMA store clips at 16-byte granularity and would write the
                        // padding columns [V, ld) that share the last 16 bytes
                        const bool ragged = cb + 64 > p.V;
                        uint8_t *box = wbuf + (n_boxes & 1) * 4096;
                        if (!ragged && n_boxes >= 2) {  // the store of two boxes ago has read it
                            if (lane == 0) tc::bulk_wait_read<1>();
                            __syncwarp();
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const uint32_t *src = j < 4 ? r : r2;
                            uint32_t w[4];
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                const int o = (j & 3) * 8 + 2 * h;  // column cb + 8j + 2h within the box
                                float g0 = __uint_as_float(src[o]), g1 = __uint_as_float(src[o + 1]);
                                if (EPI == EPI_DZ) {  // s (p - onehot); exact zeros when s == 0
                                    const int col = cb + 8 * j + 2 * h;
                                    const float p0 = ex2(fmaf(g0, kLog2e, -lse2));
                                    const float p1 = ex2(fmaf(g1, kLog2e, -lse2));
                                    g0 = sc == 0.0f ? 0.0f : sc * (p0 - (col == y ? 1.0f : 0.0f));
                                    g1 = sc == 0.0f ? 0.0f : sc * (p1 - (col + 1 == y ? 1.0f : 0.0f));
                                }
                                w[h] = pack_bf16x2(g0, g1);
                            }
                            if (ragged) {
                                if (valid) {
                                    uint16_t *dst = p.out + (int64_t)row * p.ld_out + cb + 8 * j;
#pragma unroll
                                    for (int e = 0; e < 8; ++e)
                                        if (cb + 8 * j + e < p.V)
                                            dst[e] = (uint16_t)(e & 1 ? (w[e >> 1] >> 16) : (w[e >> 1] & 0xFFFFu));
                                }
                                continue;
                            }
                            *reinterpret_cast<uint4 *>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                                make_uint4(w[0], w[1], w[2], w[3]);
                        }
                        if (ragged) continue;
                        tc::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tc::tma_store_2d(&tmO, box, cb, m_tile * (BM * CG) + (int)crank * BM + q * 32);
                            tc::bulk_commit();
                        }
                        ++n_boxes;
                    }
                }
                tc::fence_before();
                if (CG == 1) mbar_arrive(tempty + acc);
                else tc::mbar_arrive_remote(tempty + acc, 0);  // the leader's MMA waits on it
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1u;
            }
            if (EPI == EPI_STATS && valid) {
                p.part[(int64_t)split * p.n_rows + row] = RowPart{M, 0.0f, S};
                if (have_y) p.zy[row] = zy;
            }
        }
        if (EPI != EPI_STATS && lane == 0) tc::bulk_wait_all();  // stores done before smem goes away
    }
    tc::fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();  // the peer's epilogue is done with the pair's TMEM
    if (warp == 1) {
        if (CG == 2) tc::tmem_dealloc2(tmem_base, TMEM_COLS);
        else tc::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// per row: merge the n_split partials in split order (deterministic), then the
// per-token epilogue shared with the logits kernels
__global__ void __launch_bounds__(256) lmhead_combine_kernel(const RowPart *__restrict__ part,
                                                             const float *__restrict__ zy_ws,
                                                             int32_t n_split, LossArgs a) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= a.n_rows) return;
    float M = -INFINITY;
    double S = 0.0;
    for (int s = 0; s < n_split; ++s) {
        const RowPart v = part[(int64_t)s * a.n_rows + row];
        lse2_merge(M, S, v.a, v.s);
    }
    const RowInfo ri = a.rowinfo[row];
    const bool y_valid = ri.target >= 0 && ri.target < a.V;
    const float zyv = y_valid ? zy_ws[row] : __int_as_float(0x7FC00000);
    const double l2s = log2(S);
    const double logp_d = row_logp(zyv, M, l2s);
    const RowOut o = row_epilogue(logp_d, ri, a.eps_lo, a.eps_hi, a.grad_scale);
    const float logp = (float)logp_d;
    if (a.logp_out) a.logp_out[row] = logp;
    if (a.lse_out) a.lse_out[row] = (float)(((double)M + l2s) * 0.69314718055994530942);
    if (a.scale_out) a.scale_out[row] = o.s;
    a.term_ws[row] = o.term;
    a.logp_ws[row] = logp;
    a.flag_ws[row] = o.flags;
}

// tensor-parallel head: this shard's per-row partial (log2-domain max, sum, z_y, holds-y)
// from its n_split unit partials, merged in unit order
__global__ void __launch_bounds__(256) lmhead_rowpart_kernel(const RowPart *__restrict__ part,
                                                             const float *__restrict__ zy_ws,
                                                             int32_t n_split, int64_t n_rows,
                                                             const int64_t *__restrict__ targets,
                                                             int32_t col_offset, int32_t Vs,
                                                             float4 *__restrict__ out) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= n_rows) return;
    float M = -INFINITY;
    double S = 0.0;
    for (int s = 0; s < n_split; ++s) {
        const RowPart v = part[(int64_t)s * n_rows + row];
        lse2_merge(M, S, v.a, v.s);
    }
    const int64_t t = targets[row];
    const bool mine = t >= col_offset && t - col_offset < Vs;
    out[row] = pack_shard_part(M, S, mine ? zy_ws[row] : 0.0f, mine);
}

// the R shards' partials of each row merged in rank order (identical on every rank), then
// the per-token epilogue of the logits kernels
__global__ void __launch_bounds__(256) lmhead_tp_combine_kernel(const float4 *__restrict__ parts,
                                                                int32_t R, LossArgs a) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (row >= a.n_rows) return;
    float M = -INFINITY, zy = __int_as_float(0x7FC00000);
    double S = 0.0;
    for (int q = 0; q < R; ++q) {
        float qa, qz;
        double qs;
        bool holds;
        unpack_shard_part(parts[(int64_t)q * a.n_rows + row], qa, qs, qz, holds);
        lse2_merge(M, S, qa, qs);
        if (holds) zy = qz;
    }
    const RowInfo ri = a.rowinfo[row];
    const bool y_valid = ri.target >= 0 && ri.target < a.V;
    const float zyv = y_valid ? zy : __int_as_float(0x7FC00000);
    const double l2s = log2(S);
    const double logp_d = row_logp(zyv, M, l2s);
    const RowOut o = row_epilogue(logp_d, ri, a.eps_lo, a.eps_hi, a.grad_scale);
    const float logp = (float)logp_d;
    if (a.logp_out) a.logp_out[row] = logp;
    if (a.lse_out) a.lse_out[row] = (float)(((double)M + l2s) * 0.69314718055994530942);
    if (a.scale_out) a.scale_out[row] = o.s;
    a.term_ws[row] = o.term;
    a.logp_ws[row] = logp;
    a.flag_ws[row] = o.flags;
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// the store epilogues' output: bf16 [rows, cols] with leading dimension ld, box 32 rows x 64
// columns (128 B) with the 128-byte swizzle of the staging boxes
static bool make_out_map(CUtensorMap *m, void *base, int64_t rows, int64_t cols, int64_t ld) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64u, 32u};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// [rows, d] bf16 row-major, box [box_rows, 64] with the 128-byte swizzle
static bool make_map(CUtensorMap *m, const void *base, int64_t rows, int32_t d, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace lm

// vocabulary tiles per work unit: units = m_tiles x ceil(n_vt / vt_per_unit)
int32_t lmhead_vt_per_unit(int64_t n_rows) {
    const int64_t m_tiles = (n_rows + lm::BM - 1) / lm::BM;
    return (int32_t)std::max<int64_t>(1, std::min<int64_t>(8, (m_tiles + 1) / 2));
}
int32_t lmhead_n_split(int64_t n_rows, int32_t V) {
    const int32_t n_vt = (V + lm::BN - 1) / lm::BN;
    const int32_t vpu = lmhead_vt_per_unit(n_rows);
    return (n_vt + vpu - 1) / vpu;
}

cudaError_t launch_lmhead(int epi, const void *X, const void *W, int64_t n_rows, int32_t d, int32_t V,
                          const RowInfo *rowinfo, RowPart *part, float *zy, uint16_t *out, int64_t ld_out,
                          const int64_t *targets, const float *lse, const float *scale, float mult,
                          cudaStream_t s, int *launches, grpo_plan_t *plan, char *why, size_t why_len,
                          int cta_group, int32_t col_offset) {
    using namespace lm;
    if (n_rows == 0) return cudaSuccess;
    const int CG = cta_group == 1 ? 1 : 2;
    CUtensorMap mx, mw, mo;
    if (!make_map(&mx, X, n_rows, d, BM) || !make_map(&mw, W, V, d, BN / CG) ||
        (epi != EPI_STATS && !make_out_map(&mo, out, n_rows, V, ld_out))) {
        if (why) snprintf(why, why_len, "cuTensorMapEncodeTiled failed (alignment / driver entry point)");
        return cudaErrorInvalidValue;
    }
    Params p{};
    p.n_rows = (int32_t)n_rows;
    p.V = V;
    p.d = d;
    p.m_tiles = (int32_t)((n_rows + BM * CG - 1) / (BM * CG));
    p.n_vt = (V + BN - 1) / BN;
    p.vt_per_unit = lmhead_vt_per_unit(n_rows);
    const int32_t n_split = (p.n_vt + p.vt_per_unit - 1) / p.vt_per_unit;
    p.n_units = p.m_tiles * n_split;
    // 32 x 128 rows of X per raster group (42 MB at d = 5120), X kept in L2 (evict_last), W
    // streamed (evict_first): at 8190 x 5120 x 152064 DRAM reads 14.6 GB vs 17.2 GB for 16 x 128
    // rows with W evict_normal, the launch -3.5 % in the back-to-back loop; 2 and 4 pair tiles
    // per group, or all 32, are worse (profiles/r02_lmhead_raster.txt)
    p.group_m = 32 / CG;
    p.pol_x = 2;
    p.pol_w = 1;
    p.rowinfo = rowinfo;
    p.part = part;
    p.zy = zy;
    p.out = out;
    p.ld_out = ld_out;
    p.targets = targets;
    p.lse = lse;
    p.scale = scale;
    p.mult = mult;
    p.col_offset = col_offset;
    {
        int32_t *base = nullptr;
        cudaError_t ec = cudaGetSymbolAddress(reinterpret_cast<void **>(&base), g_units);
        if (ec == cudaSuccess) ec = sched::take_counter(base, s, &p.counter);
        if (ec != cudaSuccess) return ec;
    }
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int groups = std::min(p.n_units, n_sm / CG);  // persistent: one CTA (pair) per SM (pair)
    cudaError_t e;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(groups * CG));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define GRPO_LM_LAUNCH(E, CG_)                                                                         \
    do {                                                                                               \
        cfg.dynamicSmemBytes = E == EPI_STATS ? Geo<CG_>::SMEM : Geo<CG_>::SMEM_STORE;                \
        e = cudaFuncSetAttribute(lmhead_kernel<E, CG_>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                 (int)cfg.dynamicSmemBytes);                                           \
        if (e != cudaSuccess) return e;                                                                \
        e = cudaLaunchKernelEx(&cfg, lmhead_kernel<E, CG_>, mx, mw, epi == EPI_STATS ? mx : mo, p);   \
    } while (0)
    if (CG == 1) {
        if (epi == EPI_STATS) GRPO_LM_LAUNCH(EPI_STATS, 1);
        else if (epi == EPI_DZ) GRPO_LM_LAUNCH(EPI_DZ, 1);
        else GRPO_LM_LAUNCH(EPI_LOGITS, 1);
    } else {
        if (epi == EPI_STATS) GRPO_LM_LAUNCH(EPI_STATS, 2);
        else if (epi == EPI_DZ) GRPO_LM_LAUNCH(EPI_DZ, 2);
        else GRPO_LM_LAUNCH(EPI_LOGITS, 2);
    }
#undef GRPO_LM_LAUNCH
    if (e != cudaSuccess) return e;
    *launches += 1;
    if (plan) {
        *plan = grpo_plan_t{};
        plan->kernel = 4 + epi;
        plan->cluster_size = CG;
        plan->grid = groups * CG;
        plan->ctas_per_sm = 1;
        plan->stages = CG == 1 ? Geo<1>::NSTAGE : Geo<2>::NSTAGE;
        plan->vec_per_thread = p.vt_per_unit;
        plan->max_clusters = p.n_units;
        plan->smem_bytes = CG == 1 ? Geo<1>::SMEM : Geo<2>::SMEM;
    }
    return cudaSuccess;
}

cudaError_t launch_lmhead_rowpart(const RowPart *part, const float *zy, int32_t n_split, int64_t n_rows,
                                  const int64_t *targets, int32_t col_offset, int32_t Vs, float4 *out,
                                  cudaStream_t s, int *launches) {
    if (n_rows == 0) return cudaSuccess;
    lm::lmhead_rowpart_kernel<<<(unsigned)((n_rows + 255) / 256), 256, 0, s>>>(part, zy, n_split, n_rows,
                                                                               targets, col_offset, Vs, out);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_lmhead_tp_combine(const float4 *parts, int32_t R, const LossArgs &a, cudaStream_t s,
                                     int *launches) {
    if (a.n_rows == 0) return cudaSuccess;
    lm::lmhead_tp_combine_kernel<<<(unsigned)((a.n_rows + 255) / 256), 256, 0, s>>>(parts, R, a);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_lmhead_combine(const RowPart *part, const float *zy, int32_t n_split, const LossArgs &a,
                                  cudaStream_t s, int *launches) {
    if (a.n_rows == 0) return cudaSuccess;
    lm::lmhead_combine_kernel<<<(unsigned)((a.n_rows + 255) / 256), 256, 0, s>>>(part, zy, n_split, a);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace grpo
