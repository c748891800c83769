// lmhead_dx.cu -- the LM head's backward GEMMs on the tensor cores:
// dX = dz W and dW += dz^T X from the bf16 logits gradient dz (launch_lmhead_gemm_dx / _dw),
// and the tensor-parallel LM head's input gradient as ONE kernel that computes and
// communicates: dX = sum_q dz_q W_q over the R ranks of a vocabulary-parallel group
// (Megatron layout), reduce-scattered by rows.  Each rank's tcgen05 GEMM computes
// its partial dz_q W_q (A = dz_q, K-major over the shard's vocabulary; B = W_q read
// MN-major, i.e. straight from the row-major [Vs, d] weight) and the epilogue stores every
// 128 x BN fp32 tile directly into the owner rank's slot buffer over NVLink (peer
// pointers): tile t of rank q lands in slot q of the rank that owns its rows while the
// tensor cores are already on the next tile.  After a group barrier each rank sums the R
// slots of its rows in rank order (lmhead_dx_reduce_kernel) -- deterministic, and the
// transfer is hidden under the GEMM instead of following it as an all-reduce.
#include <cudaTypedefs.h>

#include <cstdio>

#include "common.cuh"
#include "sched.cuh"
#include "tc.cuh"

namespace grpo {
namespace lmdx {

constexpr int BM = 128, BK = 64, STAGES = 4, NUM_THREADS = 192;
__device__ int32_t g_units[sched::N_COUNTERS];  // unit counters of the launches (sched.cuh)

// Epilogues: EPI_SLOTS stores f32 tiles into the owner rank's slot (the tensor-parallel
// dX reduce-scatter); EPI_BF16 / EPI_F32 store D; EPI_F32_ACC adds D into an f32 array.
enum { EPI_SLOTS = 0, EPI_BF16 = 1, EPI_F32 = 2, EPI_F32_ACC = 3 };

struct Params {
    int32_t M, N, K;                  // D[M, N] = A[M, K] * B[K, N]
    int32_t m_tiles, n_tiles, n_units;
    int32_t raster_n;                 // 0: row-tile groups, 1: column tile fastest, 2: column-tile groups
    int32_t gm;                       // raster_n = 0: row tiles per raster group
    int32_t pol_a, pol_b;             // L2 policies of the A / B loads: 0 normal, 1 evict_first, 2 evict_last
    int32_t *counter;                 // the launch's unit counter, 0 at launch (sched.cuh)
    int32_t world, rank, rows_per_rank;
    float *slots[GRPO_VP_MAX_RANKS];  // EPI_SLOTS: slot buffers of every rank [world][rows_per_rank][N]
    void *out;                        // EPI_BF16 / EPI_F32 / EPI_F32_ACC: [M][ldo]
    int64_t ldo;
};

// Units (m_tile, n_tile).  raster_n = 0: groups of p.gm row tiles, row tile fastest -- the pairs
// running at the same time cover ~GM row tiles x ~grid/GM column tiles and, moving through K
// at about the same pace, share each A and B k-block in L2 instead of re-reading the long-K
// operands (dX: K = the vocabulary, tens of MB per row tile) from HBM.  raster_n = 1: column
// tile fastest -- dW = dz^T X has K = the row count and a small B (X, ~84 MB at 8190 x 5120),
// so the column tiles of one row tile (one dz column block) run together and dz streams once.
// raster_n = 2: groups of p.gm column tiles, column tile fastest inside the group (dW: a group's
// share of B stays in L2 -- shared operands are cached per die in effect, ~60 MB before they
// thrash, scripts/probes/l2_probe.cu -- while A streams once per group).
__device__ __forceinline__ void decode(const Params &p, int unit, int &m_tile, int &n_tile) {
    const int GM = p.gm;
    if (p.raster_n == 2) {  // groups of GM column tiles, column tile fastest inside a group
        const int per_group = GM * p.m_tiles;
        const int grp = unit / per_group;
        const int rem = unit - grp * per_group;
        const int gn = min(GM, p.n_tiles - grp * GM);
        m_tile = rem / gn;
        n_tile = grp * GM + (rem - m_tile * gn);
        return;
    }
    if (p.raster_n) {
        m_tile = unit / p.n_tiles;
        n_tile = unit - m_tile * p.n_tiles;
        return;
    }
    const int per_group = GM * p.n_tiles;
    const int grp = unit / per_group;
    const int rem = unit - grp * per_group;
    const int gm = min(GM, p.m_tiles - grp * GM);
    m_tile = grp * GM + rem % gm;
    n_tile = rem / gm;
}

// Shared-memory matrix descriptor, MN-major, 128-byte swizzle: 64-element rows along M or N,
// 8 K-rows per 1 KB atom (SBO = 1024 B between K atoms), MN atoms of 64 elements LBO apart.
__device__ __forceinline__ uint64_t desc_mn_sw128(const void *smem_tile, uint32_t lbo_bytes) {
    const uint64_t addr = smem_u32(smem_tile);
    return ((addr >> 4) & 0x3FFFull) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) | (64ull << 32) |
           (1ull << 46) | (2ull << 61);
}

// kind::f16, D f32, A and B bf16; A K-major (bit 15 = 0) or MN-major (1), B MN-major (bit 16)
__host__ __device__ constexpr uint32_t idesc_b_mn(int M, int N, bool a_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | (1u << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// One persistent warp-specialised tcgen05 GEMM for the LM head's backward: warp 0 issues TMA
// (A: K-major 128 x 64 boxes, or MN-major 64 x 64 boxes; B: MN-major 64 x 64 boxes, i.e. both
// read straight from row-major [K, M] / [K, N] arrays without a transpose), warp 1 of the pair
// leader issues tcgen05.mma (M = 128 * CG, N = BN) into one of two TMEM accumulators, warps
// 2-5 of each CTA drain their 128 TMEM lanes (one thread = one row of D) into the epilogue.
// CG = 2: a CTA pair (cluster of 2, tcgen05.mma.cta_group::2): each CTA stages its own 128
// rows of A and half of the tile's BN columns of B.
// The epilogue of the store variants (EPI_BF16 / EPI_F32 / EPI_F32_ACC) stages each warp's 32
// rows x 128 bytes (32 f32 or 64 bf16 columns) in shared memory with the 128-byte swizzle (a
// thread writes its row's 16-byte chunk j at chunk j ^ (row & 7): conflict-free) and one lane
// issues a TMA tile store -- or, for dW += dz^T X, a TMA reduce-add -- of the box: coalesced
// 128-byte rows instead of 32 rows written 16 bytes at a time by 32 threads, rows beyond M
// clipped by the tensor map, and no read-modify-write traffic through the SM for dW.
// Two 4 KB buffers per warp; the store issued two boxes earlier must have read its buffer.
template <int EPI, int CG>
struct Epi {
    static constexpr int STAGING = EPI == EPI_SLOTS ? 0 : 4 * 2 * 4096;  // 4 warps x 2 buffers
};

template <bool A_MN, int BN, int CG, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO, const Params p) {
    constexpr int A_BYTES = BM * BK * 2;          // 16 KB
    constexpr int NB = BN / 64 / CG;              // 64-wide N atoms staged per CTA
    constexpr int ATOM = BK * 64 * 2;             // 8 KB: 64 K-rows x 64 MN elements
    constexpr int STAGE = A_BYTES + NB * ATOM;
    constexpr int NS = CG == 1 ? STAGES : 6;  // 6 x 32 KB + 32 KB of staging fits in 227 KB
    constexpr uint32_t TMEM_COLS = 2 * BN;
    static_assert(NB >= 1, "BN / CG must be a multiple of 64");
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem, *sB = smem + NS * A_BYTES;
    uint8_t *staging = smem + NS * STAGE;  // 1 KB aligned (STAGE is a multiple of 8 KB)
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NS * STAGE + Epi<EPI, CG>::STAGING);
    uint64_t *full = bars, *empty = bars + NS, *tfull = bars + 2 * NS, *tempty = bars + 2 * NS + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NS + 4);
    sched::Queue *uq = reinterpret_cast<sched::Queue *>(bars + 2 * NS + 6);  // dynamic units (sched.cuh)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (p.K + BK - 1) / BK;
    const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 128 * CG);
        }
        sched::init<CG>(uq);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
        if (EPI != EPI_SLOTS) tc::prefetch_tmap(&tmO);
    }
    if (warp == 1) {
        if (CG == 2) tc::tmem_alloc2(tmem_slot, TMEM_COLS);
        else tc::tmem_alloc(tmem_slot, TMEM_COLS);
    }
    tc::fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            auto mkpol = [](int c) {
                return c == 1 ? policy_evict_first() : c == 2 ? policy_evict_last() : policy_evict_normal();
            };
            const uint64_t pol_a = mkpol(p.pol_a), pol_b = mkpol(p.pol_b);
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0;; ++i) {
                const int unit = crank == 0 ? sched::fetch<CG>(uq, i, p.counter, p.n_units)
                                            : sched::next<CG>(uq, i, crank);
                if (unit < 0) break;
                int m_tile, n_tile;
                decode(p, unit, m_tile, n_tile);
                const int a_row = m_tile * BM * CG + (int)crank * BM;
                const int b_col = n_tile * BN + (int)crank * (BN / CG);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1u);
                    uint8_t *dA = sA + stage * A_BYTES;
                    uint8_t *dB = sB + stage * NB * ATOM;
                    if (CG == 1) {
                        mbar_arrive_expect_tx(full + stage, STAGE);
                        if (A_MN) {
                            tc::tma_load_2d(dA, &tmA, a_row, kb * BK, full + stage, pol_a);
                            tc::tma_load_2d(dA + ATOM, &tmA, a_row + 64, kb * BK, full + stage, pol_a);
                        } else {
                            tc::tma_load_2d(dA, &tmA, kb * BK, a_row, full + stage, pol_a);
                        }
#pragma unroll
                        for (int j = 0; j < NB; ++j)
                            tc::tma_load_2d(dB + j * ATOM, &tmB, b_col + j * 64, kb * BK, full + stage, pol_b);
                    } else {
                        if (crank == 0) mbar_arrive_expect_tx(full + stage, 2 * STAGE);
                        if (A_MN) {
                            tc::tma_load_2d_pair(dA, &tmA, a_row, kb * BK, full + stage, pol_a);
                            tc::tma_load_2d_pair(dA + ATOM, &tmA, a_row + 64, kb * BK, full + stage, pol_a);
                        } else {
                            tc::tma_load_2d_pair(dA, &tmA, kb * BK, a_row, full + stage, pol_a);
                        }
#pragma unroll
                        for (int j = 0; j < NB; ++j)
                            tc::tma_load_2d_pair(dB + j * ATOM, &tmB, b_col + j * 64, kb * BK, full + stage, pol_b);
                    }
                    if (++stage == NS) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && crank == 0) {  // ---- MMA issuer (the pair's leader)
            constexpr uint32_t idesc = idesc_b_mn(BM * CG, BN, A_MN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int i = 0;; ++i) {
                const int unit = sched::next<CG>(uq, i, 0u);
                if (unit < 0) break;
                mbar_wait(tempty + acc, acc_phase ^ 1u);
                tc::fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc::fence_after();
                    const uint64_t ad = A_MN ? desc_mn_sw128(sA + stage * A_BYTES, ATOM)
                                             : tc::desc_k_sw128(sA + stage * A_BYTES);
                    const uint64_t bd = desc_mn_sw128(sB + stage * NB * ATOM, ATOM);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // K-major A: +32 B inside its swizzle atom; MN-major: +16 K-rows = 2 KB
                        const uint64_t a_k = A_MN ? ad + 128u * k : ad + 2u * k;
                        if (CG == 1) tc::mma_bf16(d_tmem, a_k, bd + 128u * k, idesc, (kb | k) != 0);
                        else tc::mma2_bf16(d_tmem, a_k, bd + 128u * k, idesc, (kb | k) != 0);
                    }
                    if (CG == 1) tc::commit(empty + stage);
                    else tc::commit2_multicast(empty + stage, 0x3);
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
    } else {  // ---- epilogue: each thread one row of the tile
        const int q = warp & 3;
        const int r_in_tile = q * 32 + lane;
        uint8_t *wbuf = staging + q * 8192;  // this warp's two 4 KB boxes
        int n_boxes = 0;                     // boxes this warp has handed to TMA
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int i = 0;; ++i) {
            int unit = 0;
            if (lane == 0) unit = sched::next<CG>(uq, i, crank);
            unit = __shfl_sync(0xffffffffu, unit, 0);
            if (unit < 0) break;
            int m_tile, n_tile;
            decode(p, unit, m_tile, n_tile);
            const int row0 = m_tile * BM * CG + (int)crank * BM;  // first row of this CTA's 128
            const int row = row0 + r_in_tile;
            mbar_wait(tfull + acc, acc_phase);
            tc::fence_after();
            const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
            if (EPI == EPI_SLOTS) {
                const bool valid = row < p.M;
                float *slot_dst = nullptr;
                if (valid) {
                    const int owner = row / p.rows_per_rank;
                    slot_dst = p.slots[owner] +
                               ((int64_t)p.rank * p.rows_per_rank + (row - owner * p.rows_per_rank)) * p.N +
                               n_tile * BN;
                }
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tc::tmem_ld32(t_row + (uint32_t)(c * 32), r);
                    tc::tmem_wait_ld();
                    if (!valid) continue;
                    uint4 *d4 = reinterpret_cast<uint4 *>(slot_dst + c * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j) d4[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
                }
            } else {
                // one box = 32 rows x 128 bytes: 32 f32 columns, or 64 bf16 columns (two loads)
                constexpr int COLS = EPI == EPI_BF16 ? 64 : 32;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += COLS) {
                    uint32_t r[32], r2[32];
                    tc::tmem_ld32(t_row + (uint32_t)c0, r);
                    if (EPI == EPI_BF16) tc::tmem_ld32(t_row + (uint32_t)(c0 + 32), r2);
                    tc::tmem_wait_ld();
                    uint8_t *box = wbuf + (n_boxes & 1) * 4096;
                    if (n_boxes >= 2) {  // the store of two boxes ago has read this buffer
                        if (lane == 0) tc::bulk_wait_read<1>();
                        __syncwarp();
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        uint4 v;
                        if (EPI == EPI_BF16) {
                            const uint32_t *src = j < 4 ? r : r2;
                            const int o = (j & 3) * 8;
                            v = make_uint4(pack_bf16x2(__uint_as_float(src[o]), __uint_as_float(src[o + 1])),
                                           pack_bf16x2(__uint_as_float(src[o + 2]), __uint_as_float(src[o + 3])),
                                           pack_bf16x2(__uint_as_float(src[o + 4]), __uint_as_float(src[o + 5])),
                                           pack_bf16x2(__uint_as_float(src[o + 6]), __uint_as_float(src[o + 7])));
                        } else {
                            v = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
                        }
                        *reinterpret_cast<uint4 *>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) = v;
                    }
                    tc::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int col = n_tile * BN + c0, rr = row0 + q * 32;
                        if (EPI == EPI_F32_ACC) tc::tma_reduce_add_2d(&tmO, box, col, rr);
                        else tc::tma_store_2d(&tmO, box, col, rr);
                        tc::bulk_commit();
                    }
                    ++n_boxes;
                }
            }
            tc::fence_before();
            if (CG == 1) mbar_arrive(tempty + acc);
            else tc::mbar_arrive_remote(tempty + acc, 0);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1u;
        }
        if (EPI != EPI_SLOTS && lane == 0) tc::bulk_wait_all();  // stores done before smem goes away
    }
    tc::fence_before();
    __syncthreads();
    if (CG == 2) cluster_sync_all();
    if (warp == 1) {
        if (CG == 2) tc::tmem_dealloc2(tmem_base, TMEM_COLS);
        else tc::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// this rank's rows: the world slots summed in rank order (f32 -> out type)
template <typename OutT>
__global__ void __launch_bounds__(256) dx_reduce_kernel(const float *__restrict__ slots, int32_t world,
                                                       int64_t rows, int32_t d, int64_t rows_per_rank,
                                                       OutT *__restrict__ out) {
    const int64_t n4 = rows * (int64_t)d / 4;
    const int64_t slot_stride = rows_per_rank * (int64_t)d / 4;
    const float4 *s4 = reinterpret_cast<const float4 *>(slots);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 acc = s4[i];
        for (int q = 1; q < world; ++q) {
            const float4 v = s4[(int64_t)q * slot_stride + i];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        if constexpr (sizeof(OutT) == 4) {
            reinterpret_cast<float4 *>(out)[i] = acc;
        } else {
            reinterpret_cast<uint2 *>(out)[i] = make_uint2(pack_bf16x2(acc.x, acc.y), pack_bf16x2(acc.z, acc.w));
        }
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// bf16 [rows, inner] with row stride `stride` elements; box [box_rows, 64] (128-byte swizzle)
static bool make_map(CUtensorMap *m, const void *base, int64_t rows, int64_t inner, int64_t stride, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)stride * 2};
    cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace lmdx

namespace lmdx {

// launch gemm_kernel<A_MN, BN, CG, EPI> persistently: one CTA (pair) per SM (pair)
template <bool A_MN, int BN, int CG, int EPI>
static cudaError_t launch_gemm(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mo, Params &p,
                               cudaStream_t s) {
    if (p.gm <= 0) p.gm = 8;
    constexpr int NB = BN / 64 / CG;
    constexpr int NS = CG == 1 ? STAGES : 6;  // 6 x 32 KB + 32 KB of staging fits in 227 KB
    constexpr int SMEM = NS * (BM * BK * 2 + NB * BK * 64 * 2) + Epi<EPI, CG>::STAGING + 1024 + 256;
    p.m_tiles = (p.M + BM * CG - 1) / (BM * CG);
    p.n_tiles = p.N / BN;
    p.n_units = p.m_tiles * p.n_tiles;
    if (p.raster_n) {  // dW (K = the row count): dynamic units; dX (K = V): static (sched.cuh)
        int32_t *base = nullptr;
        cudaError_t ec = cudaGetSymbolAddress(reinterpret_cast<void **>(&base), g_units);
        if (ec == cudaSuccess) ec = sched::take_counter(base, s, &p.counter);
        if (ec != cudaSuccess) return ec;
    }
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int groups = std::min(p.n_units, n_sm / CG);
    auto kfn = gemm_kernel<A_MN, BN, CG, EPI>;
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CG;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(groups * CG));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kfn, ma, mb, mo, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// the N tile by the GEMM's N (= d): 256 with CTA pairs, 128 with pairs, 64 on one CTA
template <bool A_MN, int EPI>
static cudaError_t launch_by_n(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mo, Params &p,
                               cudaStream_t s) {
    if (p.N % 256 == 0) return launch_gemm<A_MN, 256, 2, EPI>(ma, mb, mo, p, s);
    if (p.N % 128 == 0) return launch_gemm<A_MN, 128, 2, EPI>(ma, mb, mo, p, s);
    return launch_gemm<A_MN, 64, 1, EPI>(ma, mb, mo, p, s);
}

// the output of the store epilogues: [rows, cols] row-major (leading dimension ld elements),
// box = 32 rows x 128 bytes, 128-byte swizzle (the staging layout of the epilogue)
static bool make_out_map(CUtensorMap *m, void *base, int64_t rows, int64_t cols, int64_t ld, bool bf16) {
    auto fn = encode_fn();
    if (!fn) return false;
    const int esz = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32u};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims,
              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace lmdx

cudaError_t launch_lmhead_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W, int64_t n_rows, int32_t d,
                             int32_t Vs, int32_t world, int32_t rank, float *const *slots, cudaStream_t s,
                             int *launches, char *why, size_t why_len) {
    using namespace lmdx;
    if (n_rows == 0) return cudaSuccess;
    CUtensorMap ma, mb;
    if (!make_map(&ma, dz, n_rows, Vs, ld_dz, BM) || !make_map(&mb, W, Vs, d, d, BK)) {
        if (why) snprintf(why, why_len, "cuTensorMapEncodeTiled failed (alignment / driver entry point)");
        return cudaErrorInvalidValue;
    }
    Params p{};
    p.M = (int32_t)n_rows;
    p.N = d;
    p.K = Vs;
    p.world = world;
    p.rank = rank;
    p.rows_per_rank = (int32_t)((n_rows + world - 1) / world);
    p.gm = 16;    // as launch_lmhead_gemm_dx
    p.pol_a = 1;
    for (int q = 0; q < world; ++q) p.slots[q] = slots[q];
    cudaError_t e = d % 256 == 0 ? launch_gemm<false, 256, 2, EPI_SLOTS>(ma, mb, ma, p, s)
                                 : launch_gemm<false, 128, 2, EPI_SLOTS>(ma, mb, ma, p, s);
    if (e != cudaSuccess) return e;
    *launches += 1;
    return cudaSuccess;
}

// dX = dz W  (A = dz [n_rows, V] K-major, B = W [V, d] MN-major): out [n_rows, d] bf16 or f32
cudaError_t launch_lmhead_gemm_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W, int64_t n_rows,
                                  int32_t d, int32_t V, void *out, int out_bf16, cudaStream_t s, int *launches,
                                  char *why, size_t why_len) {
    using namespace lmdx;
    if (n_rows == 0) return cudaSuccess;
    CUtensorMap ma, mb, mo;
    if (!make_map(&ma, dz, n_rows, V, ld_dz, BM) || !make_map(&mb, W, V, d, d, BK) ||
        !make_out_map(&mo, out, n_rows, d, d, out_bf16 != 0)) {
        if (why) snprintf(why, why_len, "cuTensorMapEncodeTiled failed (alignment / driver entry point)");
        return cudaErrorInvalidValue;
    }
    Params p{};
    p.M = (int32_t)n_rows;
    p.N = d;
    p.K = V;
    // 16 pair tiles of rows per raster group, dz streamed (evict_first): back-to-back 9.9 vs
    // 10.3 ms at 8190 x 5120 x 152064 for 8 and evict_normal (profiles/r02_lmhead_raster.txt)
    p.gm = 16;
    p.pol_a = 1;
    p.out = out;
    p.ldo = d;
    const cudaError_t e = out_bf16 ? launch_by_n<false, EPI_BF16>(ma, mb, mo, p, s)
                                   : launch_by_n<false, EPI_F32>(ma, mb, mo, p, s);
    if (e != cudaSuccess) return e;
    *launches += 1;
    return cudaSuccess;
}

// dW += dz^T X  (A = dz^T: dz [n_rows, V] read MN-major, B = X [n_rows, d] MN-major, K = n_rows):
// dW [V, d] f32, accumulated
cudaError_t launch_lmhead_gemm_dw(const uint16_t *dz, int64_t ld_dz, const uint16_t *X, int64_t n_rows,
                                  int32_t d, int32_t V, float *dW, cudaStream_t s, int *launches, char *why,
                                  size_t why_len) {
    using namespace lmdx;
    if (n_rows == 0) return cudaSuccess;
    CUtensorMap ma, mb, mo;
    if (!make_map(&ma, dz, n_rows, V, ld_dz, BK) || !make_map(&mb, X, n_rows, d, d, BK) ||
        !make_out_map(&mo, dW, V, d, d, false)) {
        if (why) snprintf(why, why_len, "cuTensorMapEncodeTiled failed (alignment / driver entry point)");
        return cudaErrorInvalidValue;
    }
    Params p{};
    p.M = V;
    p.N = d;
    p.K = (int32_t)n_rows;
    // groups of 10 column tiles (half of X, 42 MB at 8190 x 5120: it stays in L2 while the
    // group's dz blocks stream twice), column tile fastest: DRAM reads 21 vs 27 GB for the
    // whole of X per row tile, back-to-back 10.3 vs 10.5 ms (profiles/r02_lmhead_raster.txt)
    p.raster_n = 2;
    p.gm = 10;
    p.out = dW;
    p.ldo = d;
    const cudaError_t e = launch_by_n<true, EPI_F32_ACC>(ma, mb, mo, p, s);
    if (e != cudaSuccess) return e;
    *launches += 1;
    return cudaSuccess;
}

cudaError_t launch_lmhead_dx_reduce(const float *own_slots, int32_t world, int64_t n_rows, int32_t d,
                                    int32_t rank, void *out, int out_bf16, cudaStream_t s, int *launches) {
    const int64_t rpr = (n_rows + world - 1) / world;
    const int64_t r0 = (int64_t)rank * rpr;
    const int64_t rows = std::max<int64_t>(0, std::min<int64_t>(rpr, n_rows - r0));
    if (rows == 0) return cudaSuccess;
    const int64_t n4 = rows * d / 4;
    const unsigned blocks = (unsigned)std::min<int64_t>((n4 + 255) / 256, 148 * 8);
    if (out_bf16)
        lmdx::dx_reduce_kernel<uint16_t><<<blocks, 256, 0, s>>>(own_slots, world, rows, d, rpr,
                                                               static_cast<uint16_t *>(out));
    else
        lmdx::dx_reduce_kernel<float><<<blocks, 256, 0, s>>>(own_slots, world, rows, d, rpr, static_cast<float *>(out));
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace grpo
