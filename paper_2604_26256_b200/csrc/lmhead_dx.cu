// lmhead_dx.cu -- the tensor-parallel LM head's input gradient as ONE kernel that computes
// and communicates: dX = sum_q dz_q W_q over the R ranks of a vocabulary-parallel group
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
#include "tc.cuh"

namespace grpo {
namespace lmdx {

constexpr int BM = 128, BK = 64, STAGES = 4, NUM_THREADS = 192;

struct Params {
    int32_t n_rows, d, Vs;
    int32_t m_tiles, n_tiles, n_units;
    int32_t world, rank, rows_per_rank;
    float *slots[GRPO_VP_MAX_RANKS];  // slot buffers of every rank: [world][rows_per_rank][d]
};

// Units (m_tile, n_tile) rastered in groups of GM row tiles (row tile fastest): the pairs
// running at the same time cover ~GM row tiles x ~grid/GM column tiles and, moving through
// K at about the same pace, share each A and B k-block in L2 instead of re-reading dz
// (K = the shard's vocabulary, tens of MB per row tile) from HBM.
constexpr int GM = 8;
__device__ __forceinline__ void dx_decode(const Params &p, int unit, int &m_tile, int &n_tile) {
    const int per_group = GM * p.n_tiles;
    const int grp = unit / per_group;
    const int rem = unit - grp * per_group;
    const int gm = min(GM, p.m_tiles - grp * GM);
    m_tile = grp * GM + rem % gm;
    n_tile = rem / gm;
}

// Shared-memory matrix descriptor, MN-major, 128-byte swizzle: 64-element rows along N,
// 8 K-rows per 1 KB atom (SBO = 1024 B between K atoms), N atoms of 64 elements LBO apart.
__device__ __forceinline__ uint64_t desc_mn_sw128(const void *smem_tile, uint32_t lbo_bytes) {
    const uint64_t addr = smem_u32(smem_tile);
    return ((addr >> 4) & 0x3FFFull) | ((uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16) | (64ull << 32) |
           (1ull << 46) | (2ull << 61);
}

// kind::f16, D f32, A bf16 K-major, B bf16 MN-major (bit 16)
__host__ __device__ constexpr uint32_t idesc_kmn(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// CG = 2: a CTA pair (cluster of 2, tcgen05.mma.cta_group::2, M = 256): each CTA stages
// its own 128 rows of dz and half of the tile's BN columns of W; the leader issues the MMA.
template <int BN, int CG>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dx_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Params p) {
    constexpr int A_BYTES = BM * BK * 2;          // 16 KB
    constexpr int NB = BN / 64 / CG;              // 64-wide N atoms staged per CTA
    constexpr int B_ATOM = BK * 64 * 2;           // 8 KB: 64 K-rows x 64 N elements
    constexpr int STAGE = A_BYTES + NB * B_ATOM;
    constexpr int NS = CG == 1 ? STAGES : 6;
    constexpr uint32_t TMEM_COLS = 2 * BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem, *sB = smem + NS * A_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NS * STAGE);
    uint64_t *full = bars, *empty = bars + NS, *tfull = bars + 2 * NS, *tempty = bars + 2 * NS + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * NS + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (p.Vs + BK - 1) / BK;
    const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;
    const int cta_id = CG == 2 ? (int)cluster_id_x() : (int)blockIdx.x;
    const int n_ctas = CG == 2 ? (int)ncluster_x() : (int)gridDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 128 * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
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
            const uint64_t pol = policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (int unit = cta_id; unit < p.n_units; unit += n_ctas) {
                int m_tile, n_tile;
                dx_decode(p, unit, m_tile, n_tile);
                const int a_row = m_tile * BM * CG + (int)crank * BM;
                const int b_col = n_tile * BN + (int)crank * (BN / CG);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1u);
                    if (CG == 1) {
                        mbar_arrive_expect_tx(full + stage, STAGE);
                        tc::tma_load_2d(sA + stage * A_BYTES, &tmA, kb * BK, a_row, full + stage, pol);
#pragma unroll
                        for (int j = 0; j < NB; ++j)
                            tc::tma_load_2d(sB + stage * NB * B_ATOM + j * B_ATOM, &tmB, b_col + j * 64, kb * BK,
                                            full + stage, pol);
                    } else {
                        if (crank == 0) mbar_arrive_expect_tx(full + stage, 2 * STAGE);
                        tc::tma_load_2d_pair(sA + stage * A_BYTES, &tmA, kb * BK, a_row, full + stage, pol);
#pragma unroll
                        for (int j = 0; j < NB; ++j)
                            tc::tma_load_2d_pair(sB + stage * NB * B_ATOM + j * B_ATOM, &tmB, b_col + j * 64,
                                                 kb * BK, full + stage, pol);
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
            constexpr uint32_t idesc = idesc_kmn(BM * CG, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int unit = cta_id; unit < p.n_units; unit += n_ctas) {
                mbar_wait(tempty + acc, acc_phase ^ 1u);
                tc::fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc::fence_after();
                    const uint64_t ad = tc::desc_k_sw128(sA + stage * A_BYTES);
                    const uint64_t bd = desc_mn_sw128(sB + stage * NB * B_ATOM, B_ATOM);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {  // A: +32 B inside its atom; B: +16 K-rows = 2 KB
                        if (CG == 1) tc::mma_bf16(d_tmem, ad + 2u * k, bd + 128u * k, idesc, (kb | k) != 0);
                        else tc::mma2_bf16(d_tmem, ad + 2u * k, bd + 128u * k, idesc, (kb | k) != 0);
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
    } else {  // ---- epilogue: each thread one row of the tile, straight to the owner's slot
        const int q = warp & 3;
        const int r_in_tile = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = cta_id; unit < p.n_units; unit += n_ctas) {
            int m_tile, n_tile;
            dx_decode(p, unit, m_tile, n_tile);
            const int row = m_tile * BM * CG + (int)crank * BM + r_in_tile;
            mbar_wait(tfull + acc, acc_phase);
            tc::fence_after();
            const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
            const bool valid = row < p.n_rows;
            const int owner = valid ? row / p.rows_per_rank : 0;
            float *dst = valid ? p.slots[owner] + ((int64_t)p.rank * p.rows_per_rank + (row - owner * p.rows_per_rank)) *
                                                      p.d + n_tile * BN
                               : nullptr;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                tc::tmem_ld32(t_row + (uint32_t)(c * 32), r);
                tc::tmem_wait_ld();
                if (valid) {
                    uint4 *d4 = reinterpret_cast<uint4 *>(dst + c * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j) d4[j] = make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
                }
            }
            tc::fence_before();
            if (CG == 1) mbar_arrive(tempty + acc);
            else tc::mbar_arrive_remote(tempty + acc, 0);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1u;
        }
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

cudaError_t launch_lmhead_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W, int64_t n_rows, int32_t d,
                             int32_t Vs, int32_t world, int32_t rank, float *const *slots, cudaStream_t s,
                             int *launches, char *why, size_t why_len) {
    using namespace lmdx;
    if (n_rows == 0) return cudaSuccess;
    const int BN = d % 256 == 0 ? 256 : 128;
    const int CG = 2;  // CTA pairs (tcgen05.mma.cta_group::2), as the LM-head kernel
    CUtensorMap ma, mb;
    if (!make_map(&ma, dz, n_rows, Vs, ld_dz, BM) || !make_map(&mb, W, Vs, d, d, BK)) {
        if (why) snprintf(why, why_len, "cuTensorMapEncodeTiled failed (alignment / driver entry point)");
        return cudaErrorInvalidValue;
    }
    Params p{};
    p.n_rows = (int32_t)n_rows;
    p.d = d;
    p.Vs = Vs;
    p.m_tiles = (int32_t)((n_rows + BM * CG - 1) / (BM * CG));
    p.n_tiles = d / BN;
    p.n_units = p.m_tiles * p.n_tiles;
    p.world = world;
    p.rank = rank;
    p.rows_per_rank = (int32_t)((n_rows + world - 1) / world);
    for (int q = 0; q < world; ++q) p.slots[q] = slots[q];
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int groups = std::min(p.n_units, n_sm / CG);
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
    if (BN == 256) {
        constexpr int SMEM = 6 * (BM * BK * 2 + 2 * BK * 64 * 2) + 1024 + 256;
        cfg.dynamicSmemBytes = SMEM;
        e = cudaFuncSetAttribute(dx_kernel<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        e = cudaLaunchKernelEx(&cfg, dx_kernel<256, 2>, ma, mb, p);
    } else {
        constexpr int SMEM = 6 * (BM * BK * 2 + 1 * BK * 64 * 2) + 1024 + 256;
        cfg.dynamicSmemBytes = SMEM;
        e = cudaFuncSetAttribute(dx_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        e = cudaLaunchKernelEx(&cfg, dx_kernel<128, 2>, ma, mb, p);
    }
    if (e != cudaSuccess) return e;
    e = cudaGetLastError();
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
