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

template <int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    dx_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Params p) {
    constexpr int A_BYTES = BM * BK * 2;          // 16 KB
    constexpr int NB = BN / 64;                   // 64-wide N atoms per tile
    constexpr int B_ATOM = BK * 64 * 2;           // 8 KB: 64 K-rows x 64 N elements
    constexpr int STAGE = A_BYTES + NB * B_ATOM;
    constexpr uint32_t TMEM_COLS = 2 * BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = smem, *sB = smem + STAGES * A_BYTES;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE);
    uint64_t *full = bars, *empty = bars + STAGES, *tfull = bars + 2 * STAGES, *tempty = bars + 2 * STAGES + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 2 * STAGES + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nk = (p.Vs + BK - 1) / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + a, 1);
            mbar_init(tempty + a, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            const uint64_t pol = policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (int unit = blockIdx.x; unit < p.n_units; unit += gridDim.x) {
                const int m_tile = unit % p.m_tiles, n_tile = unit / p.m_tiles;
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(empty + stage, phase ^ 1u);
                    mbar_arrive_expect_tx(full + stage, STAGE);
                    tc::tma_load_2d(sA + stage * A_BYTES, &tmA, kb * BK, m_tile * BM, full + stage, pol);
#pragma unroll
                    for (int j = 0; j < NB; ++j)  // 64 vocabulary rows x 64 columns of W each
                        tc::tma_load_2d(sB + stage * NB * B_ATOM + j * B_ATOM, &tmB, n_tile * BN + j * 64, kb * BK,
                                        full + stage, pol);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            constexpr uint32_t idesc = idesc_kmn(BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int unit = blockIdx.x; unit < p.n_units; unit += gridDim.x) {
                mbar_wait(tempty + acc, acc_phase ^ 1u);
                tc::fence_after();
                const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc::fence_after();
                    const uint64_t ad = tc::desc_k_sw128(sA + stage * A_BYTES);
                    const uint64_t bd = desc_mn_sw128(sB + stage * NB * B_ATOM, B_ATOM);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)  // A: +32 B inside its atom; B: +16 K-rows = 2 KB
                        tc::mma_bf16(d_tmem, ad + 2u * k, bd + 128u * k, idesc, (kb | k) != 0);
                    tc::commit(empty + stage);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                tc::commit(tfull + acc);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1u;
            }
        }
    } else {  // ---- epilogue: each thread one row of the tile, straight to the owner's slot
        const int q = warp & 3;
        const int r_in_tile = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int unit = blockIdx.x; unit < p.n_units; unit += gridDim.x) {
            const int m_tile = unit % p.m_tiles, n_tile = unit / p.m_tiles;
            const int row = m_tile * BM + r_in_tile;
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
            mbar_arrive(tempty + acc);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1u;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem_base, TMEM_COLS);
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
    CUtensorMap ma, mb;
    if (!make_map(&ma, dz, n_rows, Vs, ld_dz, BM) || !make_map(&mb, W, Vs, d, d, BK)) {
        if (why) snprintf(why, why_len, "cuTensorMapEncodeTiled failed (alignment / driver entry point)");
        return cudaErrorInvalidValue;
    }
    Params p{};
    p.n_rows = (int32_t)n_rows;
    p.d = d;
    p.Vs = Vs;
    p.m_tiles = (int32_t)((n_rows + BM - 1) / BM);
    p.n_tiles = d / BN;
    p.n_units = p.m_tiles * p.n_tiles;
    p.world = world;
    p.rank = rank;
    p.rows_per_rank = (int32_t)((n_rows + world - 1) / world);
    for (int q = 0; q < world; ++q) p.slots[q] = slots[q];
    int dev = 0, n_sm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(p.n_units, n_sm);
    cudaError_t e;
    if (BN == 256) {
        constexpr int SMEM = STAGES * (BM * BK * 2 + 4 * BK * 64 * 2) + 1024 + 256;
        e = cudaFuncSetAttribute(dx_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        dx_kernel<256><<<grid, NUM_THREADS, SMEM, s>>>(ma, mb, p);
    } else {
        constexpr int SMEM = STAGES * (BM * BK * 2 + 2 * BK * 64 * 2) + 1024 + 256;
        e = cudaFuncSetAttribute(dx_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
        if (e != cudaSuccess) return e;
        dx_kernel<128><<<grid, NUM_THREADS, SMEM, s>>>(ma, mb, p);
    }
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
