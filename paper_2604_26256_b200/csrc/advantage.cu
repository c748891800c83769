// advantage.cu -- group-relative advantages, eq:group_advantage:
// (with grpo_async_advantage_ex: DAPO token-mean weights and trajectory masks)
//   A_i = (R_i - mean_p) / std_p  over the members of prompt group p,
// population std (Z1; sample std with opts->std_unbiased), A = 0 exactly for a group whose rewards are
// bitwise equal, else denominator max(std, floor) (Z2), and the token weight
// inv_norm_i = 1 / (P * G_p * L_i) of eq:grpo_async (Z5, Z6).
//
// One warp per group.  The warp scans group_ids 32 at a time; the ballot of
// members is consumed lowest lane first, so the fp64 sums run over members
// in ascending trajectory index, one add at a time -- the same order as the
// plain definition, which makes the results bit-identical to it.
#include "common.cuh"

namespace grpo {

// A trajectory is kept in the loss when its group id is valid, L_i > 0 and the
// optional mask allows it.
__device__ __forceinline__ bool kept(const int32_t *group_ids, const int64_t *cu,
                                     const uint8_t *traj_mask, int32_t P, int32_t i) {
    const int32_t g = group_ids[i];
    return g >= 0 && g < P && cu[i + 1] > cu[i] && (!traj_mask || traj_mask[i]);
}

__global__ void __launch_bounds__(256)
    advantage_kernel(const float *__restrict__ rewards, const int32_t *__restrict__ group_ids,
                     const int64_t *__restrict__ cu, int32_t N, int32_t P, float std_floor,
                     int32_t norm, int32_t unbiased, const uint8_t *__restrict__ traj_mask,
                     float *__restrict__ adv, float *__restrict__ inv_norm,
                     int32_t *__restrict__ group_count) {
    const int lane = threadIdx.x & 31;
    const int32_t p = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (p >= P) return;
    // token-mean normalisation (DAPO): the kept tokens of the whole batch
    int64_t T_kept = 0;
    if (norm == GRPO_NORM_TOKEN) {
        for (int32_t i = lane; i < N; i += 32)
            if (kept(group_ids, cu, traj_mask, P, i)) T_kept += cu[i + 1] - cu[i];
        for (int off = 16; off > 0; off >>= 1) T_kept += __shfl_xor_sync(0xFFFFFFFFu, T_kept, off);
    }
    // pass 1: count, sum, bitwise equality
    int32_t n = 0;
    double sum = 0.0;
    bool all_equal = true;
    uint32_t first = 0;
    for (int32_t base = 0; base < N; base += 32) {
        const int32_t i = base + lane;
        const bool mine = (i < N) && (group_ids[i] == p);
        const float r = mine ? rewards[i] : 0.0f;
        uint32_t mask = __ballot_sync(0xFFFFFFFFu, mine);
        while (mask) {
            const int j = __ffs(mask) - 1;
            const float rj = __shfl_sync(0xFFFFFFFFu, r, j);
            const uint32_t bits = __float_as_uint(rj);
            if (n == 0) first = bits;
            else if (bits != first) all_equal = false;
            sum += (double)rj;
            n += 1;
            mask &= mask - 1;
        }
    }
    if (lane == 0 && group_count) group_count[p] = n;
    if (n == 0) return;
    const double mean = sum / (double)n;
    // pass 2: sum of squared deviations
    double ss = 0.0;
    for (int32_t base = 0; base < N; base += 32) {
        const int32_t i = base + lane;
        const bool mine = (i < N) && (group_ids[i] == p);
        const float r = mine ? rewards[i] : 0.0f;
        uint32_t mask = __ballot_sync(0xFFFFFFFFu, mine);
        while (mask) {
            const int j = __ffs(mask) - 1;
            const double d = (double)__shfl_sync(0xFFFFFFFFu, r, j) - mean;
            ss = __dadd_rn(ss, __dmul_rn(d, d));  // no FMA contraction
            mask &= mask - 1;
        }
    }
    const double sd = sqrt(ss / (double)(unbiased && n > 1 ? n - 1 : n));
    const double den = sd > (double)std_floor ? sd : (double)std_floor;
    // pass 3: outputs of the members (each lane writes its own)
    for (int32_t base = 0; base < N; base += 32) {
        const int32_t i = base + lane;
        if (i < N && group_ids[i] == p) {
            const double a = all_equal ? 0.0 : ((double)rewards[i] - mean) / den;
            const int64_t L = cu[i + 1] - cu[i];
            adv[i] = (float)a;
            if (!kept(group_ids, cu, traj_mask, P, i))
                inv_norm[i] = 0.0f;
            else if (norm == GRPO_NORM_TOKEN)
                inv_norm[i] = (float)(1.0 / (double)T_kept);
            else
                inv_norm[i] = (float)(1.0 / __dmul_rn(__dmul_rn((double)P, (double)n), (double)L));
        }
    }
}

// trajectories whose group id is invalid get A = 0, inv_norm = 0
__global__ void advantage_invalid_kernel(const int32_t *__restrict__ group_ids, int32_t N,
                                         int32_t P, float *__restrict__ adv,
                                         float *__restrict__ inv_norm) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const int32_t p = group_ids[i];
        if (p < 0 || p >= P) {
            adv[i] = 0.0f;
            inv_norm[i] = 0.0f;
        }
    }
}

cudaError_t launch_advantage(const float *rewards, const int32_t *group_ids, const int64_t *cu,
                             int32_t N, int32_t P, float std_floor, int32_t norm,
                             int32_t unbiased, const uint8_t *traj_mask, float *adv,
                             float *inv_norm, int32_t *group_count, cudaStream_t s, int *launches) {
    if (N > 0) {
        advantage_invalid_kernel<<<(N + 255) / 256, 256, 0, s>>>(group_ids, N, P, adv, inv_norm);
        *launches += 1;
    }
    const int64_t threads = (int64_t)P * 32;
    advantage_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
        rewards, group_ids, cu, N, P, std_floor, norm, unbiased, traj_mask, adv, inv_norm,
        group_count);
    *launches += 1;
    return cudaGetLastError();
}

// ---- sharded rewards: group partials, squared deviations, advantages from the stats
__global__ void __launch_bounds__(256)
    group_partials_kernel(const float *__restrict__ rewards, const int32_t *__restrict__ group_ids,
                          int32_t N, int32_t P, double *__restrict__ part) {
    const int lane = threadIdx.x & 31;
    const int32_t p = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (p >= P) return;
    double n = 0.0, sum = 0.0;
    uint32_t bmax = 0u, bmin = 0xFFFFFFFFu;
    for (int32_t base = 0; base < N; base += 32) {
        const int32_t i = base + lane;
        const bool mine = (i < N) && (group_ids[i] == p);
        const float r = mine ? rewards[i] : 0.0f;
        uint32_t mask = __ballot_sync(0xFFFFFFFFu, mine);
        while (mask) {  // members in ascending index, one add at a time (as the oracle)
            const int j = __ffs(mask) - 1;
            const float rj = __shfl_sync(0xFFFFFFFFu, r, j);
            sum += (double)rj;
            n += 1.0;
            bmax = max(bmax, __float_as_uint(rj));
            bmin = min(bmin, __float_as_uint(rj));
            mask &= mask - 1;
        }
    }
    if (lane == 0) {
        part[4 * (int64_t)p + 0] = n;
        part[4 * (int64_t)p + 1] = sum;
        part[4 * (int64_t)p + 2] = n > 0.0 ? (double)bmax : -1.0;            // MAX-combined
        part[4 * (int64_t)p + 3] = n > 0.0 ? -(double)bmin : -4294967296.0;  // MAX of -min
    }
}

__global__ void __launch_bounds__(256)
    kept_tokens_kernel(const int32_t *__restrict__ group_ids, const int64_t *__restrict__ cu,
                       const uint8_t *__restrict__ traj_mask, int32_t N, int32_t P, double *out) {
    __shared__ long long red[8];
    long long t = 0;
    for (int32_t i = threadIdx.x; i < N; i += blockDim.x)
        if (kept(group_ids, cu, traj_mask, P, i)) t += cu[i + 1] - cu[i];
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        *out = (double)s;
    }
}

__global__ void __launch_bounds__(256)
    group_sq_kernel(const float *__restrict__ rewards, const int32_t *__restrict__ group_ids,
                    int32_t N, int32_t P, const double *__restrict__ glob, double *__restrict__ ss) {
    const int lane = threadIdx.x & 31;
    const int32_t p = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (p >= P) return;
    const double n = glob[4 * (int64_t)p];
    const double mean = n > 0.0 ? glob[4 * (int64_t)p + 1] / n : 0.0;
    double acc = 0.0;
    for (int32_t base = 0; base < N; base += 32) {
        const int32_t i = base + lane;
        const bool mine = (i < N) && (group_ids[i] == p);
        const float r = mine ? rewards[i] : 0.0f;
        uint32_t mask = __ballot_sync(0xFFFFFFFFu, mine);
        while (mask) {
            const int j = __ffs(mask) - 1;
            const double d = (double)__shfl_sync(0xFFFFFFFFu, r, j) - mean;
            acc = __dadd_rn(acc, __dmul_rn(d, d));
            mask &= mask - 1;
        }
    }
    if (lane == 0) ss[p] = acc;
}

__global__ void advantage_from_stats_kernel(const float *__restrict__ rewards,
                                            const int32_t *__restrict__ group_ids,
                                            const int64_t *__restrict__ cu, int32_t N, int32_t P,
                                            float std_floor, int32_t norm, int32_t unbiased,
                                            const uint8_t *__restrict__ traj_mask,
                                            const double *__restrict__ glob,
                                            const double *__restrict__ ss, float *__restrict__ adv,
                                            float *__restrict__ inv_norm) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        const int32_t p = group_ids[i];
        if (p < 0 || p >= P) {
            adv[i] = 0.0f;
            inv_norm[i] = 0.0f;
            continue;
        }
        const double n = glob[4 * (int64_t)p], mean = glob[4 * (int64_t)p + 1] / n;
        const bool all_equal = glob[4 * (int64_t)p + 2] == -glob[4 * (int64_t)p + 3];
        const double sd = sqrt(ss[p] / (unbiased && n > 1.0 ? n - 1.0 : n));
        const double den = sd > (double)std_floor ? sd : (double)std_floor;
        adv[i] = all_equal ? 0.0f : (float)(((double)rewards[i] - mean) / den);
        const int64_t L = cu[i + 1] - cu[i];
        if (!kept(group_ids, cu, traj_mask, P, i)) inv_norm[i] = 0.0f;
        else if (norm == GRPO_NORM_TOKEN) inv_norm[i] = (float)(1.0 / glob[4 * (int64_t)P]);
        else inv_norm[i] = (float)(1.0 / __dmul_rn(__dmul_rn((double)P, n), (double)L));
    }
}

cudaError_t launch_group_partials(const float *rewards, const int32_t *group_ids, const int64_t *cu,
                                  int32_t N, int32_t P, const uint8_t *traj_mask, double *part,
                                  cudaStream_t s, int *launches) {
    const int64_t threads = (int64_t)P * 32;
    group_partials_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(rewards, group_ids, N, P, part);
    kept_tokens_kernel<<<1, 256, 0, s>>>(group_ids, cu, traj_mask, N, P, part + 4 * (int64_t)P);
    *launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_group_sq(const float *rewards, const int32_t *group_ids, int32_t N, int32_t P,
                            const double *glob, double *ss, cudaStream_t s, int *launches) {
    const int64_t threads = (int64_t)P * 32;
    group_sq_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(rewards, group_ids, N, P, glob, ss);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_advantage_from_stats(const float *rewards, const int32_t *group_ids, const int64_t *cu,
                                        int32_t N, int32_t P, float std_floor, int32_t norm,
                                        int32_t unbiased, const uint8_t *traj_mask, const double *glob,
                                        const double *ss, float *adv, float *inv_norm, cudaStream_t s,
                                        int *launches) {
    if (N == 0) return cudaSuccess;
    advantage_from_stats_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(
        rewards, group_ids, cu, N, P, std_floor, norm, unbiased, traj_mask, glob, ss, adv, inv_norm);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace grpo
