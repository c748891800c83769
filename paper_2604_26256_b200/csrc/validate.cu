// validate.cu -- bit-exact integer checks of the paper's constraints on a
// packed training batch:
//   C1  every token of trajectory i comes from its version v_i
//   C2  no trajectory dropped: each prompt group has G members,
//              the batch has exactly TBS trajectories
//   C3  0 <= v(theta) - v(w_j) <= K (inclusive bound, Z8)
// plus structure (cu_seqlens, target range, finite behaviour log-probs).
//
// Kernel 1 (one thread per trajectory): trajectory checks, group counts and the
// |B_j| histogram by integer atomics (order-independent, so bit-exact).
// Kernel 2 (one CTA per trajectory whose rows the call holds): token checks,
// OR-ed into the trajectory's flags.  Kernel 3 (one CTA): GROUP_SIZE flags,
// which need final counts, and the summary.  Sharded over ranks,
// every rank runs kernel 1 over all trajectories and kernel 2 over its own,
// and the token-level counts join the ranks' packed sum (validate_combine).
#include "common.cuh"

namespace grpo {

// trajectory-level checks of all N trajectories (the O(N) metadata every rank holds):
// C3 gap, zero length, group id, group counts and the |B_j| histogram
__global__ void __launch_bounds__(256)
    validate_traj_kernel(const int64_t *__restrict__ version_ids, const int64_t *__restrict__ cu,
                         const int32_t *__restrict__ group_ids, int32_t N, int32_t P,
                         int64_t v_theta, int32_t K, uint32_t *__restrict__ flags,
                         int32_t *__restrict__ group_count, int32_t *__restrict__ stale_hist) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    uint32_t g = 0;
    const int64_t L = cu[i + 1] - cu[i];
    const int64_t gap = v_theta - version_ids[i];
    const int32_t p = group_ids[i];
    if (gap > K) g |= GRPO_FLAG_STALE;
    if (gap < 0) g |= GRPO_FLAG_FUTURE;
    if (L <= 0) g |= GRPO_FLAG_ZERO_LEN;
    if (p < 0 || p >= P) {
        g |= GRPO_FLAG_BAD_GROUP_ID;
    } else {
        atomicAdd(&group_count[p], 1);
        if (gap >= 0 && gap <= K) atomicAdd(&stale_hist[(int64_t)p * (K + 1) + gap], 1);
    }
    flags[i] = g;
}

// token-level checks (C1, target range, behaviour log-probs) of the trajectories whose rows
// this call holds: CTA j takes trajectory i = traj_index[j] (j when NULL) and its rows
// [tcu[j], tcu[j+1]) of the token arrays (clipped to [0, T_tok)), OR-ing its bits into
// flags[i] after the trajectory kernel wrote them
__global__ void __launch_bounds__(256)
    validate_tokens_kernel(const int64_t *__restrict__ version_ids,
                           const int64_t *__restrict__ token_version,
                           const int64_t *__restrict__ tcu, const int32_t *__restrict__ traj_index,
                           const int64_t *__restrict__ targets,
                           const float *__restrict__ logp_behav, int32_t n_tok_traj, int64_t T_tok,
                           int32_t V, uint32_t *__restrict__ flags) {
    const int32_t j = blockIdx.x;
    if (j >= n_tok_traj) return;
    const int32_t i = traj_index ? traj_index[j] : j;
    const int64_t vi = version_ids[i];
    const int64_t b = max(tcu[j], (int64_t)0), e = min(tcu[j + 1], T_tok);
    uint32_t f = 0;
    for (int64_t t = b + threadIdx.x; t < e; t += blockDim.x) {
        if (token_version && token_version[t] != vi) f |= GRPO_FLAG_C1_MIXED;
        const int64_t y = targets[t];
        if (y < 0 || y >= V) f |= GRPO_FLAG_BAD_TARGET;
        if (logp_behav) {
            const float lw = logp_behav[t];
            if (!(isfinite(lw) && lw <= 0.0f)) f |= GRPO_FLAG_BAD_LOGP_BEHAV;
        }
    }
    const uint32_t c1 = __syncthreads_or(f & GRPO_FLAG_C1_MIXED);
    const uint32_t bt = __syncthreads_or(f & GRPO_FLAG_BAD_TARGET);
    const uint32_t bl = __syncthreads_or(f & GRPO_FLAG_BAD_LOGP_BEHAV);
    if (threadIdx.x == 0) {
        const uint32_t g = (c1 ? GRPO_FLAG_C1_MIXED : 0) | (bt ? GRPO_FLAG_BAD_TARGET : 0) |
                           (bl ? GRPO_FLAG_BAD_LOGP_BEHAV : 0);
        if (g) atomicOr(&flags[i], g);
    }
}

__device__ __forceinline__ int64_t block_sum_i64(int64_t x, int64_t *sh) {
    // fixed-size block (1024) integer sum; integers make the order irrelevant
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, off);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = x;
    __syncthreads();
    int64_t r = 0;
    if (threadIdx.x < 32) {
        r = sh[threadIdx.x];
        for (int off = 16; off > 0; off >>= 1) r += __shfl_xor_sync(0xFFFFFFFFu, r, off);
    }
    return r;  // valid in thread 0
}

__global__ void __launch_bounds__(1024)
    validate_summary_kernel(const int64_t *__restrict__ version_ids,
                            const int64_t *__restrict__ cu, const int32_t *__restrict__ group_ids,
                            int32_t N, int64_t T, int32_t P, int32_t G, int32_t tbs,
                            int64_t v_theta, uint32_t *__restrict__ flags,
                            const int32_t *__restrict__ group_count,
                            grpo_validate_summary_t *__restrict__ out,
                            double *__restrict__ token_counts) {
    __shared__ int64_t sh[32];
    int64_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t mono_bad = 0;
    int64_t gmax = INT64_MIN, gmin = INT64_MAX;
    for (int32_t i = threadIdx.x; i < N; i += blockDim.x) {
        uint32_t f = flags[i];
        const int32_t p = group_ids[i];
        if (p >= 0 && p < P && group_count[p] != G) f |= GRPO_FLAG_GROUP_SIZE;
        flags[i] = f;
#pragma unroll
        for (int q = 0; q < 8; ++q) cnt[q] += (f >> q) & 1u;
        if (cu[i + 1] < cu[i]) mono_bad += 1;
        const int64_t gap = v_theta - version_ids[i];
        gmax = max(gmax, gap);
        gmin = min(gmin, gap);
    }
    int64_t wrong = 0, dropped = 0;
    for (int32_t p = threadIdx.x; p < P; p += blockDim.x) {
        const int32_t c = group_count[p];
        wrong += (c != G);
        dropped += (c < G) ? (int64_t)(G - c) : 0;
    }
    int64_t tot[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) tot[q] = block_sum_i64(cnt[q], sh);
    const int64_t t_mono = block_sum_i64(mono_bad, sh);
    const int64_t t_wrong = block_sum_i64(wrong, sh);
    const int64_t t_drop = block_sum_i64(dropped, sh);
    // max / min of the gaps
    for (int off = 16; off > 0; off >>= 1) {
        gmax = max(gmax, (int64_t)__shfl_xor_sync(0xFFFFFFFFu, gmax, off));
        gmin = min(gmin, (int64_t)__shfl_xor_sync(0xFFFFFFFFu, gmin, off));
    }
    __shared__ int64_t smax[32], smin[32];
    if ((threadIdx.x & 31) == 0) {
        smax[threadIdx.x >> 5] = gmax;
        smin[threadIdx.x >> 5] = gmin;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            gmax = max(gmax, smax[w]);
            gmin = min(gmin, smin[w]);
        }
        grpo_validate_summary_t s;
        s.n_traj = N;
        s.n_tokens = cu[N];
        s.n_stale = tot[0];
        s.n_future = tot[1];
        s.n_zero_len = tot[2];
        s.n_bad_group_id = tot[3];
        s.n_group_size = tot[4];
        s.n_c1_mixed = tot[5];
        s.n_bad_target = tot[6];
        s.n_bad_logp_behav = tot[7];
        s.n_groups_wrong_size = t_wrong;
        s.c2_dropped = t_drop;
        s.max_staleness = N > 0 ? gmax : 0;
        s.min_staleness = N > 0 ? gmin : 0;
        s.cu_ok = (cu[0] == 0) && (cu[N] == T) && (t_mono == 0);
        s.tbs_ok = (N == tbs);
        s.c1_ok = (s.n_c1_mixed == 0);
        s.c2_ok = s.tbs_ok && s.n_groups_wrong_size == 0 && s.n_bad_group_id == 0;
        s.c3_ok = (s.n_stale == 0) && (s.n_future == 0);
        s.valid = s.cu_ok && s.c1_ok && s.c2_ok && s.c3_ok && s.n_zero_len == 0 &&
                  s.n_bad_target == 0 && s.n_bad_logp_behav == 0;
        *out = s;
        if (token_counts) {  // this call's token-level counts, for the ranks' packed sum
            token_counts[0] = (double)s.n_c1_mixed;
            token_counts[1] = (double)s.n_bad_target;
            token_counts[2] = (double)s.n_bad_logp_behav;
        }
    }
}

// the token-level counts of all ranks (summed, exact integers in fp64) into a summary whose
// trajectory-level fields every rank computed identically; the verdicts follow
__global__ void validate_combine_kernel(grpo_validate_summary_t *__restrict__ out,
                                        const double *__restrict__ token_counts) {
    grpo_validate_summary_t s = *out;
    s.n_c1_mixed = (int64_t)token_counts[0];
    s.n_bad_target = (int64_t)token_counts[1];
    s.n_bad_logp_behav = (int64_t)token_counts[2];
    s.c1_ok = (s.n_c1_mixed == 0);
    s.valid = s.cu_ok && s.c1_ok && s.c2_ok && s.c3_ok && s.n_zero_len == 0 &&
              s.n_bad_target == 0 && s.n_bad_logp_behav == 0;
    *out = s;
}

// out[k] = sum over ranks q = 0, 1, ... of gathered[q * n + k], in rank order (the same bits
// on every rank and in every run, unlike a collective's reduction order)
__global__ void combine_ranks_kernel(const double *__restrict__ gathered, int32_t world, int32_t n,
                                     double *__restrict__ out) {
    for (int32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        double acc = gathered[k];
        for (int32_t q = 1; q < world; ++q) acc += gathered[(int64_t)q * n + k];
        out[k] = acc;
    }
}

cudaError_t launch_validate(const int64_t *version_ids, const int64_t *cu, const int32_t *group_ids,
                            int32_t N, int64_t T, int32_t P, int32_t V, int32_t G, int32_t tbs,
                            int64_t v_theta, int32_t K, const int64_t *token_version,
                            const int64_t *targets, const float *logp_behav, const int64_t *tcu,
                            const int32_t *traj_index, int32_t n_tok_traj, int64_t T_tok,
                            uint32_t *flags, int32_t *group_count, int32_t *stale_hist,
                            grpo_validate_summary_t *summary, double *token_counts, cudaStream_t s,
                            int *launches) {
    cudaError_t e = cudaMemsetAsync(group_count, 0, sizeof(int32_t) * (size_t)P, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(stale_hist, 0, sizeof(int32_t) * (size_t)P * (size_t)(K + 1), s);
    if (e != cudaSuccess) return e;
    if (N > 0) {
        validate_traj_kernel<<<(N + 255) / 256, 256, 0, s>>>(version_ids, cu, group_ids, N, P, v_theta,
                                                             K, flags, group_count, stale_hist);
        *launches += 1;
    }
    if (n_tok_traj > 0) {
        validate_tokens_kernel<<<n_tok_traj, 256, 0, s>>>(version_ids, token_version, tcu, traj_index,
                                                          targets, logp_behav, n_tok_traj, T_tok, V,
                                                          flags);
        *launches += 1;
    }
    validate_summary_kernel<<<1, 1024, 0, s>>>(version_ids, cu, group_ids, N, T, P, G, tbs,
                                               v_theta, flags, group_count, summary, token_counts);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_validate_combine(grpo_validate_summary_t *summary, const double *token_counts,
                                    cudaStream_t s, int *launches) {
    validate_combine_kernel<<<1, 1, 0, s>>>(summary, token_counts);
    *launches += 1;
    return cudaGetLastError();
}

cudaError_t launch_combine_ranks(const double *gathered, int32_t world, int32_t n, double *out,
                                 cudaStream_t s, int *launches) {
    if (n <= 0) return cudaSuccess;
    combine_ranks_kernel<<<(n + 255) / 256, 256, 0, s>>>(gathered, world, n, out);
    *launches += 1;
    return cudaGetLastError();
}

}  // namespace grpo
