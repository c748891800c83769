/* examples/c_abi_example.c -- the fused async-GRPO loss from plain C through the C ABI
 * (include/grpo_async.h), no Python: one prompt group of G = 4 responses, V = 1000,
 * random bf16 logits; validate, advantages, one fused forward + backward chunk, then the
 * loss J and the stats are copied back and printed.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_example.c \
 *       -L paper_2604_26256_b200 -lgrpo_async -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2604_26256_b200 -o build/c_abi_example
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "grpo_async.h"

#define CHECK(call)                                                                    \
    do {                                                                               \
        grpo_status_t st_ = (call);                                                    \
        if (st_ != GRPO_OK) {                                                          \
            fprintf(stderr, "%s failed: %d %s\n", #call, (int)st_, grpo_last_error()); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

static uint16_t to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

int main(void) {
    enum { N = 4, P = 1, G = 4, K = 2, V = 1000 };
    const int64_t lens[N] = {5, 3, 7, 2};
    int64_t cu[N + 1] = {0};
    for (int i = 0; i < N; ++i) cu[i + 1] = cu[i] + lens[i];
    const int64_t T = cu[N], ld = V;
    int32_t gid[N] = {0, 0, 0, 0};
    int64_t ver[N] = {9, 9, 8, 10};
    float rew[N] = {1.0f, 0.0f, 0.0f, 1.0f};
    int64_t *tgt = (int64_t *)malloc(T * sizeof(int64_t));
    float *lw = (float *)malloc(T * sizeof(float));
    uint16_t *z = (uint16_t *)malloc(T * ld * sizeof(uint16_t));
    srand(7);
    for (int64_t t = 0; t < T; ++t) {
        tgt[t] = rand() % V;
        lw[t] = -7.0f - (float)(rand() % 100) / 100.0f;
        for (int v = 0; v < V; ++v) z[t * ld + v] = to_bf16((float)(rand() % 2001 - 1000) / 500.0f);
    }
    /* device copies of the batch */
    int64_t *d_cu, *d_ver, *d_tgt;
    int32_t *d_gid, *d_gc, *d_sh;
    uint32_t *d_flags;
    float *d_rew, *d_lw, *d_adv, *d_inv;
    uint16_t *d_z, *d_dz;
    double *d_ts, *d_stats;
    grpo_validate_summary_t *d_sum;
    cudaMalloc((void **)&d_cu, sizeof cu);
    cudaMalloc((void **)&d_ver, sizeof ver);
    cudaMalloc((void **)&d_gid, sizeof gid);
    cudaMalloc((void **)&d_rew, sizeof rew);
    cudaMalloc((void **)&d_tgt, T * sizeof(int64_t));
    cudaMalloc((void **)&d_lw, T * sizeof(float));
    cudaMalloc((void **)&d_z, T * ld * sizeof(uint16_t));
    cudaMalloc((void **)&d_dz, T * ld * sizeof(uint16_t));
    cudaMalloc((void **)&d_adv, N * sizeof(float));
    cudaMalloc((void **)&d_inv, N * sizeof(float));
    cudaMalloc((void **)&d_flags, N * sizeof(uint32_t));
    cudaMalloc((void **)&d_gc, P * sizeof(int32_t));
    cudaMalloc((void **)&d_sh, P * (K + 1) * sizeof(int32_t));
    cudaMalloc((void **)&d_sum, sizeof(grpo_validate_summary_t));
    cudaMalloc((void **)&d_ts, N * sizeof(double));
    cudaMalloc((void **)&d_stats, GRPO_NUM_STATS * sizeof(double));
    cudaMemcpy(d_cu, cu, sizeof cu, cudaMemcpyHostToDevice);
    cudaMemcpy(d_ver, ver, sizeof ver, cudaMemcpyHostToDevice);
    cudaMemcpy(d_gid, gid, sizeof gid, cudaMemcpyHostToDevice);
    cudaMemcpy(d_rew, rew, sizeof rew, cudaMemcpyHostToDevice);
    cudaMemcpy(d_tgt, tgt, T * sizeof(int64_t), cudaMemcpyHostToDevice);
    cudaMemcpy(d_lw, lw, T * sizeof(float), cudaMemcpyHostToDevice);
    cudaMemcpy(d_z, z, T * ld * sizeof(uint16_t), cudaMemcpyHostToDevice);
    cudaMemset(d_ts, 0, N * sizeof(double));
    cudaMemset(d_stats, 0, GRPO_NUM_STATS * sizeof(double));
    const size_t ws_bytes = grpo_async_workspace_size(T, V, N);
    void *d_ws;
    cudaMalloc(&d_ws, ws_bytes);

    grpo_validate_summary_t summary;
    const grpo_status_t vs = grpo_async_validate_sync(d_ver, NULL, d_cu, d_gid, d_tgt, d_lw, N, T, P, V, G,
                                                      N, 10, K, d_flags, d_gc, d_sh, d_sum, &summary, NULL);
    if (vs != GRPO_OK && vs != GRPO_ERR_VALIDATION) return 1;
    printf("validate: valid=%lld c3_ok=%lld max_staleness=%lld\n", (long long)summary.valid,
           (long long)summary.c3_ok, (long long)summary.max_staleness);
    CHECK(grpo_async_advantage(d_rew, d_gid, d_cu, N, P, 1e-8f, d_adv, d_inv, NULL, NULL));
    CHECK(grpo_async_loss_fwd(d_z, 0, T, V, ld, d_tgt, d_lw, d_cu, N, NULL, d_adv, d_inv, 0.2f, 1.0f, NULL,
                              NULL, NULL, d_ts, d_stats, d_dz, d_ws, ws_bytes, NULL, NULL));
    double stats[GRPO_NUM_STATS];
    cudaMemcpy(stats, d_stats, sizeof stats, cudaMemcpyDeviceToHost);
    if (cudaDeviceSynchronize() != cudaSuccess) return 1;
    printf("J=%.9g rows=%.0f clipped=%.0f active=%.0f (%s)\n", stats[GRPO_STAT_J], stats[GRPO_STAT_ROWS],
           stats[GRPO_STAT_CLIPPED], stats[GRPO_STAT_ACTIVE], grpo_version());
    return (stats[GRPO_STAT_ROWS] == (double)T && isfinite(stats[GRPO_STAT_J])) ? 0 : 1;
}
