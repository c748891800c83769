// api.cu -- the extern "C" boundary declared in include/grpo_async.h.
// Host-side argument checks, workspace carve-up, kernel selection, error text.
#include <cstdarg>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace {

thread_local std::string g_last_error;
thread_local int32_t g_last_launches = 0;
thread_local grpo_plan_t g_last_plan = {};

grpo_status_t fail(grpo_status_t st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

grpo_status_t ok(int launches) {
    g_last_error.clear();
    g_last_launches = launches;
    return GRPO_OK;
}

grpo_status_t cuda_fail(cudaError_t e, const char *where, const char *why = nullptr) {
    return fail(GRPO_ERR_CUDA, "%s: %s%s%s", where, cudaGetErrorString(e), why && *why ? " -- " : "",
                why ? why : "");
}

// ---- kernel tracing (grpo_profile_*)
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_pending, g_prof_free;

bool prof_on() {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    return g_prof_on;
}

cudaError_t prof_begin(cudaStream_t s, std::pair<cudaEvent_t, cudaEvent_t> *ev) {
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        if (!g_prof_free.empty()) {
            *ev = g_prof_free.back();
            g_prof_free.pop_back();
        } else {
            ev->first = ev->second = nullptr;
        }
    }
    cudaError_t e = cudaSuccess;
    if (!ev->first) e = cudaEventCreate(&ev->first);
    if (e == cudaSuccess && !ev->second) e = cudaEventCreate(&ev->second);
    if (e == cudaSuccess) e = cudaEventRecord(ev->first, s);
    return e;
}

cudaError_t prof_end(cudaStream_t s, const std::pair<cudaEvent_t, cudaEvent_t> &ev) {
    cudaError_t e = cudaEventRecord(ev.second, s);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_pending.push_back(ev);
    return e;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

// The fields every fused-loss entry shares, and the chunk's scratch carved from the caller's
// workspace in the layout grpo_async_workspace_size sizes (row info, term / logp / flag per
// row, 5 doubles per trajectory).  Returns the first byte past that carve-up.
uint8_t *fill_loss_args(grpo::LossArgs &a, int64_t row_begin, int64_t n_rows, int32_t V,
                        const int64_t *target_ids, const float *logp_behav, const int64_t *cu_seqlens,
                        int32_t N, const int32_t *traj_index, const float *adv, const float *inv_norm,
                        float eps_lo, float eps_hi, float grad_scale, float *logp_out, float *lse_out,
                        float *token_scale_out, double *traj_sum, double *stats, void *workspace) {
    a.V = V;
    a.row_begin = row_begin;
    a.n_rows = n_rows;
    a.target_ids = target_ids;
    a.logp_behav = logp_behav;
    a.cu_seqlens = cu_seqlens;
    a.N = N;
    a.traj_index = traj_index;
    a.adv = adv;
    a.inv_norm = inv_norm;
    a.eps_lo = eps_lo;
    a.eps_hi = eps_hi;
    a.grad_scale = grad_scale;
    a.logp_out = logp_out;
    a.lse_out = lse_out;
    a.scale_out = token_scale_out;
    a.traj_sum = traj_sum;
    a.stats = stats;
    uint8_t *w = reinterpret_cast<uint8_t *>(align256(reinterpret_cast<uintptr_t>(workspace)));
    a.rowinfo = reinterpret_cast<grpo::RowInfo *>(w);
    w += align256((size_t)n_rows * sizeof(grpo::RowInfo));
    a.term_ws = reinterpret_cast<double *>(w);
    w += align256((size_t)n_rows * 8);
    a.logp_ws = reinterpret_cast<float *>(w);
    w += align256((size_t)n_rows * 4);
    a.flag_ws = w;
    w += align256((size_t)n_rows);
    a.part_ws = reinterpret_cast<double *>(w);
    return w + align256((size_t)N * 5 * sizeof(double));
}

}  // namespace

// shared with the host control plane (transfer_queue.cu)
grpo_status_t grpo_internal_fail(grpo_status_t st, const char *msg) { return fail(st, "%s", msg); }

extern "C" {

const char *grpo_last_error(void) { return g_last_error.c_str(); }

grpo_status_t grpo_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = on != 0;
    return ok(0);
}

grpo_status_t grpo_profile_collect(int32_t *n_launches, double *total_ms) {
    if (!n_launches || !total_ms) return fail(GRPO_ERR_INVALID_ARG, "profile_collect: NULL output");
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pend;
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        pend.swap(g_prof_pending);
    }
    double tot = 0.0;
    cudaError_t err = cudaSuccess;
    for (auto &ev : pend) {
        float ms = 0.0f;
        cudaError_t e = cudaEventSynchronize(ev.second);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev.first, ev.second);
        if (e != cudaSuccess && err == cudaSuccess) err = e;
        tot += ms;
    }
    {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof_free.insert(g_prof_free.end(), pend.begin(), pend.end());
    }
    if (err != cudaSuccess) return cuda_fail(err, "profile_collect");
    *n_launches = (int32_t)pend.size();
    *total_ms = tot;
    return ok(0);
}

int32_t grpo_last_launch_count(void) { return g_last_launches; }

grpo_status_t grpo_async_last_plan(grpo_plan_t *out) {
    if (!out) return fail(GRPO_ERR_INVALID_ARG, "last_plan: NULL output");
    *out = g_last_plan;
    return GRPO_OK;
}

const char *grpo_version(void) { return "grpo_async 0.1.0 (sm_100a)"; }

size_t grpo_async_workspace_size(int64_t n_rows, int32_t V, int32_t N) {
    (void)V;
    if (n_rows < 0) n_rows = 0;
    if (N < 0) N = 0;
    return align256((size_t)n_rows * sizeof(grpo::RowInfo)) + align256((size_t)n_rows * 8) +
           align256((size_t)n_rows * 4) + align256((size_t)n_rows) +
           align256((size_t)N * 5 * sizeof(double)) +
           align256(GRPO_VP_MAX_RANKS * sizeof(unsigned long long)) + 256;
}

grpo_status_t grpo_async_validate(const int64_t *version_ids, const int64_t *token_version,
                                  const int64_t *cu_seqlens, const int32_t *group_ids,
                                  const int64_t *target_ids, const float *logp_behav,
                                  int32_t N, int64_t T, int32_t P, int32_t V, int32_t G,
                                  int32_t tbs, int64_t v_theta, int32_t K,
                                  uint32_t *traj_flags, int32_t *group_count,
                                  int32_t *stale_hist, grpo_validate_summary_t *summary,
                                  grpo_stream_t stream) {
    if (!cu_seqlens || !summary || !group_count || !stale_hist)
        return fail(GRPO_ERR_INVALID_ARG, "validate: NULL cu_seqlens/group_count/stale_hist/summary");
    if (N < 0 || T < 0 || P <= 0 || V <= 0 || G <= 0 || K < 0)
        return fail(GRPO_ERR_INVALID_ARG, "validate: bad sizes N=%d T=%lld P=%d V=%d G=%d K=%d", N,
                    (long long)T, P, V, G, K);
    if (N > 0 && (!version_ids || !group_ids || !traj_flags))
        return fail(GRPO_ERR_INVALID_ARG, "validate: NULL version_ids/group_ids/traj_flags");
    if (T > 0 && !target_ids) return fail(GRPO_ERR_INVALID_ARG, "validate: NULL target_ids");
    int launches = 0;
    cudaError_t e = grpo::launch_validate(version_ids, cu_seqlens, group_ids, N, T, P, V, G, tbs,
                                          v_theta, K, token_version, target_ids, logp_behav,
                                          cu_seqlens, nullptr, N, T, traj_flags, group_count,
                                          stale_hist, summary, nullptr, (cudaStream_t)stream,
                                          &launches);
    if (e != cudaSuccess) return cuda_fail(e, "validate");
    return ok(launches);
}

grpo_status_t grpo_async_validate_local(const int64_t *version_ids, const int64_t *cu_seqlens,
                                        const int32_t *group_ids, int32_t N, int64_t T, int32_t P,
                                        int32_t V, int32_t G, int32_t tbs, int64_t v_theta,
                                        int32_t K, const int64_t *local_cu,
                                        const int32_t *traj_index, int32_t n_local,
                                        const int64_t *token_version_local,
                                        const int64_t *target_ids_local,
                                        const float *logp_behav_local, uint32_t *traj_flags,
                                        int32_t *group_count, int32_t *stale_hist,
                                        grpo_validate_summary_t *summary, double *token_counts,
                                        grpo_stream_t stream) {
    if (!cu_seqlens || !summary || !group_count || !stale_hist)
        return fail(GRPO_ERR_INVALID_ARG, "validate_local: NULL cu_seqlens/group_count/stale_hist/summary");
    if (N < 0 || T < 0 || P <= 0 || V <= 0 || G <= 0 || K < 0 || n_local < 0 || n_local > N)
        return fail(GRPO_ERR_INVALID_ARG, "validate_local: bad sizes N=%d T=%lld P=%d V=%d G=%d K=%d n_local=%d",
                    N, (long long)T, P, V, G, K, n_local);
    if (N > 0 && (!version_ids || !group_ids || !traj_flags))
        return fail(GRPO_ERR_INVALID_ARG, "validate_local: NULL version_ids/group_ids/traj_flags");
    if (n_local > 0 && (!local_cu || !traj_index || !target_ids_local))
        return fail(GRPO_ERR_INVALID_ARG, "validate_local: NULL local_cu/traj_index/target_ids_local");
    int launches = 0;
    // the local token arrays are exactly the local packing: no clip beyond local_cu
    cudaError_t e = grpo::launch_validate(version_ids, cu_seqlens, group_ids, N, T, P, V, G, tbs,
                                          v_theta, K, token_version_local, target_ids_local,
                                          logp_behav_local, local_cu, traj_index, n_local,
                                          INT64_MAX, traj_flags, group_count, stale_hist, summary,
                                          token_counts, (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "validate_local");
    return ok(launches);
}

grpo_status_t grpo_async_validate_combine(grpo_validate_summary_t *summary,
                                          const double *token_counts, grpo_stream_t stream) {
    if (!summary || !token_counts) return fail(GRPO_ERR_INVALID_ARG, "validate_combine: NULL argument");
    int launches = 0;
    cudaError_t e = grpo::launch_validate_combine(summary, token_counts, (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "validate_combine");
    return ok(launches);
}

grpo_status_t grpo_async_combine_ranks(const double *gathered, int32_t world, int32_t n,
                                       double *out, grpo_stream_t stream) {
    if (world < 1 || n < 0 || (n > 0 && (!gathered || !out)))
        return fail(GRPO_ERR_INVALID_ARG, "combine_ranks: world=%d n=%d", world, n);
    int launches = 0;
    cudaError_t e = grpo::launch_combine_ranks(gathered, world, n, out, (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "combine_ranks");
    return ok(launches);
}

grpo_status_t grpo_async_validate_sync(const int64_t *version_ids, const int64_t *token_version,
                                       const int64_t *cu_seqlens, const int32_t *group_ids,
                                       const int64_t *target_ids, const float *logp_behav,
                                       int32_t N, int64_t T, int32_t P, int32_t V, int32_t G,
                                       int32_t tbs, int64_t v_theta, int32_t K,
                                       uint32_t *traj_flags, int32_t *group_count,
                                       int32_t *stale_hist, grpo_validate_summary_t *summary,
                                       grpo_validate_summary_t *host_summary,
                                       grpo_stream_t stream) {
    if (!host_summary) return fail(GRPO_ERR_INVALID_ARG, "validate_sync: NULL host_summary");
    grpo_status_t st = grpo_async_validate(version_ids, token_version, cu_seqlens, group_ids,
                                           target_ids, logp_behav, N, T, P, V, G, tbs, v_theta, K,
                                           traj_flags, group_count, stale_hist, summary, stream);
    if (st != GRPO_OK) return st;
    const int launches = g_last_launches;
    cudaError_t e = cudaMemcpyAsync(host_summary, summary, sizeof(grpo_validate_summary_t),
                                    cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "validate_sync");
    if (!host_summary->valid) {
        g_last_launches = launches;
        return fail(GRPO_ERR_VALIDATION,
                    "batch violates constraints: c1_ok=%lld c2_ok=%lld c3_ok=%lld cu_ok=%lld "
                    "stale=%lld future=%lld zero_len=%lld bad_target=%lld bad_logp=%lld",
                    (long long)host_summary->c1_ok, (long long)host_summary->c2_ok,
                    (long long)host_summary->c3_ok, (long long)host_summary->cu_ok,
                    (long long)host_summary->n_stale, (long long)host_summary->n_future,
                    (long long)host_summary->n_zero_len, (long long)host_summary->n_bad_target,
                    (long long)host_summary->n_bad_logp_behav);
    }
    return ok(launches);
}

grpo_status_t grpo_async_advantage(const float *rewards, const int32_t *group_ids,
                                   const int64_t *cu_seqlens, int32_t N, int32_t P,
                                   float std_floor, float *adv, float *inv_norm,
                                   int32_t *group_count, grpo_stream_t stream) {
    if (N < 0 || P <= 0) return fail(GRPO_ERR_INVALID_ARG, "advantage: N=%d P=%d", N, P);
    if (!(std_floor > 0.0f)) return fail(GRPO_ERR_INVALID_ARG, "advantage: std_floor must be > 0");
    if (N > 0 && (!rewards || !group_ids || !cu_seqlens || !adv || !inv_norm))
        return fail(GRPO_ERR_INVALID_ARG, "advantage: NULL pointer");
    int launches = 0;
    cudaError_t e = grpo::launch_advantage(rewards, group_ids, cu_seqlens, N, P, std_floor,
                                           GRPO_NORM_SEQ, 0, nullptr, adv, inv_norm, group_count,
                                           (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "advantage");
    return ok(launches);
}

grpo_status_t grpo_async_group_partials(const float *rewards, const int32_t *group_ids,
                                        const int64_t *cu_seqlens, int32_t N, int32_t P,
                                        const grpo_loss_opts_t *opts, double *part,
                                        grpo_stream_t stream) {
    if (N < 0 || P <= 0) return fail(GRPO_ERR_INVALID_ARG, "group_partials: N=%d P=%d", N, P);
    if (!part || (N > 0 && (!rewards || !group_ids || !cu_seqlens)))
        return fail(GRPO_ERR_INVALID_ARG, "group_partials: NULL pointer");
    int launches = 0;
    cudaError_t e = grpo::launch_group_partials(rewards, group_ids, cu_seqlens, N, P,
                                                opts ? opts->traj_mask : nullptr, part,
                                                (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "group_partials");
    return ok(launches);
}

grpo_status_t grpo_async_group_sq_partials(const float *rewards, const int32_t *group_ids,
                                           int32_t N, int32_t P, const double *glob, double *ss,
                                           grpo_stream_t stream) {
    if (N < 0 || P <= 0) return fail(GRPO_ERR_INVALID_ARG, "group_sq_partials: N=%d P=%d", N, P);
    if (!glob || !ss || (N > 0 && (!rewards || !group_ids)))
        return fail(GRPO_ERR_INVALID_ARG, "group_sq_partials: NULL pointer");
    int launches = 0;
    cudaError_t e = grpo::launch_group_sq(rewards, group_ids, N, P, glob, ss, (cudaStream_t)stream,
                                          &launches);
    if (e != cudaSuccess) return cuda_fail(e, "group_sq_partials");
    return ok(launches);
}

grpo_status_t grpo_async_advantage_from_stats(const float *rewards, const int32_t *group_ids,
                                              const int64_t *cu_seqlens, int32_t N, int32_t P,
                                              float std_floor, const grpo_loss_opts_t *opts,
                                              const double *glob, const double *ss, float *adv,
                                              float *inv_norm, grpo_stream_t stream) {
    if (N < 0 || P <= 0) return fail(GRPO_ERR_INVALID_ARG, "advantage_from_stats: N=%d P=%d", N, P);
    if (!(std_floor > 0.0f)) return fail(GRPO_ERR_INVALID_ARG, "advantage_from_stats: std_floor must be > 0");
    if (opts && opts->norm != GRPO_NORM_SEQ && opts->norm != GRPO_NORM_TOKEN)
        return fail(GRPO_ERR_INVALID_ARG, "advantage_from_stats: norm %d", opts->norm);
    if (!glob || !ss || (N > 0 && (!rewards || !group_ids || !cu_seqlens || !adv || !inv_norm)))
        return fail(GRPO_ERR_INVALID_ARG, "advantage_from_stats: NULL pointer");
    int launches = 0;
    cudaError_t e = grpo::launch_advantage_from_stats(
        rewards, group_ids, cu_seqlens, N, P, std_floor, opts ? opts->norm : GRPO_NORM_SEQ,
        opts && opts->std_unbiased ? 1 : 0, opts ? opts->traj_mask : nullptr, glob, ss, adv, inv_norm,
        (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "advantage_from_stats");
    return ok(launches);
}

grpo_status_t grpo_async_advantage_ex(const float *rewards, const int32_t *group_ids,
                                      const int64_t *cu_seqlens, int32_t N, int32_t P,
                                      float std_floor, const grpo_loss_opts_t *opts, float *adv,
                                      float *inv_norm, int32_t *group_count,
                                      grpo_stream_t stream) {
    if (!opts) return fail(GRPO_ERR_INVALID_ARG, "advantage_ex: NULL opts");
    if (opts->norm != GRPO_NORM_SEQ && opts->norm != GRPO_NORM_TOKEN)
        return fail(GRPO_ERR_INVALID_ARG, "advantage_ex: norm %d", opts->norm);
    if (N < 0 || P <= 0) return fail(GRPO_ERR_INVALID_ARG, "advantage_ex: N=%d P=%d", N, P);
    if (!(std_floor > 0.0f)) return fail(GRPO_ERR_INVALID_ARG, "advantage_ex: std_floor must be > 0");
    if (N > 0 && (!rewards || !group_ids || !cu_seqlens || !adv || !inv_norm))
        return fail(GRPO_ERR_INVALID_ARG, "advantage_ex: NULL pointer");
    int launches = 0;
    cudaError_t e = grpo::launch_advantage(rewards, group_ids, cu_seqlens, N, P, std_floor,
                                           opts->norm, opts->std_unbiased ? 1 : 0,
                                           opts->traj_mask, adv, inv_norm,
                                           group_count, (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "advantage_ex");
    return ok(launches);
}

grpo_status_t grpo_async_loss_fwd(const uint16_t *logits, int64_t row_begin, int64_t n_rows,
                                  int32_t V, int64_t ld, const int64_t *target_ids,
                                  const float *logp_behav, const int64_t *cu_seqlens,
                                  int32_t N, const int32_t *traj_index, const float *adv,
                                  const float *inv_norm, float eps, float grad_scale,
                                  float *logp_out, float *lse_out, float *token_scale_out,
                                  double *traj_sum, double *stats, uint16_t *dlogits,
                                  void *workspace, size_t workspace_bytes,
                                  const grpo_tune_t *tune, grpo_stream_t stream) {
    if (!(eps > 0.0f && eps < 1.0f)) return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: eps not in (0,1)");
    const grpo_loss_opts_t opts = {eps, eps, GRPO_NORM_SEQ, nullptr};
    return grpo_async_loss_fwd_ex(logits, row_begin, n_rows, V, ld, target_ids, logp_behav,
                                  cu_seqlens, N, traj_index, adv, inv_norm, &opts, grad_scale,
                                  logp_out, lse_out, token_scale_out, traj_sum, stats, dlogits,
                                  workspace, workspace_bytes, tune, stream);
}

grpo_status_t grpo_async_loss_fwd_ex(const uint16_t *logits, int64_t row_begin, int64_t n_rows,
                                     int32_t V, int64_t ld, const int64_t *target_ids,
                                     const float *logp_behav, const int64_t *cu_seqlens,
                                     int32_t N, const int32_t *traj_index, const float *adv,
                                     const float *inv_norm, const grpo_loss_opts_t *opts,
                                     float grad_scale, float *logp_out, float *lse_out,
                                     float *token_scale_out, double *traj_sum, double *stats,
                                     uint16_t *dlogits, void *workspace, size_t workspace_bytes,
                                     const grpo_tune_t *tune, grpo_stream_t stream) {
    if (!opts) return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: NULL opts");
    if (n_rows < 0 || N <= 0 || V <= 0 || row_begin < 0)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: n_rows=%lld N=%d V=%d row_begin=%lld",
                    (long long)n_rows, N, V, (long long)row_begin);
    if (!(opts->eps_lo > 0.0f && opts->eps_lo < 1.0f) || !(opts->eps_hi > 0.0f))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: eps_lo not in (0,1) or eps_hi <= 0");
    if (!cu_seqlens || !adv || !inv_norm || !traj_sum || !stats)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: NULL cu_seqlens/adv/inv_norm/traj_sum/stats");
    if (n_rows > 0 && (!logits || !target_ids || !logp_behav))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: NULL logits/target_ids/logp_behav");
    if (ld < V || (ld % 8) != 0)
        return fail(GRPO_ERR_ALIGNMENT, "loss_fwd: ld=%lld must be >= V=%d and a multiple of 8",
                    (long long)ld, V);
    if ((logits && !aligned16(logits)) || (dlogits && !aligned16(dlogits)))
        return fail(GRPO_ERR_ALIGNMENT, "loss_fwd: logits/dlogits must be 16-byte aligned");
    const size_t need = grpo_async_workspace_size(n_rows, V, N);
    if (!workspace || workspace_bytes < need)
        return fail(GRPO_ERR_WORKSPACE, "loss_fwd: workspace %zu B < required %zu B",
                    workspace_bytes, need);
    // kernel 1 (the cluster-resident K3a) is retired: K3c streams the same rows through the
    // bulk-copy ring at 1.7x its throughput
    if (tune && (tune->kernel < 0 || tune->kernel > 3 || tune->kernel == 1))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: tune->kernel %d (0 auto, 2 row-wise, 3 ring)",
                    tune->kernel);
    if (tune && tune->kernel == 3 && (tune->cluster_size < 0 || tune->cluster_size > 2))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: tune->cluster_size %d (kernel 3: 0, 1 or 2)",
                    tune->cluster_size);
    if (tune && tune->kernel == 2 && tune->cluster_size != 0 && tune->cluster_size != 1 &&
        tune->cluster_size != 2 && tune->cluster_size != 4)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: tune->cluster_size %d (kernel 2: 0, 1, 2 or 4)",
                    tune->cluster_size);

    grpo::LossArgs a{};
    fill_loss_args(a, row_begin, n_rows, V, target_ids, logp_behav, cu_seqlens, N, traj_index, adv,
                   inv_norm, opts->eps_lo, opts->eps_hi, grad_scale, logp_out, lse_out, token_scale_out,
                   traj_sum, stats, workspace);
    a.logits = logits;
    a.dlogits = dlogits;
    a.ld = ld;

    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    cudaError_t e = grpo::launch_rowinfo(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "loss_fwd/rowinfo");
    const int kernel = tune ? tune->kernel : 0;
    char why[256] = {0};
    const bool traced = n_rows > 0 && prof_on();
    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    if (traced && (e = prof_begin(s, &ev)) != cudaSuccess) return cuda_fail(e, "loss_fwd/profile");
    // kernel 0 (auto), by row length (plans by V):
    //   V >= 90000          K3c, one CTA per SM, 7 x 32 KB ring slots (V = 152064: 0.96-0.98
    //                       of the measured copy bandwidth vs 0.88 for K3b);
    //   34000 <= V < 90000  K3c, two CTAs per SM of 256 consumer threads, 6 x 16 KB slots
    //                       each (V = 50688: 0.89 vs 0.84; 76032: 0.93 vs 0.87);
    //   below               the row-wise two-pass kernel K3b (V = 30000: 0.81 vs 0.80);
    //   V >= 240000         K3c with every row split over a cluster of two SMs
    //                       (cluster_size 2): at V = 262144 the one-SM row's pass-2
    //                       re-loads miss L2 (DRAM reads 1.185x the row, ncu) and the split
    //                       brings them to 1.005x; with the partner exchange in the epilogue
    //                       warp a launch runs at 0.943 vs 0.844 on one SM; below 240000 the
    //                       one-SM plan wins (the halves' ragged last chunks).
    const bool untuned = !tune || (tune->ctas_per_sm == 0 && tune->stages == 0 && tune->lag == 0 &&
                                   tune->row_cache == 0 && tune->cluster_size == 0 &&
                                   tune->chunk_kb == 0);
    const int n_vec_row = (V + 7) / 8;
    const bool auto_stream = kernel == 0 && untuned && n_vec_row >= 4250;
    grpo_tune_t stream_tune{};
    stream_tune.prefetch = tune ? tune->prefetch : 0;  // K3c look-ahead (kept by the auto plan)
    if (auto_stream && n_vec_row >= 11250) {
        stream_tune.kernel = 3;
        stream_tune.chunk_kb = 32;
        stream_tune.stages = 6;
        // free slots at the end of pass 1: 3, or 1 on long rows (> 10 slots of 32 KB) where
        // the re-read part of every SM's row would crowd L2; rows split over a two-SM cluster
        // from V = 240000 (profiles/r02_split_sweep.jsonl, 65536-row launches, fraction of the
        // measured copy bandwidth: V = 152064 lag 3 0.955 / lag 1 0.946 / split 0.847;
        // 180000 0.933 / 0.951 / 0.859; 200000 0.878 / 0.912 / 0.845; 230000 0.829 / 0.856 /
        // 0.860; 262144 0.805 / 0.844 / 0.943)
        // 7 slots (224 KB of ring), one left free at the end of pass 1: 6 chunks of the row stay
        // resident and pass 2 re-reads the rest from L2 (prod, same-box A/B pairs: 6 / 3 -> 7 / 3
        // +0.5 %, 7 / 3 -> 7 / 2 +0.4 %, and with the bulk-copy stores 7 / 2 -> 7 / 1 +0.5 %;
        // long rows, 65536-row launches: V = 180000 / 200000 / 220000 at 0.961 / 0.933 / 0.893 of
        // the measured copy bandwidth vs 0.951 / 0.922 / 0.896 with 6 / 1;
        // profiles/r02_k3c_variants_t22_t25.txt, r02_plan_sweep.txt)
        stream_tune.stages = 7;
        stream_tune.lag = 1;
        // split rows from V = 240000, the same ring (large, same-box pairs: 6 / 3 -> 7 / 3 +0.9 %,
        // 7 / 3 -> 7 / 1 +0.9 %)
        if (V >= 240000) stream_tune.cluster_size = 2;
        tune = &stream_tune;
    } else if (auto_stream) {
        stream_tune.kernel = 3;
        stream_tune.chunk_kb = 16;
        stream_tune.stages = 6;
        stream_tune.lag = 3;
        stream_tune.row_cache = 2;     // CTAs per SM
        stream_tune.ctas_per_sm = 256;  // consumer threads per CTA
        tune = &stream_tune;
    }
    if ((kernel == 0 && !auto_stream) || kernel == 2) {
        e = grpo::launch_fused_rowwise(a, tune, s, &launches, &g_last_plan);
        // no compiled instantiation for this (threads, vectors, cluster) tune: nothing launched
        if (e == cudaErrorInvalidValue && launches == 1)
            return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: no row-wise kernel for this tune");
        if (e != cudaSuccess) return cuda_fail(e, "loss_fwd/rowwise");
    } else {
        e = grpo::launch_fused_stream(a, tune, s, &launches, &g_last_plan, why, sizeof why);
        // a tune the kernel rejects on the host (its own check, no CUDA call made)
        if (e == cudaErrorInvalidValue && why[0]) return fail(GRPO_ERR_INVALID_ARG, "loss_fwd: %s", why);
        if (e != cudaSuccess) return cuda_fail(e, "loss_fwd/stream", why);
    }
    if (traced && (e = prof_end(s, ev)) != cudaSuccess) return cuda_fail(e, "loss_fwd/profile");
    e = grpo::launch_segment_reduce(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "loss_fwd/segment_reduce");
    return ok(launches);
}

grpo_status_t grpo_async_loss_fwd_vp(const grpo_vp_comm_t *comm, int64_t row_begin,
                                     int64_t n_rows, int32_t V, int64_t ld,
                                     const int64_t *target_ids, const float *logp_behav,
                                     const int64_t *cu_seqlens, int32_t N,
                                     const int32_t *traj_index, const float *adv,
                                     const float *inv_norm, const grpo_loss_opts_t *opts,
                                     float grad_scale, float *logp_out, float *lse_out,
                                     float *token_scale_out, double *traj_sum, double *stats,
                                     void *workspace, size_t workspace_bytes,
                                     grpo_stream_t stream) {
    if (!comm || !opts) return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: NULL comm/opts");
    if (comm->world < 1 || comm->world > GRPO_VP_MAX_RANKS || comm->n_local < 1 ||
        comm->rank_begin < 0 || comm->rank_begin + comm->n_local > comm->world)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: world=%d rank_begin=%d n_local=%d",
                    comm->world, comm->rank_begin, comm->n_local);
    if (comm->shard_cols <= 0 || comm->shard_cols % 8 != 0 ||
        (int64_t)comm->shard_cols * comm->world < V)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: shard_cols=%d (multiple of 8, world*shard_cols >= V=%d)",
                    comm->shard_cols, V);
    if (n_rows < 0 || N <= 0 || V <= 0 || row_begin < 0)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: n_rows/N/V/row_begin");
    if (comm->lag < 0 || comm->lag > 4 || (comm->lag >= 2 && comm->dynamic_rows))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: lag=%d (0..4; 2..4 with static rows only)",
                    comm->lag);
    if (comm->slots < n_rows)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: n_rows=%lld > comm->slots=%lld",
                    (long long)n_rows, (long long)comm->slots);
    if (!(opts->eps_lo > 0.0f && opts->eps_lo < 1.0f) || !(opts->eps_hi > 0.0f))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: eps_lo not in (0,1) or eps_hi <= 0");
    if (!cu_seqlens || !adv || !inv_norm || !traj_sum || !stats)
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: NULL cu_seqlens/adv/inv_norm/traj_sum/stats");
    if (n_rows > 0 && (!target_ids || !logp_behav))
        return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: NULL target_ids/logp_behav");
    if (ld < comm->shard_cols || ld % 8 != 0)
        return fail(GRPO_ERR_ALIGNMENT, "loss_fwd_vp: ld=%lld < shard_cols or not a multiple of 8",
                    (long long)ld);
    for (int q = 0; q < comm->n_local; ++q) {
        if (!comm->logits[q]) return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: NULL logits[%d]", q);
        if (!aligned16(comm->logits[q]) || (comm->dlogits[q] && !aligned16(comm->dlogits[q])))
            return fail(GRPO_ERR_ALIGNMENT, "loss_fwd_vp: logits/dlogits[%d] not 16-byte aligned", q);
    }
    for (int q = 0; q < comm->world; ++q)
        if (!comm->xbuf[q] || !aligned16(comm->xbuf[q]))
            return fail(GRPO_ERR_INVALID_ARG, "loss_fwd_vp: xbuf[%d] NULL or misaligned", q);
    const size_t need = grpo_async_workspace_size(n_rows, V, N);
    if (!workspace || workspace_bytes < need)
        return fail(GRPO_ERR_WORKSPACE, "loss_fwd_vp: workspace %zu B < required %zu B",
                    workspace_bytes, need);
    grpo::LossArgs a{};
    uint8_t *w = fill_loss_args(a, row_begin, n_rows, V, target_ids, logp_behav, cu_seqlens, N, traj_index,
                                adv, inv_norm, opts->eps_lo, opts->eps_hi, grad_scale, logp_out, lse_out,
                                token_scale_out, traj_sum, stats, workspace);
    a.ld = ld;
    unsigned long long *row_ctr = reinterpret_cast<unsigned long long *>(w);
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = cudaMemsetAsync(row_ctr, 0, GRPO_VP_MAX_RANKS * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_fail(e, "loss_fwd_vp/memset");
    e = grpo::launch_rowinfo(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "loss_fwd_vp/rowinfo");
    const bool traced = n_rows > 0 && prof_on();
    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    if (traced && (e = prof_begin(s, &ev)) != cudaSuccess) return cuda_fail(e, "loss_fwd_vp/profile");
    e = grpo::launch_vp(a, comm, row_ctr, s, &launches, &g_last_plan, why, sizeof why);
    if (e != cudaSuccess) return cuda_fail(e, "loss_fwd_vp/vp_kernel", why);
    if (traced && (e = prof_end(s, ev)) != cudaSuccess) return cuda_fail(e, "loss_fwd_vp/profile");
    e = grpo::launch_segment_reduce(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "loss_fwd_vp/segment_reduce");
    return ok(launches);
}

grpo_status_t grpo_async_loss_bwd(const uint16_t *logits, int64_t n_rows, int32_t V, int64_t ld,
                                  const int64_t *target_ids, const float *lse,
                                  const float *token_scale, float grad_scale_mult,
                                  uint16_t *dlogits, grpo_stream_t stream) {
    if (n_rows < 0 || V <= 0) return fail(GRPO_ERR_INVALID_ARG, "loss_bwd: n_rows/V");
    if (n_rows > 0 && (!logits || !target_ids || !lse || !token_scale || !dlogits))
        return fail(GRPO_ERR_INVALID_ARG, "loss_bwd: NULL pointer");
    if (ld < V || (ld % 8) != 0)
        return fail(GRPO_ERR_ALIGNMENT, "loss_bwd: ld=%lld must be >= V and a multiple of 8",
                    (long long)ld);
    if ((logits && !aligned16(logits)) || (dlogits && !aligned16(dlogits)))
        return fail(GRPO_ERR_ALIGNMENT, "loss_bwd: logits/dlogits must be 16-byte aligned");
    int launches = 0;
    cudaError_t e = grpo::launch_loss_bwd(logits, n_rows, V, ld, target_ids, lse, token_scale,
                                          grad_scale_mult, dlogits, (cudaStream_t)stream,
                                          &launches);
    if (e != cudaSuccess) return cuda_fail(e, "loss_bwd");
    return ok(launches);
}

}  // extern "C"

// ---------------------------------------------------------------- LM head (NEXT(2))
namespace {

grpo_status_t lm_check(const char *fn, const uint16_t *hidden, const uint16_t *W, int64_t n_rows,
                       int32_t d, int32_t V) {
    if (n_rows < 0 || V <= 0 || d < 64 || d % 64 != 0 || n_rows > INT32_MAX)
        return fail(GRPO_ERR_INVALID_ARG, "%s: n_rows=%lld d=%d V=%d (d a positive multiple of 64)", fn,
                    (long long)n_rows, d, V);
    if (!W || (n_rows > 0 && !hidden)) return fail(GRPO_ERR_INVALID_ARG, "%s: NULL hidden/W", fn);
    if (!aligned16(W) || (hidden && !aligned16(hidden)))
        return fail(GRPO_ERR_ALIGNMENT, "%s: hidden/W must be 16-byte aligned", fn);
    return GRPO_OK;
}

thread_local int g_lm_cta_group = 2;


}  // namespace

extern "C" {

grpo_status_t grpo_async_lmhead_set_cta_group(int32_t cta_group) {
    if (cta_group != 1 && cta_group != 2)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_set_cta_group: %d (1 or 2)", cta_group);
    g_lm_cta_group = cta_group;
    return ok(0);
}

size_t grpo_async_lmhead_workspace_size(int64_t n_rows, int32_t V, int32_t N) {
    if (n_rows < 0) n_rows = 0;
    if (V < 1) V = 1;
    const size_t split = (size_t)grpo::lmhead_n_split(n_rows, V);
    return grpo_async_workspace_size(n_rows, V, N) + align256(split * (size_t)n_rows * 16) +
           align256((size_t)n_rows * 4) + 256;
}

grpo_status_t grpo_async_lmhead_fwd(const uint16_t *hidden, const uint16_t *W, int64_t row_begin,
                                    int64_t n_rows, int32_t d, int32_t V,
                                    const int64_t *target_ids, const float *logp_behav,
                                    const int64_t *cu_seqlens, int32_t N,
                                    const int32_t *traj_index, const float *adv,
                                    const float *inv_norm, const grpo_loss_opts_t *opts,
                                    float grad_scale, float *logp_out, float *lse_out,
                                    float *token_scale_out, double *traj_sum, double *stats,
                                    void *workspace, size_t workspace_bytes, grpo_stream_t stream) {
    grpo_status_t st = lm_check("lmhead_fwd", hidden, W, n_rows, d, V);
    if (st != GRPO_OK) return st;
    if (!opts) return fail(GRPO_ERR_INVALID_ARG, "lmhead_fwd: NULL opts");
    if (!(opts->eps_lo > 0.0f && opts->eps_lo < 1.0f) || !(opts->eps_hi > 0.0f))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_fwd: eps_lo not in (0,1) or eps_hi <= 0");
    if (N <= 0 || row_begin < 0) return fail(GRPO_ERR_INVALID_ARG, "lmhead_fwd: N/row_begin");
    if (!cu_seqlens || !adv || !inv_norm || !traj_sum || !stats)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_fwd: NULL cu_seqlens/adv/inv_norm/traj_sum/stats");
    if (n_rows > 0 && (!target_ids || !logp_behav))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_fwd: NULL target_ids/logp_behav");
    const size_t need = grpo_async_lmhead_workspace_size(n_rows, V, N);
    if (!workspace || workspace_bytes < need)
        return fail(GRPO_ERR_WORKSPACE, "lmhead_fwd: workspace %zu B < required %zu B", workspace_bytes,
                    need);
    grpo::LossArgs a{};
    fill_loss_args(a, row_begin, n_rows, V, target_ids, logp_behav, cu_seqlens, N, traj_index, adv, inv_norm,
                   opts->eps_lo, opts->eps_hi, grad_scale, logp_out, lse_out, token_scale_out, traj_sum, stats,
                   workspace);
    // past the standard carve-up (grpo_async_workspace_size's layout, incl. its trailing slack)
    uint8_t *w = reinterpret_cast<uint8_t *>(align256(reinterpret_cast<uintptr_t>(workspace))) +
                 grpo_async_workspace_size(n_rows, V, N) - 256;
    const int32_t n_split = grpo::lmhead_n_split(n_rows, V);
    grpo::RowPart *part = reinterpret_cast<grpo::RowPart *>(w);
    w += align256((size_t)n_split * (size_t)n_rows * 16);
    float *zy = reinterpret_cast<float *>(w);
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_rowinfo(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_fwd/rowinfo");
    const bool traced = n_rows > 0 && prof_on();
    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    if (traced && (e = prof_begin(s, &ev)) != cudaSuccess) return cuda_fail(e, "lmhead_fwd/profile");
    e = grpo::launch_lmhead(0, hidden, W, n_rows, d, V, a.rowinfo, part, zy, nullptr, 0, nullptr, nullptr,
                            nullptr, 1.0f, s, &launches, &g_last_plan, why, sizeof why, g_lm_cta_group);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_fwd/tcgen05", why);
    if (traced && (e = prof_end(s, ev)) != cudaSuccess) return cuda_fail(e, "lmhead_fwd/profile");
    e = grpo::launch_lmhead_combine(part, zy, n_split, a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_fwd/combine");
    e = grpo::launch_segment_reduce(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_fwd/segment_reduce");
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_bwd(const uint16_t *hidden, const uint16_t *W, int64_t n_rows,
                                    int32_t d, int32_t V, const int64_t *target_ids,
                                    const float *lse, const float *token_scale,
                                    float grad_scale_mult, uint16_t *dz, int64_t ld_dz,
                                    uint16_t *dhidden, float *dW, grpo_stream_t stream) {
    grpo_status_t st = lm_check("lmhead_bwd", hidden, W, n_rows, d, V);
    if (st != GRPO_OK) return st;
    if (n_rows > 0 && (!target_ids || !lse || !token_scale || !dz))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_bwd: NULL target_ids/lse/token_scale/dz");
    if (ld_dz < V || ld_dz % 8 != 0 || (dz && !aligned16(dz)))
        return fail(GRPO_ERR_ALIGNMENT, "lmhead_bwd: ld_dz=%lld must be >= V, a multiple of 8, dz aligned",
                    (long long)ld_dz);
    if (n_rows == 0) return ok(0);
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_lmhead(1, hidden, W, n_rows, d, V, nullptr, nullptr, nullptr, dz, ld_dz,
                                        target_ids, lse, token_scale, grad_scale_mult, s, &launches,
                                        &g_last_plan, why, sizeof why, g_lm_cta_group);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_bwd/tcgen05", why);
    // dX = dz W and dW += dz^T X on the tensor cores (lmhead_dx.cu gemm_kernel)
    if (dhidden) {
        e = grpo::launch_lmhead_gemm_dx(dz, ld_dz, W, n_rows, d, V, dhidden, 1, s, &launches, why, sizeof why);
        if (e != cudaSuccess) return cuda_fail(e, "lmhead_bwd/dX", why);
    }
    if (dW) {
        e = grpo::launch_lmhead_gemm_dw(dz, ld_dz, hidden, n_rows, d, V, dW, s, &launches, why, sizeof why);
        if (e != cudaSuccess) return cuda_fail(e, "lmhead_bwd/dW", why);
    }
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_tp_partials(const uint16_t *hidden, const uint16_t *W_shard,
                                            int64_t n_rows, int32_t d, int32_t Vs,
                                            int32_t col_offset, const int64_t *target_ids,
                                            float *row_part, void *workspace,
                                            size_t workspace_bytes, grpo_stream_t stream) {
    grpo_status_t st = lm_check("lmhead_tp_partials", hidden, W_shard, n_rows, d, Vs);
    if (st != GRPO_OK) return st;
    if (col_offset < 0) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_partials: col_offset %d", col_offset);
    if (n_rows > 0 && (!target_ids || !row_part))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_partials: NULL target_ids/row_part");
    const size_t need = grpo_async_lmhead_workspace_size(n_rows, Vs, 1);
    if (!workspace || workspace_bytes < need)
        return fail(GRPO_ERR_WORKSPACE, "lmhead_tp_partials: workspace %zu B < required %zu B",
                    workspace_bytes, need);
    if (n_rows == 0) return ok(0);
    uint8_t *w = reinterpret_cast<uint8_t *>(align256(reinterpret_cast<uintptr_t>(workspace)));
    const int32_t n_split = grpo::lmhead_n_split(n_rows, Vs);
    grpo::RowPart *part = reinterpret_cast<grpo::RowPart *>(w);
    w += align256((size_t)n_split * (size_t)n_rows * 16);
    float *zy = reinterpret_cast<float *>(w);
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_lmhead(0, hidden, W_shard, n_rows, d, Vs, nullptr, part, zy, nullptr, 0,
                                        target_ids, nullptr, nullptr, 1.0f, s, &launches, &g_last_plan, why,
                                        sizeof why, g_lm_cta_group, col_offset);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_partials/tcgen05", why);
    e = grpo::launch_lmhead_rowpart(part, zy, n_split, n_rows, target_ids, col_offset, Vs,
                                    reinterpret_cast<float4 *>(row_part), s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_partials/rowpart");
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_tp_fwd(const float *row_parts, int32_t R, int64_t row_begin,
                                       int64_t n_rows, int32_t V, const int64_t *target_ids,
                                       const float *logp_behav, const int64_t *cu_seqlens,
                                       int32_t N, const int32_t *traj_index, const float *adv,
                                       const float *inv_norm, const grpo_loss_opts_t *opts,
                                       float grad_scale, float *logp_out, float *lse_out,
                                       float *token_scale_out, double *traj_sum, double *stats,
                                       void *workspace, size_t workspace_bytes,
                                       grpo_stream_t stream) {
    if (R < 1) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_fwd: R=%d", R);
    if (!opts) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_fwd: NULL opts");
    if (!(opts->eps_lo > 0.0f && opts->eps_lo < 1.0f) || !(opts->eps_hi > 0.0f))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_fwd: eps_lo not in (0,1) or eps_hi <= 0");
    if (n_rows < 0 || N <= 0 || V <= 0 || row_begin < 0)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_fwd: n_rows/N/V/row_begin");
    if (!cu_seqlens || !adv || !inv_norm || !traj_sum || !stats)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_fwd: NULL cu_seqlens/adv/inv_norm/traj_sum/stats");
    if (n_rows > 0 && (!target_ids || !logp_behav || !row_parts))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_fwd: NULL target_ids/logp_behav/row_parts");
    const size_t need = grpo_async_workspace_size(n_rows, V, N);
    if (!workspace || workspace_bytes < need)
        return fail(GRPO_ERR_WORKSPACE, "lmhead_tp_fwd: workspace %zu B < required %zu B", workspace_bytes,
                    need);
    grpo::LossArgs a{};
    fill_loss_args(a, row_begin, n_rows, V, target_ids, logp_behav, cu_seqlens, N, traj_index, adv, inv_norm,
                   opts->eps_lo, opts->eps_hi, grad_scale, logp_out, lse_out, token_scale_out, traj_sum, stats,
                   workspace);
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    cudaError_t e = grpo::launch_rowinfo(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_fwd/rowinfo");
    e = grpo::launch_lmhead_tp_combine(reinterpret_cast<const float4 *>(row_parts), R, a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_fwd/combine");
    e = grpo::launch_segment_reduce(a, s, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_fwd/segment_reduce");
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_tp_bwd(const uint16_t *hidden, const uint16_t *W_shard,
                                       int64_t n_rows, int32_t d, int32_t Vs, int32_t col_offset,
                                       const int64_t *target_ids, const float *lse,
                                       const float *token_scale, float grad_scale_mult,
                                       uint16_t *dz, int64_t ld_dz, float *dhidden_partial,
                                       float *dW_shard, grpo_stream_t stream) {
    grpo_status_t st = lm_check("lmhead_tp_bwd", hidden, W_shard, n_rows, d, Vs);
    if (st != GRPO_OK) return st;
    if (col_offset < 0) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_bwd: col_offset %d", col_offset);
    if (n_rows > 0 && (!target_ids || !lse || !token_scale || !dz))
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_bwd: NULL target_ids/lse/token_scale/dz");
    if (ld_dz < Vs || ld_dz % 8 != 0 || (dz && !aligned16(dz)))
        return fail(GRPO_ERR_ALIGNMENT, "lmhead_tp_bwd: ld_dz=%lld must be >= Vs, a multiple of 8, dz aligned",
                    (long long)ld_dz);
    if (n_rows == 0) return ok(0);
    cudaStream_t s = (cudaStream_t)stream;
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_lmhead(1, hidden, W_shard, n_rows, d, Vs, nullptr, nullptr, nullptr, dz, ld_dz,
                                        target_ids, lse, token_scale, grad_scale_mult, s, &launches,
                                        &g_last_plan, why, sizeof why, g_lm_cta_group, col_offset);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_bwd/tcgen05", why);
    if (dhidden_partial) {  // f32 partial (summed over the ranks by the caller)
        e = grpo::launch_lmhead_gemm_dx(dz, ld_dz, W_shard, n_rows, d, Vs, dhidden_partial, 0, s, &launches, why,
                                        sizeof why);
        if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_bwd/dX", why);
    }
    if (dW_shard) {
        e = grpo::launch_lmhead_gemm_dw(dz, ld_dz, hidden, n_rows, d, Vs, dW_shard, s, &launches, why, sizeof why);
        if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_bwd/dW", why);
    }
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_dw(const uint16_t *hidden, int64_t n_rows, int32_t d, int32_t V,
                                   const uint16_t *dz, int64_t ld_dz, float *dW,
                                   grpo_stream_t stream) {
    if (n_rows < 0 || V <= 0 || d <= 0 || n_rows > INT32_MAX)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_dw: n_rows/V/d");
    if (n_rows > 0 && (!hidden || !dz || !dW)) return fail(GRPO_ERR_INVALID_ARG, "lmhead_dw: NULL pointer");
    if (ld_dz < V || ld_dz % 8 != 0) return fail(GRPO_ERR_ALIGNMENT, "lmhead_dw: ld_dz=%lld", (long long)ld_dz);
    if (n_rows == 0) return ok(0);
    if (d < 64 || d % 64 != 0) return fail(GRPO_ERR_INVALID_ARG, "lmhead_dw: d=%d (a positive multiple of 64)", d);
    if (!aligned16(hidden) || !aligned16(dz) || !aligned16(dW))
        return fail(GRPO_ERR_ALIGNMENT, "lmhead_dw: hidden/dz/dW must be 16-byte aligned");
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_lmhead_gemm_dw(dz, ld_dz, hidden, n_rows, d, V, dW, (cudaStream_t)stream,
                                                &launches, why, sizeof why);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_dw", why);
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W,
                                   int64_t n_rows, int32_t d, int32_t V, void *dhidden,
                                   int32_t out_bf16, grpo_stream_t stream) {
    if (n_rows < 0 || V <= 0 || d < 64 || d % 64 != 0 || n_rows > INT32_MAX)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_dx: n_rows=%lld d=%d V=%d", (long long)n_rows, d, V);
    if (n_rows > 0 && (!W || !dz || !dhidden)) return fail(GRPO_ERR_INVALID_ARG, "lmhead_dx: NULL pointer");
    if (ld_dz < V || ld_dz % 8 != 0 || (dz && !aligned16(dz)) || (W && !aligned16(W)) ||
        (dhidden && !aligned16(dhidden)))
        return fail(GRPO_ERR_ALIGNMENT, "lmhead_dx: ld_dz=%lld (>= V, multiple of 8), 16-byte aligned",
                    (long long)ld_dz);
    if (n_rows == 0) return ok(0);
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_lmhead_gemm_dx(dz, ld_dz, W, n_rows, d, V, dhidden, out_bf16 ? 1 : 0,
                                                (cudaStream_t)stream, &launches, why, sizeof why);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_dx", why);
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_tp_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W_shard,
                                      int64_t n_rows, int32_t d, int32_t Vs, int32_t world,
                                      int32_t rank, float *const *slots, uint32_t epoch,
                                      grpo_stream_t stream) {
    if (n_rows < 0 || n_rows > INT32_MAX || Vs <= 0 || d < 128 || d % 128 != 0)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_dx: n_rows=%lld d=%d Vs=%d (d a multiple of 128)",
                    (long long)n_rows, d, Vs);
    if (world < 1 || world > GRPO_VP_MAX_RANKS || rank < 0 || rank >= world || !slots)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_dx: world=%d rank=%d", world, rank);
    for (int q = 0; q < world; ++q)
        if (!slots[q] || !aligned16(slots[q])) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_dx: slots[%d]", q);
    if (n_rows > 0 && (!dz || !W_shard)) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_dx: NULL dz/W_shard");
    if (ld_dz < Vs || ld_dz % 8 != 0 || (dz && !aligned16(dz)) || (W_shard && !aligned16(W_shard)))
        return fail(GRPO_ERR_ALIGNMENT, "lmhead_tp_dx: ld_dz=%lld (>= Vs, multiple of 8), 16-byte aligned",
                    (long long)ld_dz);
    int launches = 0;
    char why[256] = {0};
    // half epoch % 2 of every slot buffer (the header's double buffering)
    const int64_t half = (int64_t)(epoch & 1u) * world * ((n_rows + world - 1) / world) * d;
    float *sl[GRPO_VP_MAX_RANKS];
    for (int q = 0; q < world; ++q) sl[q] = slots[q] + half;
    cudaError_t e = grpo::launch_lmhead_dx(dz, ld_dz, W_shard, n_rows, d, Vs, world, rank, sl,
                                           (cudaStream_t)stream, &launches, why, sizeof why);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_dx", why);
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_tp_dx_reduce(const float *own_slots, int32_t world, int64_t n_rows,
                                             int32_t d, int32_t rank, void *out, int32_t out_bf16,
                                             uint32_t epoch, grpo_stream_t stream) {
    if (n_rows < 0 || d < 4 || d % 4 != 0 || world < 1 || world > GRPO_VP_MAX_RANKS || rank < 0 || rank >= world)
        return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_dx_reduce: n_rows/d/world/rank");
    if (n_rows > 0 && (!own_slots || !out)) return fail(GRPO_ERR_INVALID_ARG, "lmhead_tp_dx_reduce: NULL");
    int launches = 0;
    const int64_t half = (int64_t)(epoch & 1u) * world * ((n_rows + world - 1) / world) * d;
    cudaError_t e = grpo::launch_lmhead_dx_reduce(own_slots + half, world, n_rows, d, rank, out, out_bf16,
                                                  (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_tp_dx_reduce");
    return ok(launches);
}

grpo_status_t grpo_async_lmhead_logits(const uint16_t *hidden, const uint16_t *W, int64_t n_rows,
                                       int32_t d, int32_t V, uint16_t *out, int64_t ld_out,
                                       grpo_stream_t stream) {
    grpo_status_t st = lm_check("lmhead_logits", hidden, W, n_rows, d, V);
    if (st != GRPO_OK) return st;
    if (n_rows > 0 && !out) return fail(GRPO_ERR_INVALID_ARG, "lmhead_logits: NULL out");
    if (ld_out < V || ld_out % 8 != 0 || (out && !aligned16(out)))
        return fail(GRPO_ERR_ALIGNMENT, "lmhead_logits: ld_out=%lld must be >= V, a multiple of 8",
                    (long long)ld_out);
    int launches = 0;
    char why[256] = {0};
    cudaError_t e = grpo::launch_lmhead(2, hidden, W, n_rows, d, V, nullptr, nullptr, nullptr, out, ld_out,
                                        nullptr, nullptr, nullptr, 1.0f, (cudaStream_t)stream, &launches,
                                        &g_last_plan, why, sizeof why, g_lm_cta_group);
    if (e != cudaSuccess) return cuda_fail(e, "lmhead_logits/tcgen05", why);
    return ok(launches);
}

}  // extern "C"
