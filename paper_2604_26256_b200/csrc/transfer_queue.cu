// transfer_queue.cu -- host control plane: DORA's sliding version
// window and TransferQueue, which hand the trainer
// group-atomic batches of exactly TBS trajectories (C2) whose staleness
// is bounded by K (C3).  Host C++ only; declared in include/grpo_transfer_queue.h.
#include <cstdio>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "grpo_transfer_queue.h"

grpo_status_t grpo_internal_fail(grpo_status_t st, const char *msg);  // api.cu

namespace {

struct Traj {
    int64_t request_id, prompt_id, version, length, seq;
    float reward;
};

struct VersionCount {
    int64_t in_flight = 0, queued = 0;
};

grpo_status_t err(grpo_status_t st, const char *fmt, long long a = 0, long long b = 0) {
    char buf[256];
    snprintf(buf, sizeof buf, fmt, a, b);
    return grpo_internal_fail(st, buf);
}

}  // namespace

struct grpo_tq {
    int32_t G, K;
    int64_t newest, oldest;                         // window [oldest, newest], consecutive
    std::map<int64_t, VersionCount> counts;         // per version in the window
    std::unordered_map<int64_t, std::vector<Traj>> members;  // prompt -> queued responses
    std::map<int64_t, int64_t> order;               // seq of first queued response -> prompt
    std::unordered_map<int64_t, int64_t> first_seq; // prompt -> key in `order`
    int64_t seq = 0, queued = 0, in_flight = 0, pushed = 0, consumed = 0, batches = 0;
    int64_t max_staleness = INT64_MIN;

    bool in_window(int64_t v) const { return v >= oldest && v <= newest; }
};

extern "C" {

grpo_tq_t *grpo_tq_create(int32_t G, int32_t K, int64_t first_version) {
    if (G < 1 || K < 1) return nullptr;
    grpo_tq_t *q = new grpo_tq();
    q->G = G;
    q->K = K;
    q->newest = q->oldest = first_version;
    q->counts[first_version] = VersionCount{};
    return q;
}

void grpo_tq_destroy(grpo_tq_t *q) { delete q; }

grpo_status_t grpo_tq_dispatch(grpo_tq_t *q, int64_t version, int32_t n) {
    if (!q || n < 0) return err(GRPO_ERR_INVALID_ARG, "tq_dispatch: NULL queue or n=%lld", n);
    if (!q->in_window(version))
        return err(GRPO_ERR_VALIDATION, "tq_dispatch: version %lld outside the window (newest %lld)",
                   version, q->newest);
    q->counts[version].in_flight += n;
    q->in_flight += n;
    return GRPO_OK;
}

grpo_status_t grpo_tq_push(grpo_tq_t *q, int64_t request_id, int64_t prompt_id, int64_t version,
                           int64_t length, float reward) {
    if (!q || length <= 0) return err(GRPO_ERR_INVALID_ARG, "tq_push: NULL queue or length=%lld", length);
    if (!q->in_window(version))
        return err(GRPO_ERR_VALIDATION,
                   "tq_push: version %lld is not in the window (oldest %lld): the window advanced "
                   "before the version drained",
                   version, q->oldest);
    VersionCount &c = q->counts[version];
    if (c.in_flight <= 0)
        return err(GRPO_ERR_VALIDATION, "tq_push: no request of version %lld in flight (request %lld)",
                   version, request_id);
    c.in_flight -= 1;
    c.queued += 1;
    q->in_flight -= 1;
    q->queued += 1;
    q->pushed += 1;
    const int64_t s = q->seq++;
    std::vector<Traj> &m = q->members[prompt_id];
    if (m.empty()) {
        q->order[s] = prompt_id;
        q->first_seq[prompt_id] = s;
    }
    m.push_back(Traj{request_id, prompt_id, version, length, s, reward});
    return GRPO_OK;
}

grpo_status_t grpo_tq_form_batch(grpo_tq_t *q, int32_t tbs, int64_t v_theta, int32_t *formed,
                                 int64_t *request_ids, int64_t *prompt_ids, int32_t *group_ids,
                                 int64_t *version_ids, int64_t *lengths, float *rewards) {
    if (!q || !formed || !request_ids || !prompt_ids || !group_ids || !version_ids || !lengths ||
        !rewards)
        return err(GRPO_ERR_INVALID_ARG, "tq_form_batch: NULL argument");
    if (tbs <= 0 || tbs % q->G != 0)
        return err(GRPO_ERR_INVALID_ARG, "tq_form_batch: tbs=%lld must be a positive multiple of G=%lld",
                   tbs, q->G);
    *formed = 0;
    const int32_t need = tbs / q->G;
    std::vector<int64_t> picked;  // prompts, oldest first
    for (const auto &kv : q->order) {
        if ((int32_t)q->members[kv.second].size() >= q->G) picked.push_back(kv.second);
        if ((int32_t)picked.size() == need) break;
    }
    if ((int32_t)picked.size() < need) return GRPO_OK;  // not enough complete groups
    // C3 at formation time: every member within K versions of the trained weights
    for (int64_t p : picked) {
        const std::vector<Traj> &m = q->members[p];
        for (int32_t k = 0; k < q->G; ++k) {
            const int64_t gap = v_theta - m[k].version;
            if (gap < 0 || gap > q->K)
                return err(GRPO_ERR_VALIDATION, "tq_form_batch: C3 violated, staleness %lld > K=%lld",
                           gap, q->K);
        }
    }
    int32_t j = 0;
    for (int32_t gi = 0; gi < need; ++gi) {
        const int64_t p = picked[gi];
        std::vector<Traj> &m = q->members[p];
        for (int32_t k = 0; k < q->G; ++k, ++j) {
            const Traj &t = m[k];
            request_ids[j] = t.request_id;
            prompt_ids[j] = t.prompt_id;
            group_ids[j] = gi;
            version_ids[j] = t.version;
            lengths[j] = t.length;
            rewards[j] = t.reward;
            q->counts[t.version].queued -= 1;
            const int64_t gap = v_theta - t.version;
            if (gap > q->max_staleness) q->max_staleness = gap;
        }
        // extra responses of the same prompt (beyond G) stay queued as a new group
        q->order.erase(q->first_seq[p]);
        m.erase(m.begin(), m.begin() + q->G);
        if (m.empty()) {
            q->members.erase(p);
            q->first_seq.erase(p);
        } else {
            q->order[m.front().seq] = p;
            q->first_seq[p] = m.front().seq;
        }
    }
    q->queued -= tbs;
    q->consumed += tbs;
    q->batches += 1;
    *formed = 1;
    return GRPO_OK;
}

grpo_status_t grpo_tq_advance(grpo_tq_t *q, int64_t new_version, int32_t *advanced,
                              int64_t *residual_in_flight, int64_t *residual_queued) {
    if (!q || !advanced || !residual_in_flight || !residual_queued)
        return err(GRPO_ERR_INVALID_ARG, "tq_advance: NULL argument");
    if (new_version != q->newest + 1)
        return err(GRPO_ERR_VALIDATION, "tq_advance: version %lld is not newest + 1 = %lld",
                   new_version, q->newest + 1);
    *advanced = 0;
    *residual_in_flight = 0;
    *residual_queued = 0;
    if (q->newest - q->oldest + 1 < q->K) {
        q->newest = new_version;
        q->counts[new_version] = VersionCount{};
        *advanced = 1;
        return GRPO_OK;
    }
    const VersionCount &o = q->counts[q->oldest];
    if (o.in_flight != 0 || o.queued != 0) {  // blocked until the oldest version drains
        *residual_in_flight = o.in_flight;
        *residual_queued = o.queued;
        return GRPO_OK;
    }
    q->counts.erase(q->oldest);
    q->oldest += 1;
    q->newest = new_version;
    q->counts[new_version] = VersionCount{};
    *advanced = 1;
    return GRPO_OK;
}

grpo_status_t grpo_tq_stats(const grpo_tq_t *q, grpo_tq_stats_t *out, int64_t *versions_out) {
    if (!q || !out) return err(GRPO_ERR_INVALID_ARG, "tq_stats: NULL argument");
    out->newest = q->newest;
    out->oldest = q->oldest;
    out->window_size = (int32_t)(q->newest - q->oldest + 1);
    out->queued = q->queued;
    out->in_flight = q->in_flight;
    out->pushed = q->pushed;
    out->consumed = q->consumed;
    out->batches = q->batches;
    out->max_staleness = q->batches ? q->max_staleness : 0;
    if (versions_out)
        for (int64_t v = q->newest, k = 0; v >= q->oldest; --v, ++k) versions_out[k] = v;
    return GRPO_OK;
}

}  // extern "C"
