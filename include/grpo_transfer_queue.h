/*
 * grpo_transfer_queue.h -- host control plane that produces the batches the
 * async-GRPO loss consumes: the sliding version window and the
 * TransferQueue of DORA (arxiv 2604.26256).
 *
 *   PAPER.md P:175   "Completed trajectories stream into an asynchronous TransferQueue
 *                     equipped with staleness monitoring ... The Trainer consumes the
 *                     number of TBS samples"
 *   PAPER.md P:193-194  "Active versions are managed through a sliding window
 *                     W = {w_j, ..., w_{j-K+1}} of size |W| <= K ... The window slides
 *                     forward only when all trajectories from the oldest version w_{j-K+1}
 *                     have been collected and forwarded to training."
 *   PAPER.md P:46, P:49 (C2: no trajectory abandoned; the batch holds TBS trajectories),
 *   P:39 (C3: v(theta) - v(w_j) <= K), P:7 (a prompt's G responses may span versions).
 * Interface and examples follow SPEC.md transfer_queue; readings where the
 * paper is silent (group-atomic, oldest-first batches; blocking advance) are SPEC's and
 * are listed in DESIGN.md.
 *
 * Host-only, single-threaded per queue object (calls on one object must not overlap).
 * All pointers are HOST pointers.  Status codes are grpo_status_t (grpo_async.h):
 * GRPO_ERR_VALIDATION for protocol violations the paper's constraints forbid (a push
 * for a version outside the window, a non-consecutive window advance, a trajectory
 * that would break C3), GRPO_ERR_INVALID_ARG for bad arguments.  grpo_last_error()
 * holds the text.
 */
#ifndef GRPO_TRANSFER_QUEUE_H
#define GRPO_TRANSFER_QUEUE_H

#include <stdint.h>

#include "grpo_async.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct grpo_tq grpo_tq_t;

/* A queue for groups of G responses and a window of at most K consecutive versions,
 * starting with the single version first_version.  Returns NULL for G < 1 or K < 1. */
grpo_tq_t *grpo_tq_create(int32_t G, int32_t K, int64_t first_version);
void grpo_tq_destroy(grpo_tq_t *q);

/* The RolloutManager dispatched n requests under `version` (in-flight accounting).
 * Errors: GRPO_ERR_VALIDATION if version is not in the window; GRPO_ERR_INVALID_ARG n < 0. */
grpo_status_t grpo_tq_dispatch(grpo_tq_t *q, int64_t version, int32_t n);

/* A completed trajectory arrives (FIFO).  Decrements the version's in-flight count.
 * Errors: GRPO_ERR_VALIDATION if version is not in the window (the window advanced before
 * the version drained: a C3 bug) or nothing of that version is in flight;
 * GRPO_ERR_INVALID_ARG for length <= 0. */
grpo_status_t grpo_tq_push(grpo_tq_t *q, int64_t request_id, int64_t prompt_id, int64_t version,
                           int64_t length, float reward);

/* Form one training batch of exactly tbs trajectories from the oldest complete groups
 * (a group is complete when G of its responses are queued; groups are ordered by the
 * arrival of their first queued response).  On success *formed = 1 and the tbs entries
 * of every output array are written group by group, members in arrival order:
 * group_ids are 0..tbs/G-1 in batch order, prompt_ids the caller's ids.  If fewer than
 * tbs/G groups are complete, *formed = 0 and nothing is consumed.  C3 is checked
 * against v_theta: a member with v_theta - version > K or < 0 is GRPO_ERR_VALIDATION.
 * Errors: GRPO_ERR_INVALID_ARG for tbs <= 0, tbs % G != 0, NULL outputs. */
grpo_status_t grpo_tq_form_batch(grpo_tq_t *q, int32_t tbs, int64_t v_theta, int32_t *formed,
                                 int64_t *request_ids, int64_t *prompt_ids, int32_t *group_ids,
                                 int64_t *version_ids, int64_t *lengths, float *rewards);

/* Slide the window to new_version (must be newest + 1).  While |W| < K the version is
 * appended; at |W| == K the oldest version is evicted only if it has nothing in flight
 * and nothing queued, otherwise *advanced = 0 and the oldest version's residual
 * in-flight / queued counts are returned.
 * Errors: GRPO_ERR_VALIDATION for a non-consecutive version; GRPO_ERR_INVALID_ARG NULLs. */
grpo_status_t grpo_tq_advance(grpo_tq_t *q, int64_t new_version, int32_t *advanced,
                              int64_t *residual_in_flight, int64_t *residual_queued);

/* Snapshot: window [oldest, newest] and counters.  versions_out (nullable) receives the
 * window newest first (capacity K).  Audits: pushed == consumed + queued. */
typedef struct {
    int64_t newest, oldest;     /* window bounds                       */
    int32_t window_size;        /* |W| <= K                            */
    int64_t queued;             /* trajectories waiting in the queue   */
    int64_t in_flight;          /* dispatched, not yet pushed          */
    int64_t pushed, consumed;   /* lifetime counters                   */
    int64_t batches;            /* batches formed                      */
    int64_t max_staleness;      /* max v_theta - version over consumed */
} grpo_tq_stats_t;

grpo_status_t grpo_tq_stats(const grpo_tq_t *q, grpo_tq_stats_t *out, int64_t *versions_out);

#ifdef __cplusplus
}
#endif
#endif /* GRPO_TRANSFER_QUEUE_H */
