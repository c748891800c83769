/*
 * grpo_async.h -- C ABI of the B200 (sm_100a) hot path of the asynchronous
 * GRPO objective of arxiv 2604.26256 ("DORA"), §3.1.
 *
 *   J_async = E_x [ (1/G) sum_j sum_{i in B_j} (1/L_i) sum_t min(r A, clip_eps(r) A) ]
 *             eq:grpo_async
 *   r_{i,t} = pi_theta(y_t|.) / pi_{w_j}(y_t|.)            eq:ratio_async
 *   C1 one version per trajectory, C2 no trajectory dropped and
 *   N == TBS, C3 v(theta) - v(w_j) <= K
 *   A_i = (R_i - mean) / std over the G responses           eq:group_advantage
 *
 * Conventions shared by every call
 *   - All array pointers are DEVICE pointers unless the parameter name starts
 *     with host_.  The caller owns every buffer; no call allocates device
 *     memory or keeps a pointer after it returns.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t; NULL = the
 *     legacy default stream) and never synchronizes, except *_sync.
 *   - bf16 tensors are passed as uint16_t bit patterns (IEEE bfloat16).
 *   - Status codes: GRPO_OK on success.  Argument errors are detected on the
 *     host before any launch and leave every output untouched.  Data-dependent
 *     violations (C1/C2/C3, bad targets) are never synchronous errors: they
 *     land in the validate outputs; grpo_async_validate_sync converts them
 *     into GRPO_ERR_VALIDATION.  grpo_last_error() returns a thread-local
 *     description of the last non-OK status of the calling thread.
 *   - The loss calls assume validated input (targets in [0, V)); an invalid
 *     target never causes an out-of-bounds access, only a meaningless value.
 *   - Functions are reentrant; distinct streams may run them concurrently on
 *     disjoint outputs.
 * Readings of the paper where it is silent or ambiguous (population std,
 * A = 0 for a group with bitwise-equal rewards, per-prompt weight 1/P,
 * symmetric eps, ties at the clip boundary let the gradient flow, loss = -J)
 * are listed in DESIGN.md "Readings" (Z1-Z20).
 */
#ifndef GRPO_ASYNC_H
#define GRPO_ASYNC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *grpo_stream_t; /* a cudaStream_t */

typedef enum {
    GRPO_OK = 0,
    GRPO_ERR_VALIDATION = 1,  /* C1/C2/C3 or structural violation (validate_sync only)       */
    GRPO_ERR_INVALID_ARG = 2, /* NULL required pointer, N <= 0, eps not in (0,1), K < 0, ...  */
    GRPO_ERR_ALIGNMENT = 3,   /* logits/dlogits not 16-byte aligned, or ld % 8 != 0, ld < V   */
    GRPO_ERR_WORKSPACE = 4,   /* workspace NULL or smaller than grpo_async_workspace_size()   */
    GRPO_ERR_CUDA = 5         /* a CUDA runtime error (text in grpo_last_error)               */
} grpo_status_t;

/* Per-trajectory validation flags (traj_flags bits). */
#define GRPO_FLAG_STALE          (1u << 0) /* v_theta - v_i > K              (C3)  */
#define GRPO_FLAG_FUTURE         (1u << 1) /* v_theta - v_i < 0              (C3 reading) */
#define GRPO_FLAG_ZERO_LEN       (1u << 2) /* L_i = cu[i+1] - cu[i] <= 0                  */
#define GRPO_FLAG_BAD_GROUP_ID   (1u << 3) /* group id not in [0, P)                      */
#define GRPO_FLAG_GROUP_SIZE     (1u << 4) /* its group does not have exactly G members (C2) */
#define GRPO_FLAG_C1_MIXED       (1u << 5) /* a token version differs from v_i   (C1) */
#define GRPO_FLAG_BAD_TARGET     (1u << 6) /* a target id not in [0, V)                   */
#define GRPO_FLAG_BAD_LOGP_BEHAV (1u << 7) /* a behaviour log-prob not finite or > 0      */

/* Validation summary (all int64; mirrors SPEC metrics.audit S:619-625). */
typedef struct {
    int64_t n_traj;              /* N                                                   */
    int64_t n_tokens;            /* cu[N]                                               */
    int64_t n_stale, n_future, n_zero_len, n_bad_group_id, n_group_size,
            n_c1_mixed, n_bad_target, n_bad_logp_behav; /* trajectories per flag      */
    int64_t n_groups_wrong_size; /* #{p : count_p != G}                                 */
    int64_t c2_dropped;          /* sum_p max(0, G - count_p)                           */
    int64_t max_staleness;       /* max_i (v_theta - v_i)   (0 when N == 0)             */
    int64_t min_staleness;       /* min_i (v_theta - v_i)                               */
    int64_t cu_ok;               /* cu[0] == 0, cu non-decreasing, cu[N] == T           */
    int64_t tbs_ok;              /* N == tbs                                            */
    int64_t c1_ok, c2_ok, c3_ok; /* the paper's constraints (C2: tbs_ok, all groups G,   */
                                 /*  all group ids valid; C3: no STALE/FUTURE)          */
    int64_t valid;               /* all of the above and no ZERO_LEN/BAD_TARGET/BAD_LOGP */
} grpo_validate_summary_t;

/* Index of the per-chunk statistics accumulated by grpo_async_loss_fwd into stats[]. */
enum {
    GRPO_STAT_J = 0,         /* sum over rows of inv_norm_i * term_t (this chunk's part of J) */
    GRPO_STAT_ROWS = 1,      /* rows processed                                                */
    GRPO_STAT_CLIPPED = 2,   /* rows whose clipped branch binds: (A>0, r>1+eps) or (A<0, r<1-eps) */
    GRPO_STAT_ACTIVE = 3,    /* rows with nonzero gradient: not clipped and A != 0            */
    GRPO_STAT_ABS = 4,       /* sum of inv_norm_i * |term_t| (L1 mass of J's summands)        */
    GRPO_STAT_LOGP = 5,      /* sum of log pi_theta(y_t) (diagnostic)                         */
    GRPO_NUM_STATS = 6
};

/* Loss options of the DAPO setting the paper trains with ("we follow the
 * setting of DAPO").  grpo_async_loss_fwd / grpo_async_advantage
 * are the paper's equation as written (eps_lo = eps_hi = eps, GRPO_NORM_SEQ, no mask). */
enum {
    GRPO_NORM_SEQ = 0,   /* eq:grpo_async: 1/L_i per trajectory, 1/G_p per group, 1/P per prompt */
    GRPO_NORM_TOKEN = 1  /* DAPO token-level: 1 / (sum of L_i over kept trajectories)            */
};
typedef struct {
    float eps_lo;              /* clip below at 1 - eps_lo, in (0, 1)                             */
    float eps_hi;              /* clip above at 1 + eps_hi, > 0 ("clip-higher": eps_hi > eps_lo)  */
    int32_t norm;              /* GRPO_NORM_SEQ or GRPO_NORM_TOKEN                                */
    const uint8_t *traj_mask;  /* device uint8[N] or NULL: 0 drops trajectory i from the loss and */
                               /* from the token-mean denominator (overlong filtering, masking of */
                               /* C1-violating partial rollouts); group statistics keep    */
                               /* every member                                                    */
    int32_t std_unbiased;      /* 0: population std (eq:group_advantage as read, Z1); 1: sample   */
                               /* std with n - 1 (verl-style); a one-member group has A = 0      */
} grpo_loss_opts_t;

/* Optional tuning of the fused loss kernel (NULL = automatic). */
typedef struct {
    int32_t kernel;        /* 0 auto: 2 for V < 34000; 3 with 2 CTAs x 6 x 16 KB up to 90000, */
                           /* else 3 with 1 CTA x 7 x 32 KB slots per SM, rows split over 2 */
                           /* SMs from V = 240000 (an explicit                               */
                           /* tune with other fields set is never redirected); 1 cluster-    */
                           /* resident; 2 row-wise; 3 one row per SM through a bulk-copy ring */
    int32_t cluster_size;  /* 0 auto, else 1,2,4,8,16: CTAs sharing one row (kernel 1);      */
                           /* kernel 3: 2 = each row split over a 2-CTA cluster (the auto  */
                           /* plan for V >= 240000; 512 threads, 1 CTA/SM, 16/32 KB slots, */
                           /* V >= 16384, else GRPO_ERR_CUDA)                               */
    int32_t ctas_per_sm;   /* 0 auto, else 1..4 (kernel 1); 1,2,4,8 (kernel 2: 1024/512/256/256 threads); */
                           /* kernel 3: 256 consumer threads (default 512)                     */
    int32_t stages;        /* 0 auto, else lag+2..8 shared-memory row stages per CTA (kernel 1); */
                           /* kernel 2: 4, 8 or 16 vectors in flight per thread; kernel 3:  */
                           /* ring slots (0 = 13 of 16 KB, 6 of 32 KB; at most 14 / 7, 224 KB) */
    int32_t lag;           /* 0 auto, else 1..2: rows between a row's reduction and its       */
                           /* backward, hiding the cluster exchange (kernel 1); kernel 3:    */
                           /* ring slots left free at the end of pass 1 (0 = 3)              */
    int32_t prefetch;      /* kernel 2: 1 = TMA-prefetch each CTA's next row into L2;        */
                           /* kernel 3: chunks of the next row streamed before a row's pass */
                           /* 2, hiding its epilogue (0 = 1, -1 = none; capped at stages -  */
                           /* resident)                                                      */
    int32_t row_cache;     /* kernel 2: leading vectors per thread of each row kept in shared */
                           /* memory for the second pass (0 auto = 160 KB per SM, -1 none); */
                           /* kernel 3: CTAs per SM, 1 (default) or 2                        */
    int32_t chunk_kb;      /* kernel 3: ring slot size in KB: 16 (default), 24, 32, 48 or 64   */
} grpo_tune_t;

/*
 * grpo_async_validate -- bit-exact integer checks of C1, C2, C3 and batch
 * structure.
 *   version_ids   int64[N]  behaviour version v(w_j) of trajectory i
 *   token_version int64[T]  per-token behaviour version, or NULL (C1 check skipped)
 *   cu_seqlens    int64[N+1] packed row offsets: trajectory i owns rows [cu[i], cu[i+1])
 *   group_ids     int32[N]  prompt index of trajectory i, any order
 *   target_ids    int64[T]  sampled token y_t
 *   logp_behav    float[T]  log pi_{w_j}(y_t), or NULL (check skipped)
 *   N, T, P, V, G, tbs      sizes; v_theta = v(theta); K = staleness bound
 * Outputs (device): traj_flags uint32[N], group_count int32[P],
 *   stale_hist int32[P*(K+1)] (|B_j| per prompt p and gap v_theta-v in [0,K]),
 *   summary (one grpo_validate_summary_t).
 * Errors: GRPO_ERR_INVALID_ARG for NULL required pointers, N < 0, T < 0, P <= 0,
 *   V <= 0, G <= 0, K < 0.
 */
grpo_status_t grpo_async_validate(const int64_t *version_ids, const int64_t *token_version,
                                  const int64_t *cu_seqlens, const int32_t *group_ids,
                                  const int64_t *target_ids, const float *logp_behav,
                                  int32_t N, int64_t T, int32_t P, int32_t V, int32_t G,
                                  int32_t tbs, int64_t v_theta, int32_t K,
                                  uint32_t *traj_flags, int32_t *group_count,
                                  int32_t *stale_hist, grpo_validate_summary_t *summary,
                                  grpo_stream_t stream);

/* Same, then synchronizes `stream` and copies the summary to host_summary.
 * Returns GRPO_ERR_VALIDATION when host_summary->valid == 0. */
grpo_status_t grpo_async_validate_sync(const int64_t *version_ids, const int64_t *token_version,
                                       const int64_t *cu_seqlens, const int32_t *group_ids,
                                       const int64_t *target_ids, const float *logp_behav,
                                       int32_t N, int64_t T, int32_t P, int32_t V, int32_t G,
                                       int32_t tbs, int64_t v_theta, int32_t K,
                                       uint32_t *traj_flags, int32_t *group_count,
                                       int32_t *stale_hist, grpo_validate_summary_t *summary,
                                       grpo_validate_summary_t *host_summary,
                                       grpo_stream_t stream);

/*
 * grpo_async_validate_local -- grpo_async_validate for one rank of a trajectory-sharded batch
 * (the paper's trainer spreads one batch over the GPUs of a node): the
 * trajectory-level checks (C3 gap P:39, C2 group counts and TBS P:46-49, zero length, group
 * ids, the |B_j| histogram) run over all N trajectories of the replicated metadata, the
 * token-level checks (C1 P:44, target range, behaviour log-probs) only over this rank's
 * trajectories, from its own token arrays:
 *   version_ids int64[N], cu_seqlens int64[N+1] (global packing), group_ids int32[N];
 *   local_cu int64[n_local+1]: local trajectory j owns rows [local_cu[j], local_cu[j+1]) of
 *   the local token arrays and is global trajectory traj_index[j] (int32[n_local]);
 *   token_version_local (nullable), target_ids_local, logp_behav_local (nullable): local rows.
 * Outputs as grpo_async_validate, except that the summary's token-level counts
 * (n_c1_mixed, n_bad_target, n_bad_logp_behav) and the verdicts that use them (c1_ok,
 * valid) cover this rank's trajectories, and traj_flags carries token bits only for them.
 * token_counts (double[3], nullable) receives those three counts as exact doubles, to be
 * summed over the ranks with the loss partials; grpo_async_validate_combine then writes the
 * sums into the summary and recomputes c1_ok / valid -- the whole batch's verdict, identical
 * on every rank.  n_local = N with traj_index = identity and local_cu = cu_seqlens is
 * grpo_async_validate.  All pointers are device pointers; stream-ordered, no sync.
 * Errors: GRPO_ERR_INVALID_ARG (NULL required pointers, bad sizes, n_local > N).
 */
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
                                        grpo_stream_t stream);
grpo_status_t grpo_async_validate_combine(grpo_validate_summary_t *summary,
                                          const double *token_counts, grpo_stream_t stream);

/*
 * grpo_async_combine_ranks -- the data-parallel step's one exchange: after the
 * caller all-gathers every rank's packed fp64 partials (the stats of grpo_async_loss_fwd,
 * i.e. this rank's share of J = sum_t inv_norm_i term_t of eq:grpo_async P:9-26, plus the
 * token-level validation counts) into gathered[world][n] in rank order,
 *   out[k] = gathered[0][k] + gathered[1][k] + ... + gathered[world-1][k]
 * summed in that order -- the same bits on every rank and in every run (a collective's
 * SUM has no fixed order).  Device pointers; out may not alias gathered.
 * Errors: GRPO_ERR_INVALID_ARG (world < 1, n < 0, NULL pointers).
 */
grpo_status_t grpo_async_combine_ranks(const double *gathered, int32_t world, int32_t n,
                                       double *out, grpo_stream_t stream);

/*
 * grpo_async_advantage -- group-relative advantages, eq:group_advantage.
 *   rewards float[N], group_ids int32[N] (any order), cu_seqlens int64[N+1].
 *   For each group p: fp64 mean and population std over its members in
 *   ascending i; A_i = (R_i - mean) / max(std, std_floor), and A_i = 0 exactly
 *   when all rewards of the group are bitwise equal (Z1, Z2).
 *   inv_norm_i = 1 / (P * count_p * L_i): the weight of one token of i in J
 *   (eq:grpo_async's 1/L_i, 1/G and the mean over prompts, Z5, Z6).
 * Outputs: adv float[N], inv_norm float[N], group_count int32[P] (nullable).
 * A trajectory with an invalid group id or L_i <= 0 gets A = 0 and inv_norm = 0.
 * Errors: GRPO_ERR_INVALID_ARG for NULL pointers, N < 0, P <= 0, std_floor <= 0.
 */
grpo_status_t grpo_async_advantage(const float *rewards, const int32_t *group_ids,
                                   const int64_t *cu_seqlens, int32_t N, int32_t P,
                                   float std_floor, float *adv, float *inv_norm,
                                   int32_t *group_count, grpo_stream_t stream);

/*
 * grpo_async_advantage_ex -- grpo_async_advantage with grpo_loss_opts_t:
 *   inv_norm_i = 1/(P * count_p * L_i) (GRPO_NORM_SEQ) or 1/sum_kept L (GRPO_NORM_TOKEN),
 *   and 0 for trajectories the mask drops; opts->std_unbiased selects the sample std
 *   (n - 1) for A_i.  opts->eps_* are not used here.
 * Errors: as grpo_async_advantage, plus GRPO_ERR_INVALID_ARG for NULL opts or a bad norm.
 */
grpo_status_t grpo_async_advantage_ex(const float *rewards, const int32_t *group_ids,
                                      const int64_t *cu_seqlens, int32_t N, int32_t P,
                                      float std_floor, const grpo_loss_opts_t *opts, float *adv,
                                      float *inv_norm, int32_t *group_count,
                                      grpo_stream_t stream);

/*
 * Sharded rewards (the north_star "group reward statistics" all-reduce): when a
 * rank holds only its own trajectories' rewards, eq:group_advantage needs the
 * group statistics of all ranks.  Three calls around two all-reduces of the caller's
 * collective library (NCCL):
 *   grpo_async_group_partials   part[P*4 + 1] (double) <- per group p of the local
 *       trajectories: part[4p] = count, part[4p+1] = sum of rewards (ascending local index),
 *       part[4p+2] = max and part[4p+3] = -min of the rewards' float32 bit patterns (as
 *       exact doubles), and part[4P] = the local kept tokens (token-mean normalisation).
 *       Combine entries 4p, 4p+1 and 4P with SUM and 4p+2, 4p+3 with MAX over ranks.
 *   grpo_async_group_sq_partials  ss[P] (double) <- sum over local members of (R - mean)^2
 *       with mean = glob[4p+1] / glob[4p] from the combined partials; combine with SUM.
 *   grpo_async_advantage_from_stats  A_i and inv_norm_i of the local trajectories from the
 *       combined partials: A_i = 0 when the group's rewards are bitwise equal (max == min),
 *       else (R_i - mean) / max(std, std_floor) (population std, or n - 1 with
 *       opts->std_unbiased); inv_norm_i = 1/(P * count_p * L_i) or 1/T_kept (opts->norm)
 *       and 0 for masked / invalid trajectories -- the same readings as grpo_async_advantage_ex.
 * The sums are fp64; across ranks they are added in the collective's order, so A_i agrees
 * with the single-rank result to fp64 rounding (bit-identical for rewards whose partial sums
 * are exact, e.g. 0/1 rewards).  N may be 0 on a rank.  All pointers are device pointers.
 * Errors: GRPO_ERR_INVALID_ARG (NULL pointers, P <= 0, N < 0, std_floor <= 0, bad opts),
 * GRPO_ERR_CUDA.
 */
grpo_status_t grpo_async_group_partials(const float *rewards, const int32_t *group_ids,
                                        const int64_t *cu_seqlens, int32_t N, int32_t P,
                                        const grpo_loss_opts_t *opts, double *part,
                                        grpo_stream_t stream);
grpo_status_t grpo_async_group_sq_partials(const float *rewards, const int32_t *group_ids,
                                           int32_t N, int32_t P, const double *glob, double *ss,
                                           grpo_stream_t stream);
grpo_status_t grpo_async_advantage_from_stats(const float *rewards, const int32_t *group_ids,
                                              const int64_t *cu_seqlens, int32_t N, int32_t P,
                                              float std_floor, const grpo_loss_opts_t *opts,
                                              const double *glob, const double *ss, float *adv,
                                              float *inv_norm, grpo_stream_t stream);

/*
 * grpo_async_loss_fwd -- fused log-softmax + target gather + ratio + clip +
 * min + segmented mean, and (if dlogits != NULL) the backward in the same pass:
 *   log pi_theta(y_t | .) = z_{t,y_t} - logsumexp_v z_{t,v}   (P:136 pi(y|x) = prod_t pi(y_t|.),
 *                                                             P:32-33 the token probabilities)
 *   r_t = exp(log pi_theta - log pi_{w_j})                   (eq:ratio_async)
 *   term_t = min(r_t A_i, clip_eps(r_t) A_i)                  (eq:grpo_async P:19-22, clip P:151)
 *   traj_sum_i = sum_t term_t;  J = sum_i inv_norm_i traj_sum_i (the 1/L_i, 1/G and 1/P of
 *                                                             eq:grpo_async P:14-18, folded)
 *   dlogits = d(-J)/dz = s_t (softmax(z_t) - onehot(y_t))     (the chain rule of the above;
 *                                                             DESIGN.md Z19: the paper
 *                                                             maximises J, the loss is -J)
 * The chunk is rows [row_begin, row_begin + n_rows) of this rank's packing.
 *   logits      bf16[n_rows, ld] row k scores target_ids[k] (caller-shifted,
 *               response tokens only); ld >= V, ld % 8 == 0, 16-byte aligned.
 *   target_ids  int64[n_rows], logp_behav float[n_rows]   (chunk-local, row k)
 *   cu_seqlens  int64[N+1] over this rank's N trajectories (row_begin is an
 *               offset into this packing; a trajectory may straddle chunks).
 *   traj_index  int32[N] or NULL: trajectory i of this packing reads
 *               adv[traj_index[i]] / inv_norm[traj_index[i]] (NULL = identity),
 *               so replicated whole-batch advantages can feed a shard.
 *   adv, inv_norm  float[*] from grpo_async_advantage.
 *   eps in (0,1); grad_scale multiplies the gradient (1 = d(-J)/dz).
 * Outputs (each nullable): logp_out, lse_out, token_scale_out float[n_rows]
 *   (token_scale s_t = grad_scale * inv_norm * A * r * [not clipped]);
 *   traj_sum double[N]: += sum of term_t over this chunk's rows of i;
 *   stats double[GRPO_NUM_STATS]: += this chunk's GRPO_STAT_* values;
 *   dlogits bf16[n_rows, ld]: d(-J)/dz = s_t (softmax - onehot(y_t)), written
 *   once per element in [0, V) (padding columns untouched).  dlogits may
 *   equal logits (in place).
 * workspace: device scratch of grpo_async_workspace_size(n_rows, V, N) bytes.
 * tune: NULL or kernel selection (grpo_tune_t).
 * Errors: GRPO_ERR_INVALID_ARG (NULL logits/targets/logp_behav/cu/adv/inv_norm/
 *   traj_sum/stats, n_rows < 0, N <= 0, V <= 0, eps not in (0,1)),
 *   GRPO_ERR_ALIGNMENT, GRPO_ERR_WORKSPACE, GRPO_ERR_CUDA.
 */
grpo_status_t grpo_async_loss_fwd(const uint16_t *logits, int64_t row_begin, int64_t n_rows,
                                  int32_t V, int64_t ld, const int64_t *target_ids,
                                  const float *logp_behav, const int64_t *cu_seqlens,
                                  int32_t N, const int32_t *traj_index, const float *adv,
                                  const float *inv_norm, float eps, float grad_scale,
                                  float *logp_out, float *lse_out, float *token_scale_out,
                                  double *traj_sum, double *stats, uint16_t *dlogits,
                                  void *workspace, size_t workspace_bytes,
                                  const grpo_tune_t *tune, grpo_stream_t stream);

/*
 * grpo_async_loss_fwd_ex -- grpo_async_loss_fwd with the clip range [1 - opts->eps_lo,
 * 1 + opts->eps_hi] (the weights come from grpo_async_advantage_ex).  Same arguments
 * otherwise; eps is replaced by opts.
 * Errors: as grpo_async_loss_fwd, plus GRPO_ERR_INVALID_ARG for NULL opts, eps_lo not in
 * (0,1) or eps_hi <= 0.
 */
grpo_status_t grpo_async_loss_fwd_ex(const uint16_t *logits, int64_t row_begin, int64_t n_rows,
                                     int32_t V, int64_t ld, const int64_t *target_ids,
                                     const float *logp_behav, const int64_t *cu_seqlens,
                                     int32_t N, const int32_t *traj_index, const float *adv,
                                     const float *inv_norm, const grpo_loss_opts_t *opts,
                                     float grad_scale, float *logp_out, float *lse_out,
                                     float *token_scale_out, double *traj_sum, double *stats,
                                     uint16_t *dlogits, void *workspace, size_t workspace_bytes,
                                     const grpo_tune_t *tune, grpo_stream_t stream);

/*
 * grpo_async_loss_fwd_vp -- the fused loss for vocabulary-parallel logits (
 * Megatron-style tensor parallelism of the LM head): rank q of a group of R
 * GPUs holds the columns [q*shard_cols, (q+1)*shard_cols) of every row of the chunk.
 * The per-row logsumexp needs all R shards: the kernel exchanges one 32-byte partial
 * per row and rank through peer memory (NVLink P2P stores of 64-bit words tagged with
 * the call's epoch) inside the loss kernel, then writes this rank's slice of dlogits.
 * With lag 0 and static rows, shards of >= 90000 columns run the streamed ring kernel
 * (plan kernel 8), shards of 16384..89999 columns the ring kernel with pass 2 delayed by
 * one row (plan kernel 9), narrower shards or lag 1 / dynamic rows the row-wise kernel
 * (plan kernel 7); lag 2..4 forces kernel 9 with pass 2 delayed by lag - 1 rows; same
 * results.  Every
 * rank computes identical per-row outputs, traj_sum and stats (no further reduction).
 * comm describes the group (host struct of device pointers):
 *   world R <= GRPO_VP_MAX_RANKS; the call computes ranks [rank_begin, rank_begin+n_local)
 *   (n_local = 1 on a multi-GPU run; n_local = R when one GPU runs the whole group as a
 *   cooperative grid); shard_cols % 8 == 0; logits[i] / dlogits[i] bf16 [n_rows, ld] of
 *   local rank i (ld >= shard_cols, 16-byte aligned; dlogits may be NULL = forward only);
 *   xbuf[q] >= 2*slots*world*32 bytes of EVERY rank q, mapped into this process (peer
 *   pointers), zero-initialised once; slots >= n_rows; epoch = number of earlier calls
 *   on these buffers (the same on every rank): call e uses the half e % 2 and tags its
 *   words with e + 1, so a fast rank's next call never overwrites a partial a slow rank
 *   has not yet read and stale words are never mistaken for new ones.  All ranks must
 *   call with the same arguments except the pointers they own; a rank whose peers never
 *   arrive traps (GRPO_ERR_CUDA, context lost).
 * Other arguments as grpo_async_loss_fwd_ex (per-row outputs written by local rank 0).
 * Errors: GRPO_ERR_INVALID_ARG (bad comm, NULL pointers), GRPO_ERR_ALIGNMENT,
 *   GRPO_ERR_WORKSPACE, GRPO_ERR_CUDA.
 */
#define GRPO_VP_MAX_RANKS 8
typedef struct {
    int32_t world;
    int32_t rank_begin;
    int32_t n_local;
    int32_t shard_cols;
    int64_t slots;
    const uint16_t *logits[GRPO_VP_MAX_RANKS];
    uint16_t *dlogits[GRPO_VP_MAX_RANKS];
    void *xbuf[GRPO_VP_MAX_RANKS];
    uint32_t epoch;
    int32_t lag;          /* 0 (default): the plan by shard width (see above);              */
                          /* 1: row-wise, wait after pass 1 of the next row (same results);  */
                          /* 2..4: the streamed ring kernel with pass 2 of row k run after   */
                          /* pass 1 of row k + lag - 1, the row re-read from L2 (plan kernel */
                          /* 9; static rows only; same results); else GRPO_ERR_INVALID_ARG   */
    int32_t dynamic_rows; /* 0 (default): CTA g takes rows g, g + grid, ...; 1: CTAs take     */
                          /* rows in the order they ask for them (same results)             */
} grpo_vp_comm_t;

grpo_status_t grpo_async_loss_fwd_vp(const grpo_vp_comm_t *comm, int64_t row_begin,
                                     int64_t n_rows, int32_t V, int64_t ld,
                                     const int64_t *target_ids, const float *logp_behav,
                                     const int64_t *cu_seqlens, int32_t N,
                                     const int32_t *traj_index, const float *adv,
                                     const float *inv_norm, const grpo_loss_opts_t *opts,
                                     float grad_scale, float *logp_out, float *lse_out,
                                     float *token_scale_out, double *traj_sum, double *stats,
                                     void *workspace, size_t workspace_bytes,
                                     grpo_stream_t stream);

/*
 * grpo_async_loss_bwd -- unfused backward: one streaming pass that re-reads
 * the logits and writes dlogits = grad_scale_mult * s_t * (exp(z - lse_t) - onehot(y_t))
 * from the lse and token_scale saved by grpo_async_loss_fwd: the gradient of -J of
 * eq:grpo_async with respect to the logits through log pi_theta(y_t) (P:32-33,
 * P:136); s_t = 0 for clipped tokens (the clipped branch of the min carries no
 * gradient) and zero advantages (Z19, Z10).
 *   logits, dlogits bf16[n_rows, ld] (may alias), target_ids int64[n_rows],
 *   lse, token_scale float[n_rows].
 * Errors: GRPO_ERR_INVALID_ARG, GRPO_ERR_ALIGNMENT, GRPO_ERR_CUDA.
 */
grpo_status_t grpo_async_loss_bwd(const uint16_t *logits, int64_t n_rows, int32_t V, int64_t ld,
                                  const int64_t *target_ids, const float *lse,
                                  const float *token_scale, float grad_scale_mult,
                                  uint16_t *dlogits, grpo_stream_t stream);

/*
 * ---- LM-head-fused loss (the step before the path: the trainer's LM
 * head, Megatron-LM).  z = X W^T is computed on the tensor cores (tcgen05.mma,
 * bf16 x bf16 -> f32 in TMEM) and consumed tile by tile in the kernel's epilogue, so the
 * [n_rows, V] logits never reach HBM (Cut-Cross-Entropy style).
 *   hidden  bf16 [n_rows, d] row-major (the final hidden states of the chunk's rows)
 *   W       bf16 [V, d] row-major (the LM-head weight, vocabulary-major)
 *   d % 64 == 0, 64 <= d; both 16-byte aligned; V >= 1.
 *
 * grpo_async_lmhead_fwd -- as grpo_async_loss_fwd_ex but with logits = hidden W^T:
 *   per-row logp / lse / token_scale, per-trajectory term sums and the stats, with the
 *   same row chunking (row_begin, cu_seqlens, traj_index) and options.  Workspace:
 *   grpo_async_lmhead_workspace_size(n_rows, V, N) bytes.
 * grpo_async_lmhead_bwd -- the backward from the forward's lse and token_scale:
 *   recomputes z tile by tile and writes dz = grad_scale_mult * s_t (softmax(z) - onehot(y))
 *   as bf16 [n_rows, ld_dz] (ld_dz >= V, multiple of 8; columns [V, ld_dz) untouched), then
 *   dhidden = dz W (bf16 [n_rows, d], NULL to skip) and dW += dz^T hidden (f32 [V, d],
 *   accumulated so chunks add up; NULL to skip) as two tcgen05 GEMMs (lmhead_dx.cu: dz read
 *   K-major for dX and MN-major -- transposed in the descriptor, not in memory -- for dW).
 * grpo_async_lmhead_dx -- dhidden = dz W alone from an existing dz (bf16 [n_rows, ld_dz]):
 *   dhidden bf16 (out_bf16 = 1) or f32 [n_rows, d]; the unfused pipeline's dX GEMM.
 * grpo_async_lmhead_logits -- the plain logits hidden W^T as bf16 [n_rows, ld_out] (the
 *   unfused producer for grpo_async_loss_fwd, and the check of the GEMM).
 * Scheduling: the forward, dz and dW kernels hand their work units out dynamically from a
 * unit counter in library-owned device memory (one of 64 slots, zeroed by a 4-byte
 * cudaMemsetAsync on `stream` before each launch; more than 64 of these launches in flight
 * at once on different streams would share a slot); results never depend on the order.
 * Errors: GRPO_ERR_INVALID_ARG, GRPO_ERR_ALIGNMENT, GRPO_ERR_WORKSPACE, GRPO_ERR_CUDA.
 */
size_t grpo_async_lmhead_workspace_size(int64_t n_rows, int32_t V, int32_t N);

/*
 * Tensor-parallel LM head (NEXT(2) in the trainer's Megatron layout; NEXT(3)'s
 * vocabulary split): rank q holds W rows [col_offset, col_offset + Vs) and the full hidden
 * states.  Forward: grpo_async_lmhead_tp_partials computes this shard's per-row partial
 *   row_part[4*row .. 4*row+3] = 16 opaque bytes per row: (max in log2 units as float, z_y
 *   as float, the sum of 2^(t - max) as a double whose sign bit says "this shard holds
 *   y_t")   (workspace: grpo_async_lmhead_workspace_size(n_rows, Vs, 1));
 * the caller all-gathers the R ranks' row_part arrays in rank order ([R][n_rows][4]) and
 * grpo_async_lmhead_tp_fwd finishes logp / lse / token_scale / traj_sum / stats identically on
 * every rank (arguments as grpo_async_lmhead_fwd; workspace grpo_async_workspace_size).
 * Backward: grpo_async_lmhead_tp_bwd writes this shard's dz columns and, with dhidden_partial
 * (float [n_rows, d]), this shard's dz_q W_q -- the caller all-reduces (SUM) the partials
 * over the ranks -- and dW_q += dz_q^T hidden (float [Vs, d]).
 * Errors: as the single-GPU LM-head calls; GRPO_ERR_INVALID_ARG for R < 1 or col_offset < 0.
 */
grpo_status_t grpo_async_lmhead_tp_partials(const uint16_t *hidden, const uint16_t *W_shard,
                                            int64_t n_rows, int32_t d, int32_t Vs,
                                            int32_t col_offset, const int64_t *target_ids,
                                            float *row_part, void *workspace,
                                            size_t workspace_bytes, grpo_stream_t stream);
grpo_status_t grpo_async_lmhead_tp_fwd(const float *row_parts, int32_t R, int64_t row_begin,
                                       int64_t n_rows, int32_t V, const int64_t *target_ids,
                                       const float *logp_behav, const int64_t *cu_seqlens,
                                       int32_t N, const int32_t *traj_index, const float *adv,
                                       const float *inv_norm, const grpo_loss_opts_t *opts,
                                       float grad_scale, float *logp_out, float *lse_out,
                                       float *token_scale_out, double *traj_sum, double *stats,
                                       void *workspace, size_t workspace_bytes,
                                       grpo_stream_t stream);
grpo_status_t grpo_async_lmhead_tp_bwd(const uint16_t *hidden, const uint16_t *W_shard,
                                       int64_t n_rows, int32_t d, int32_t Vs, int32_t col_offset,
                                       const int64_t *target_ids, const float *lse,
                                       const float *token_scale, float grad_scale_mult,
                                       uint16_t *dz, int64_t ld_dz, float *dhidden_partial,
                                       float *dW_shard, grpo_stream_t stream);

/*
 * The tensor-parallel dhidden as one kernel that computes and communicates (GEMM ->
 * reduce-scatter over NVLink peer memory): rank `rank` of `world` multiplies its dz shard
 * (bf16 [n_rows, ld_dz], columns [0, Vs)) by its W shard (bf16 [Vs, d]) on the tensor cores
 * and its epilogue stores each f32 tile of rows r into slot `rank` of the rank that owns r
 * (rows_per_rank = ceil(n_rows / world); rank q owns rows [q*rpr, (q+1)*rpr)).
 *   slots[q]  device pointer (peer mapping) of rank q's slot buffer, f32
 *             [2][world][rows_per_rank][d], for q < world (host array of world pointers)
 *   epoch     the caller's count of tp_dx calls on these slots: call e writes half e % 2
 * After every rank's grpo_async_lmhead_tp_dx has completed (a group barrier, e.g. a NCCL
 * collective on the same stream), grpo_async_lmhead_tp_dx_reduce (same epoch) sums this rank's
 * world slots of that half in rank order into out [rows owned, d] (f32, or bf16 with
 * out_bf16 = 1): deterministic.  The two halves make one barrier per call enough: a fast rank
 * can write call e+1 while a slow one still reduces call e, and it reaches call e+2 (the half
 * of call e again) only after the barrier of call e+1, i.e. after every rank's reduce of e.
 * d % 128 == 0, world <= GRPO_VP_MAX_RANKS.  Errors: GRPO_ERR_INVALID_ARG, GRPO_ERR_ALIGNMENT,
 * GRPO_ERR_CUDA.
 */
grpo_status_t grpo_async_lmhead_tp_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W_shard,
                                      int64_t n_rows, int32_t d, int32_t Vs, int32_t world,
                                      int32_t rank, float *const *slots, uint32_t epoch,
                                      grpo_stream_t stream);
grpo_status_t grpo_async_lmhead_tp_dx_reduce(const float *own_slots, int32_t world, int64_t n_rows,
                                             int32_t d, int32_t rank, void *out, int32_t out_bf16,
                                             uint32_t epoch, grpo_stream_t stream);

grpo_status_t grpo_async_lmhead_dx(const uint16_t *dz, int64_t ld_dz, const uint16_t *W,
                                   int64_t n_rows, int32_t d, int32_t V, void *dhidden,
                                   int32_t out_bf16, grpo_stream_t stream);

/* dW (+)= dz^T hidden from an existing dz (bf16 [n_rows, ld_dz], as written by
 * grpo_async_lmhead_bwd / _tp_bwd), f32 [V, d] accumulated: lets a caller run the dW GEMM
 * while the tensor-parallel dhidden all-reduce is in flight.  tcgen05 GEMM (bf16 in, f32 out).
 * Errors: GRPO_ERR_INVALID_ARG, GRPO_ERR_ALIGNMENT, GRPO_ERR_CUDA. */
grpo_status_t grpo_async_lmhead_dw(const uint16_t *hidden, int64_t n_rows, int32_t d, int32_t V,
                                   const uint16_t *dz, int64_t ld_dz, float *dW,
                                   grpo_stream_t stream);

/* Tensor-core mode of the calling thread's later LM-head calls: 1 = one CTA per MMA
 * (tcgen05.mma.cta_group::1, 128 x 256 tiles), 2 = CTA pairs on one TPC (cta_group::2,
 * 256 x 256 tiles, each CTA stages half of the W tile; the default).  Same results.
 * Errors: GRPO_ERR_INVALID_ARG for other values. */
grpo_status_t grpo_async_lmhead_set_cta_group(int32_t cta_group);

grpo_status_t grpo_async_lmhead_fwd(const uint16_t *hidden, const uint16_t *W, int64_t row_begin,
                                    int64_t n_rows, int32_t d, int32_t V,
                                    const int64_t *target_ids, const float *logp_behav,
                                    const int64_t *cu_seqlens, int32_t N,
                                    const int32_t *traj_index, const float *adv,
                                    const float *inv_norm, const grpo_loss_opts_t *opts,
                                    float grad_scale, float *logp_out, float *lse_out,
                                    float *token_scale_out, double *traj_sum, double *stats,
                                    void *workspace, size_t workspace_bytes, grpo_stream_t stream);

grpo_status_t grpo_async_lmhead_bwd(const uint16_t *hidden, const uint16_t *W, int64_t n_rows,
                                    int32_t d, int32_t V, const int64_t *target_ids,
                                    const float *lse, const float *token_scale,
                                    float grad_scale_mult, uint16_t *dz, int64_t ld_dz,
                                    uint16_t *dhidden, float *dW, grpo_stream_t stream);

grpo_status_t grpo_async_lmhead_logits(const uint16_t *hidden, const uint16_t *W, int64_t n_rows,
                                       int32_t d, int32_t V, uint16_t *out, int64_t ld_out,
                                       grpo_stream_t stream);

/* Launch plan of the last fused-loss launch made by the calling thread. */
typedef struct {
    int32_t kernel;        /* 1 cluster-resident, 2 row-wise, 3 streamed ring, 4/5/6 LM-head */
                           /* (tcgen05) loss partials / logits gradient / logits, 7 vocab-  */
                           /* parallel row-wise, 8 vocab-parallel streamed ring, 9 the same  */
                           /* with pass 2 delayed by lag - 1 rows                            */
    int32_t cluster_size;  /* CTAs per row (kernel 1); CTAs per MMA (4-6)                     */
    int32_t ctas_per_sm;   /* requested residency                                            */
    int32_t stages;        /* kernel 1: row stages per CTA; 2: cached vectors per thread;   */
                           /* 3, 8: ring slots; 4-6: pipeline stages                         */
    int32_t vec_per_thread;/* kernels 1-3, 7, 8: threads per CTA (consumer threads for 3, 8); */
                           /* 4-6: vocabulary tiles per work unit                            */
    int32_t grid;          /* CTAs launched                                                  */
    int32_t max_clusters;  /* kernels 1, 2, 7: co-resident CTAs / clusters per SM the        */
                           /* occupancy query allows; 4-6: work units                        */
    int32_t smem_bytes;    /* dynamic shared memory per CTA                                  */
    int32_t lag;           /* kernel 1: reduction-to-backward lag in rows; 3: free ring     */
                           /* slots at the end of pass 1 (also 8); 7: deferred exchange wait; */
                           /* 9: grpo_vp_comm_t.lag (pass 2 after lag - 1 further rows)      */
} grpo_plan_t;

grpo_status_t grpo_async_last_plan(grpo_plan_t *out);

/* Bytes of device workspace grpo_async_loss_fwd needs for a chunk. */
size_t grpo_async_workspace_size(int64_t n_rows, int32_t V, int32_t N);

/*
 * Kernel tracing for benchmarks.  While enabled (process-wide), every launch
 * of the fused loss kernel (grpo_async_loss_fwd's main kernel, whichever
 * variant tune selects) is bracketed by two CUDA events recorded on the
 * launch's stream.  grpo_profile_collect() waits for the recorded events,
 * returns how many launches were traced since the last collect and the sum of
 * their durations in milliseconds, and recycles the events.
 * Errors: GRPO_ERR_CUDA (event creation/synchronization), GRPO_ERR_INVALID_ARG
 * (NULL outputs).
 */
grpo_status_t grpo_profile_enable(int32_t on);
grpo_status_t grpo_profile_collect(int32_t *n_launches, double *total_ms);

/* Number of kernels the last successful call of the calling thread launched
 * (for launch accounting in benchmarks). */
int32_t grpo_last_launch_count(void);

/* Thread-local text of the last error ("" if none). */
const char *grpo_last_error(void);

/* Library version string. */
const char *grpo_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GRPO_ASYNC_H */
