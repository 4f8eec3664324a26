/*
 * rlo.h — C ABI of the B200-native RL-objective hot path ("rlo" = ROLL objective).
 *
 * This is the drop-in boundary for the per-token RL objective that the ROLL
 * reference ("rollmini", /root/reference/proj) computes on the CPU between
 * generation and the actor update.  Every entry point names the reference
 * interface it replaces (file:line, relative to proj/core/).
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ / torch types cross this boundary.
 *  - Device pointers (suffix "device" in the comments) must be CUDA device
 *    memory of the handle's device.  The caller owns every buffer.
 *  - Calls taking a `stream` are asynchronous, stream-ordered on that
 *    cudaStream_t (NULL = legacy default stream), unless documented to sync.
 *  - One handle per (device, host thread, stream): the handle owns scratch
 *    workspace exactly like the reference's one PolicyWorkspace per worker
 *    (include/rollmini/policy_workers.hpp:41).
 *  - Errors are status codes; the message of the last failure on the calling
 *    thread is returned by rlo_last_error().  The codes map 1:1 onto the
 *    reference exception classes (include/rollmini/errors.hpp:11-82).
 *
 * Batch layout (the padded form of SampleBatch, include/rollmini/sample.hpp:16-60):
 *  B sequences, row stride T.  Per-token arrays are [B*T], token (b,t) at
 *  index b*T+t, valid iff t < lengths[b].  A NULL mask means "every response
 *  token participates" (the empty action_mask of sample.hpp:31).
 *  Logits row for token (b,t) starts at data + (b*T+t)*row_stride elements.
 */
#ifndef RLO_H_
#define RLO_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library is built -fvisibility=hidden; export exactly this header */
#endif

#define RLO_ABI_VERSION 5

/* Status codes — reference exception taxonomy (include/rollmini/errors.hpp). */
typedef enum rlo_status {
  RLO_OK = 0,
  RLO_ERR_INPUT = 1,    /* InputError    errors.hpp:33-37: OOV tokens, missing rewards/advantages/logprobs */
  RLO_ERR_CONFIG = 2,   /* ConfigError   errors.hpp:21-25: TrainConfig::validate, policy.cpp:29-37 */
  RLO_ERR_TRAINING = 3, /* TrainingError errors.hpp:65-69: zero tokens / non-finite loss or gradient */
  RLO_ERR_CUDA = 4,     /* device failure (no reference counterpart) */
  RLO_ERR_NCCL = 5,     /* collective failure; the reference's CollectError (errors.hpp:51-57) */
  RLO_ERR_DISPATCH = 6  /* DispatchError errors.hpp:39-43: unknown method name */
} rlo_status;

typedef enum rlo_dtype { RLO_DTYPE_F32 = 0, RLO_DTYPE_BF16 = 1 } rlo_dtype;

typedef enum rlo_adv_estimator {
  RLO_ADV_REINFORCE = 0, /* reference compute_advantages, policy.cpp:257-311 */
  RLO_ADV_GRPO = 1,      /* group-normalised sequence reward */
  RLO_ADV_GAE = 2        /* generalised advantage estimation over critic values */
} rlo_adv_estimator;

typedef enum rlo_kl_estimator {
  RLO_KL_K1 = 0, /* r = lp - ref_lp, the reference's term (policy.cpp:364-368) */
  RLO_KL_K2 = 1, /* r^2 / 2 */
  RLO_KL_K3 = 2  /* exp(-r) - 1 + r */
} rlo_kl_estimator;

typedef enum rlo_loss_agg {
  RLO_AGG_TOKEN_MEAN = 0,          /* reference: sum / tokens (policy.cpp:437-443) */
  RLO_AGG_SEQ_MEAN_TOKEN_MEAN = 1, /* GRPO sample-level mean */
  RLO_AGG_SEQ_MEAN_TOKEN_SUM = 2,
  RLO_AGG_GROUP_MEAN = 3           /* mean over groups of the group's token-mean */
} rlo_loss_agg;

/* TrainConfig (include/rollmini/policy.hpp:57-67) plus the ROLL extensions
 * the north star asks for.  rlo_train_config_default() gives the reference
 * defaults (policy.hpp:58-64; config keys config.cpp:197-205). */
typedef struct rlo_train_config {
  double clip_eps;          /* 0.2,  (0,1) */
  double kl_coef;           /* 0.0,  >= 0 */
  double learning_rate;     /* 0.05, >= 0 (validated for parity; the update is outside this path) */
  double advantage_clip;    /* 10.0, > 0 */
  double reward_clip;       /* 20.0, > 0 */
  double gamma;             /* 1.0,  (0,1] */
  int32_t whiten_advantages;/* 0 */
  /* extensions */
  int32_t adv_estimator;    /* rlo_adv_estimator, REINFORCE */
  double lambd;             /* GAE lambda, 0.95, [0,1] */
  int32_t kl_estimator;     /* rlo_kl_estimator, K1 */
  double dual_clip_c;       /* 0 = off; otherwise > 1 (dual-clip PPO) */
  int32_t loss_agg;         /* rlo_loss_agg, TOKEN_MEAN */
  int32_t group_size;       /* G: GRPO group / group-mean aggregation, 1 */
  int32_t grpo_std_ddof;    /* 0 (population std, like policy.cpp:301) or 1 */
  double grpo_eps;          /* 1e-6 */
} rlo_train_config;

/* Padded device view of a SampleBatch. */
typedef struct rlo_batch {
  int32_t B;               /* sequences in this view */
  int32_t T;               /* row stride of the per-token arrays */
  int32_t seq_offset;      /* index of this view's first sequence in the rank-local batch (micro-batching) */
  int32_t reserved;
  const int32_t* lengths;  /* [B] device: response lengths, 0..T */
  const int32_t* tokens;   /* [B*T] device: response_tokens (sample.hpp:21) */
  const uint8_t* mask;     /* [B*T] device or NULL: action_mask (sample.hpp:26) */
} rlo_batch;

/* One model's logits over the batch rows.  Padded layout (seq_start NULL):
 * token (b, t) is row b*T + t.  Packed / varlen layout: token (b, t) is row
 * seq_start[b] + t (e.g. cu_seqlens[b] of a [sum(lengths), V] tensor), only
 * rows t < lengths[b] exist and are read or written — the logits of a
 * ragged batch need no padding rows.  The per-token arrays of rlo_batch /
 * rlo_token_out stay [B*T]. */
typedef struct rlo_logits {
  const void* data;          /* device; dtype elements */
  int32_t dtype;             /* rlo_dtype */
  int32_t V;                 /* vocab size */
  int64_t row_stride;        /* elements between consecutive rows (>= V) */
  const int64_t* seq_start;  /* device [B] or NULL (padded) */
} rlo_logits;

/* Optional per-token outputs of rlo_ppo_gradient ([B*T] device, any may be NULL). */
typedef struct rlo_token_out {
  float* logp;      /* actor log-prob of the realised token */
  float* old_logp;  /* old-policy log-prob (when computed from old logits) */
  float* ref_logp;  /* reference log-prob (when computed from ref logits) */
  float* entropy;   /* actor entropy of the position */
  float* dlogp;     /* d(loss_t)/d(logp_t), policy.cpp:372-374 */
  float* loss;      /* per-token loss contribution (0 for non-participating tokens) */
  float* lse;       /* actor log-sum-exp of the row (input of rlo_logits_backward) */
  double* lse64;    /* the same in fp64 (input of rlo_logits_backward64: exact at any logit offset) */
} rlo_token_out;

/* Critic value-loss statistics (value_gradient, policy.cpp:474-540). */
typedef struct rlo_value_stats {
  double loss;           /* token-mean of 0.5*err^2 (clipped form when value_clip > 0) */
  double clip_fraction;  /* tokens where the clipped branch was taken */
  double mean_value;
  uint64_t tokens;
} rlo_value_stats;

/* UpdateStats (include/rollmini/policy.hpp:130-136) plus extension stats. */
typedef struct rlo_stats {
  double loss;               /* aggregated per cfg.loss_agg */
  double mean_ratio;
  double clip_fraction;
  double mean_kl;
  uint64_t tokens;
  double mean_entropy;       /* over loss-participating tokens */
  double dual_clip_fraction;
  uint64_t seqs;             /* sequences with >= 1 participating token */
  uint64_t groups;           /* groups with >= 1 participating token */
} rlo_stats;

/* Result of rlo_merge_gradients_async, written by the device (no host
 * synchronisation, so a whole step can be captured in a CUDA graph).
 * status: 0 ok, else the rlo_status merge_gradients would have returned
 * (with the reason in `reason`: 1 no loss-participating tokens, 2 non-finite
 * gradient, 3 non-finite loss, 4 a device-side input error — `dev_error` /
 * `dev_error_value` as reported by the kernels).  rlo_step_result_check()
 * turns a host copy into the same status and message. */
typedef struct rlo_step_result {
  rlo_stats stats;
  int32_t status;
  int32_t reason;
  int32_t dev_error;
  int32_t dev_error_value;
} rlo_step_result;

/* Per-rank partial sums: the scalar part of GradAccum (policy.hpp:121-128),
 * extended.  Merged in rank order exactly like merge_gradients
 * (policy.cpp:428-436).  Layout of v[] (all fp64; counts are exact integers): */
#define RLO_NPARTIAL 16
enum {
  RLO_P_LOSS_SUM = 0,   /* sum of per-token loss */
  RLO_P_RATIO_SUM = 1,
  RLO_P_KL_SUM = 2,
  RLO_P_ENTROPY_SUM = 3,
  RLO_P_CLIPPED = 4,
  RLO_P_DUAL_CLIPPED = 5,
  RLO_P_TOKENS = 6,
  RLO_P_SEQ_MEAN_SUM = 7,   /* sum over non-empty seqs of (seq loss sum / seq tokens) */
  RLO_P_SEQS = 8,           /* non-empty sequences */
  RLO_P_GROUP_MEAN_SUM = 9, /* sum over non-empty groups of (group loss sum / group tokens) */
  RLO_P_GROUPS = 10,        /* non-empty groups */
  RLO_P_NONFINITE_GRAD = 11,/* tokens whose dlogp is not finite */
  RLO_P_NONFINITE_LOSS = 12
};
typedef struct rlo_partials { double v[RLO_NPARTIAL]; } rlo_partials;

typedef struct rlo_handle rlo_handle;

/* ---- library / config (host only; callable without a GPU) -------------- */
int rlo_abi_version(void);
const char* rlo_last_error(void);
void rlo_train_config_default(rlo_train_config* cfg);
/* TrainConfig::validate (policy.cpp:29-37), same messages; plus extensions. */
rlo_status rlo_train_config_validate(const rlo_train_config* cfg);
/* split_sizes (sample.hpp:51-53, sample.cpp:99-105): contiguous, larger first. */
rlo_status rlo_split_sizes(int64_t n, int32_t parts, int64_t* out_sizes);
/* Group-aligned data-parallel shard of B sequences in groups of G: the
 * split_sizes rule applied to whole groups (G=1 reproduces split_batch,
 * sample.cpp:107-116).  Returns this rank's first sequence and count. */
rlo_status rlo_shard_plan(int32_t B, int32_t G, int32_t world, int32_t rank,
                          int32_t* out_seq_begin, int32_t* out_seq_count);
/* merge_gradients scalar part (policy.cpp:421-450): rank-ordered sum of
 * `nranks` partials, then normalisation; TrainingError on zero tokens or
 * non-finite values, with the reference's messages. */
rlo_status rlo_merge_partials(const rlo_partials* parts, int32_t nranks,
                              const rlo_train_config* cfg, rlo_stats* out);

/* Whitening parameters (policy.cpp:288-302) from rank-ordered statistics
 * stats_all[r*4 + {0,1,2}] = (sum, sum of squares, count) over masked
 * positions of rank r: mean, inv = 1/(sqrt(max(0, E[x^2]-mean^2)) + 1e-8).
 * Returns 1 when whitening applies (count > 0), else 0.  The device
 * normalise pass runs this same code on the all-gathered statistics. */
int32_t rlo_whiten_combine(const double* stats_all, int32_t world, double* mean, double* inv);

/* ---- handle ------------------------------------------------------------ */
rlo_status rlo_create(int32_t device, rlo_handle** out);
rlo_status rlo_destroy(rlo_handle* h);
/* NCCL data-parallel group (ranks = GPUs of one node, one handle per rank).
 * unique_id is 128 bytes from rlo_comm_unique_id on rank 0, shared by the caller. */
rlo_status rlo_comm_unique_id(void* unique_id_128);
rlo_status rlo_comm_init(rlo_handle* h, const void* unique_id_128, int32_t rank, int32_t world);
/* Kernel launches issued by this library since load (process-wide). */
uint64_t rlo_launch_count(void);

/* ---- the path ---------------------------------------------------------- */

/* forward_logprobs (policy.hpp:107-109, policy.cpp:210-233): log-softmax of
 * every valid response position (mask ignored, as the reference) gathered at
 * the realised token.  Single pass over each logits row (online
 * log-sum-exp); the softmax is never written.  Out-of-vocabulary tokens are
 * reported as RLO_ERR_INPUT by the next synchronising call (rlo_sync or
 * rlo_merge_gradients), with the reference message (policy.cpp:224-225).
 * out_logp required; out_entropy / out_token_logit optional.  Invalid
 * positions (t >= length) are written as 0. */
rlo_status rlo_forward_logprobs(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits,
                                float* out_logp, float* out_entropy, float* out_token_logit,
                                void* stream);

/* compute_advantages (policy.hpp:114-118, policy.cpp:257-311) and the ROLL
 * estimators.  Rewards: rewards_tok [B*T] (per-token, sample.hpp:24) or
 * rewards_seq [B] (scalar_reward, placed on the last token for
 * REINFORCE/GAE); values [B*T] for GAE.  With a communicator, the whitening
 * statistics are reduced over all ranks (NCCL all-gather + rank-ordered
 * sum) on the stream.  out_adv [B*T] required; out_returns optional (GAE:
 * A+V; REINFORCE: the discounted returns before whitening/clipping). */
rlo_status rlo_compute_advantages(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                                  const float* rewards_tok, const float* rewards_seq,
                                  const float* values, float* out_adv, float* out_returns,
                                  void* stream);

/* ppo_gradient loss part (policy.hpp:138-141, policy.cpp:313-374): fused
 * single pass over the actor logits (and, when given, the old-policy and
 * reference logits) computing log-probs, entropy, ratio, clip / dual-clip,
 * KL (k1/k2/k3), per-token loss and dlogp for every loss-participating
 * token.  Old / ref log-probs come from `old_logits` / `ref_logits` when
 * non-NULL, else from `old_logp` / `ref_logp` [B*T] (sampling-time
 * response_logprobs and ref_logprobs, sample.hpp:22-23).  ref may be absent
 * entirely (no KL), unless kl_coef > 0 (InputError, policy.cpp:342-343).
 * Per-sequence partial sums are accumulated in the handle (micro-batches:
 * call repeatedly with batch->seq_offset) until rlo_merge_gradients. */
rlo_status rlo_ppo_gradient(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                            const rlo_logits* actor_logits, const rlo_logits* old_logits,
                            const rlo_logits* ref_logits, const float* old_logp,
                            const float* ref_logp, const float* advantages,
                            const rlo_token_out* out, void* stream);

/* merge_gradients (policy.hpp:143-145, policy.cpp:421-450): reduces the
 * accumulated per-sequence sums in a fixed order into this rank's partials,
 * all-gathers them over the communicator (if any), merges in rank order and
 * normalises per cfg.loss_agg.  Synchronises `stream`; resets the
 * accumulator.  out_partials (this rank's, optional) may be NULL. */
rlo_status rlo_merge_gradients(rlo_handle* h, const rlo_train_config* cfg, rlo_stats* out,
                               rlo_partials* out_partials, void* stream);

/* merge_gradients without host synchronisation: the accumulated sequences
 * are reduced, all-gathered over the communicator (NCCL on `stream`) and
 * merged in rank order on the device into `out` (device or host-mapped
 * memory).  Every launch is capturable: warm the handle up with one eager
 * step of the same shapes, then capture compute_advantages -> ppo_gradient ->
 * merge_gradients_async in a CUDA graph and replay it (launch-bound small
 * batches).  Errors are reported in out->status, not returned. */
rlo_status rlo_merge_gradients_async(rlo_handle* h, const rlo_train_config* cfg, rlo_step_result* out, void* stream);

/* Status (and rlo_last_error message) of a host copy of an rlo_step_result:
 * exactly what the synchronous rlo_merge_gradients would have returned. */
rlo_status rlo_step_result_check(const rlo_step_result* host_result);

/* The rank-local GradAccum scalars of everything accumulated since the last
 * merge (what ppo_gradient returns per rank, policy.hpp:141): fixed-order
 * reduction of the per-sequence records, no cross-rank exchange and no
 * zero-token / non-finite checks (those belong to merge_gradients).
 * Synchronises `stream`; resets the accumulator. */
rlo_status rlo_rank_partials(rlo_handle* h, const rlo_train_config* cfg, rlo_partials* out, void* stream);

/* The whole path for one step (compute_advantages -> ppo_gradient ->
 * merge_gradients) on device-resident inputs. */
rlo_status rlo_objective_step(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                              const float* rewards_tok, const float* rewards_seq, const float* values,
                              const rlo_logits* actor_logits, const rlo_logits* old_logits,
                              const rlo_logits* ref_logits, const float* old_logp, const float* ref_logp,
                              float* out_adv, const rlo_token_out* out, rlo_stats* stats,
                              void* stream);

/* Host-buffer form of rlo_objective_step, the reference-facing call: the
 * SampleBatch arrays live in (preferably pinned) host memory and are copied
 * to device inside the call; advantages and actor log-probs are copied back.
 * Logits stay device-resident (they are the model's on-device output).
 * Host pointers: lengths [B]; tokens [B*T]; mask [B*T] or NULL; rewards_tok
 * [B*T] or NULL; rewards_seq [B] or NULL; values [B*T] or NULL; old_logp /
 * ref_logp [B*T] or NULL; host_adv_out / host_logp_out [B*T] or NULL.
 * Synchronises `stream`. */
rlo_status rlo_objective_step_host(rlo_handle* h, const rlo_train_config* cfg, int32_t B, int32_t T,
                                   const int32_t* lengths, const int32_t* tokens, const uint8_t* mask,
                                   const float* rewards_tok, const float* rewards_seq,
                                   const float* values, const rlo_logits* actor_logits,
                                   const rlo_logits* old_logits, const rlo_logits* ref_logits,
                                   const float* old_logp, const float* ref_logp,
                                   float* host_adv_out, float* host_logp_out, rlo_stats* stats,
                                   void* stream);

/* Micro-batched host-buffer step — the reference-facing call when the logits
 * of the whole batch do not fit in HBM at once (Qwen-vocabulary batches:
 * 1.3 TB per model for BASELINE cfg 3).  The SampleBatch arrays of all B
 * sequences are in (preferably pinned) host memory and are copied to the
 * device once; advantages (with the global whitening statistics) are computed
 * over the whole batch; then for every micro-batch of mb_seqs consecutive
 * sequences (the last may be shorter) `logits_fn` is called on the calling
 * thread to name that micro-batch's device logits — a trainer runs the model
 * forward for those sequences there, on `stream` — and the fused loss pass
 * runs on them; finally advantages and actor log-probs are copied back and the
 * partials merged (merge_gradients).  Host array layout as
 * rlo_objective_step_host.  The logits rows of micro-batch i are its own
 * n_seqs*T padded rows (or packed via seq_start relative to the micro-batch).
 * logits_fn fills *actor (required) and *old_logits / *ref_logits (leave
 * data = NULL for "not given": old_logp / ref_logp host arrays are used).
 * A non-RLO_OK return from logits_fn aborts the step with that status.
 * Synchronises `stream`. */
typedef rlo_status (*rlo_logits_fn)(void* user, int32_t micro_batch, int32_t seq_begin, int32_t n_seqs,
                                    rlo_logits* actor, rlo_logits* old_logits, rlo_logits* ref_logits);
rlo_status rlo_objective_step_host_mb(rlo_handle* h, const rlo_train_config* cfg, int32_t B, int32_t T,
                                      int32_t mb_seqs, const int32_t* lengths, const int32_t* tokens,
                                      const uint8_t* mask, const float* rewards_tok, const float* rewards_seq,
                                      const float* values, rlo_logits_fn logits_fn, void* user,
                                      const float* old_logp, const float* ref_logp, float* host_adv_out,
                                      float* host_logp_out, rlo_stats* stats, void* stream);

/* ---- next rows: the callers either side of the path ------ */

/* Aggregation weight of every loss-participating token (0 elsewhere): the
 * factor from d(loss_t)/d(logp_t) to d(L)/d(logp_t) under cfg.loss_agg, using
 * the merged (global) counts of `stats` (from rlo_merge_gradients):
 * token-mean 1/tokens (policy.cpp:438-440), seq-mean-token-mean
 * 1/(seqs*m_b), seq-mean-token-sum 1/seqs, group-mean 1/(groups*M_g), with
 * m_b / M_g the participating tokens of the sample / group.  out_w [B*T]. */
rlo_status rlo_loss_weights(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                            const rlo_stats* stats, float* out_w, void* stream);

/* The aggregation normalisers of a batch BEFORE its vocab pass: loss-
 * participating tokens, sequences with at least one such token and groups
 * (cfg.group_size consecutive samples) with at least one, summed over the
 * communicator's ranks in rank order (the counts merge_gradients derives,
 * policy.cpp:437-440).  Fills out->tokens / seqs / groups, zeroes the rest, so
 * `out` can feed rlo_loss_weights ahead of rlo_ppo_gradient_fused.
 * Synchronises `stream`. */
rlo_status rlo_batch_counts(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch, rlo_stats* out,
                            void* stream);

/* Actor backward epilogue (policy.cpp:375-379): for every row with
 * weight*dlogp != 0, grad[v] = weight*dlogp*(1[v == token] - exp(z_v - lse)),
 * recomputing the softmax from the row and its lse (never stored); all
 * other rows of `grad` are zeroed (with packed logits, rlo_logits.seq_start,
 * gradient rows follow the same layout and only existing rows are written).
 * The lse is fp32, so p carries its rounding (relative <= ulp(lse)/2: 4e-6 at
 * |lse| < 64); rlo_logits_backward64 (fp64 lse) and the fused pass have no
 * such term.  grad has grad_dtype (rlo_dtype) and
 * grad_row_stride; lse / dlogp / weight are [B*T] (rlo_token_out.lse,
 * rlo_token_out.dlogp, rlo_loss_weights). */
rlo_status rlo_logits_backward(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits, const float* lse,
                               const float* dlogp, const float* weight, void* grad, int32_t grad_dtype,
                               int64_t grad_row_stride, void* stream);

/* rlo_logits_backward with the fp64 lse (rlo_token_out.lse64): the softmax is
 * rebuilt as 2^(z*log2e - (lse*log2e)_hi - (lse*log2e)_lo), so the fp32
 * rounding of the lse drops out (relative error ~1e-7 at any logit offset). */
rlo_status rlo_logits_backward64(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits, const double* lse64,
                                 const float* dlogp, const float* weight, void* grad, int32_t grad_dtype,
                                 int64_t grad_row_stride, void* stream);

/* Fused update pass: rlo_ppo_gradient (same inputs, outputs, accumulation and
 * errors) and the actor backward epilogue in ONE read of the actor logits
 * (policy.cpp:355-379).  A thread-block cluster holds each actor row in shared
 * memory while the row's log-sum-exp, entropy, KL and surrogate are formed,
 * then writes grad[v] = weight*dlogp*(1[v == token] - softmax_v) from it;
 * rows without loss participation get zeros.  weight [B*T] must be known
 * before the pass (rlo_batch_counts -> rlo_loss_weights).  HBM traffic per
 * participating row P*V*s + V*s_grad instead of (P+1)*V*s + V*s_grad.  Runs
 * for fp32 rows of <= 128 KB (4 CTAs of 32 KB shared memory); bf16 rows,
 * larger rows and rows that are not 16-byte aligned take the two-pass form
 * transparently (measured faster there). */
rlo_status rlo_ppo_gradient_fused(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                                  const rlo_logits* actor, const rlo_logits* old_logits, const rlo_logits* ref_logits,
                                  const float* old_logp, const float* ref_logp, const float* advantages,
                                  const float* weight, void* grad, int32_t grad_dtype, int64_t grad_row_stride,
                                  const rlo_token_out* out, void* stream);

/* Critic value loss (value_gradient, policy.cpp:474-540): per
 * loss-participating token err = v - return, loss 0.5*err^2, d/dv = err.
 * With old_values and value_clip > 0: the clipped PPO value loss
 * 0.5*max((v-R)^2, (v_old + clamp(v - v_old, +-c) - R)^2).  Reduced over the
 * communicator like merge_gradients.  out_dvalue [B*T] optional (0 off-mask).
 * Synchronises `stream`; TrainingError when no token participates. */
rlo_status rlo_value_loss(rlo_handle* h, const rlo_batch* batch, const float* values, const float* old_values,
                          const float* returns, double value_clip, float* out_dvalue, rlo_value_stats* out,
                          void* stream);

/* Sampling-time log-probs: decode_next (policy.cpp:143-169) for n_rows logits
 * rows — a tempered categorical draw by a CDF walk in token order with the
 * reference's keyed uniform u = keyed_double({seed, version, sample_key[i],
 * position[i]}) (rng.hpp:82-85), returning the token and its UNtempered
 * log-prob (policy.cpp:168), i.e. response_logprobs, so the PPO ratio needs
 * no separate old-policy logits pass.  The token is the fp64 CDF walk's (the
 * reference's unless u*total falls within fp64 rounding of a CDF boundary):
 * an fp32 screen certifies most draws (u*total more than an error bound away
 * from the picked token's CDF boundaries), the rest are redone with fp64
 * weights; the untempered log-sum-exp in fp32.  Two kernel launches, no host
 * synchronisation; out_tokens is written twice (uncertified rows hold -1
 * between the launches).  RLO_DECODE_MARGIN overrides the certificate margin
 * (<= 0: fp64 only).
 * sample_keys / positions [n_rows] device uint64; out_tokens int32 [n_rows];
 * out_logp float [n_rows].  ConfigError for temperature <= 0 (policy.cpp:146). */
rlo_status rlo_decode_sample(rlo_handle* h, const rlo_logits* logits, int32_t n_rows, double temperature,
                             uint64_t seed, uint64_t version, const uint64_t* sample_keys, const uint64_t* positions,
                             int32_t* out_tokens, float* out_logp, void* stream);

/* rng::hash_str (rng.hpp:34-41): the per-sample key of a sample_id. Host only. */
uint64_t rlo_sample_key(const char* sample_id);

/* ---- wire format + parameter sync (§8f row 4) ---------------------------- */

/* A SampleBatch parsed from the reference's JSONL wire format
 * (SampleBatch::from_jsonl, sample.cpp:124-159) into padded HOST arrays
 * (malloc'ed; free with rlo_host_batch_free).  T = longest response.  Arrays a
 * batch does not carry at all are NULL.  mask: 1 for samples with an empty
 * action_mask (sample.hpp:31).  rewards: per-token rewards, with a sample
 * that has only scalar_reward getting it on its last token (policy.cpp:265-271);
 * scalar_rewards: NaN where absent.  first_missing_reward: first sample with
 * neither (compute_advantages' InputError, policy.cpp:274-275), else -1.
 * sample_keys = rng::hash_str(sample_id); group_index = group_id in order of
 * first appearance. */
typedef struct rlo_host_batch {
  int32_t B, T;
  int32_t first_missing_reward;
  int32_t reserved;
  int32_t* lengths;
  int32_t* tokens;
  uint8_t* mask;
  float* rewards;
  float* scalar_rewards;
  float* response_logprobs;
  float* ref_logprobs;
  float* advantages;
  uint64_t* sample_keys;
  int32_t* group_index;
} rlo_host_batch;

/* Parse + SampleBatch::validate (sample.cpp:85-102, same messages).  Host only. */
rlo_status rlo_batch_from_jsonl(const char* text, size_t len, rlo_host_batch** out);
void rlo_host_batch_free(rlo_host_batch* batch);

/* bucket_plan (policy.cpp:542-548): contiguous bucket sizes (each <=
 * bucket) covering total elements, ceiling division with a short tail
 * ({0} for total 0).  out has room for *n_buckets entries on input; the count
 * is returned in *n_buckets.  Host only. */
rlo_status rlo_bucket_plan(uint64_t total, uint64_t bucket, uint64_t* out, int64_t* n_buckets);

/* ModelUpdateGroup (sync_params policy_workers.cpp:234-260):
 * broadcast a device buffer from `root` to every rank of the handle's NCCL
 * group in contiguous buckets of at most bucket_bytes (NVLink; the
 * reference's bucketed train -> infer parameter sync).  Destinations end
 * bit-identical.  Stream-ordered. */
rlo_status rlo_broadcast_params(rlo_handle* h, void* buffer, uint64_t bytes, uint64_t bucket_bytes, int32_t root,
                                void* stream);

/* Synchronise `stream` and report device-side input errors (OOV tokens). */
rlo_status rlo_sync(rlo_handle* h, void* stream);

/* ---- synthetic inputs (bench / tests; not on the path) ------------------ */
/* Counter-hash logits identical to oracle/ synth twin: row r of model m is a
 * pure function of (seed, m, r mod key_rows) — see DESIGN.md §synthetic. */
rlo_status rlo_synth_logits(void* dst, int32_t dtype, int64_t rows, int32_t V, int64_t row_stride,
                            uint64_t seed, int32_t model_id, int64_t row_key_offset, void* stream);
rlo_status rlo_synth_tokens(int32_t* dst, int64_t rows, int32_t V, uint64_t seed,
                            int64_t row_key_offset, int64_t key_rows, void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* RLO_H_ */
