/*
 * oracle.h — CPU restatement of the reference's RL-objective path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_2506_06122_b200/) never links, loads or calls it.
 *
 * Every function restates /root/reference/proj/core/src/policy.cpp (cited
 * per function) in fp64 with the reference's fixed summation order, on the
 * padded [B, T] batch layout of include/rlo.h.  Extensions the reference
 * does not have (entropy, k2/k3, dual-clip, GRPO, GAE, seq/group
 * aggregation) are restated from their standard definitions (SURVEY.md
 * Appendix A); their parity is pinned only by this restatement ("parity
 * unpinned by reference tests").  The reference-backed parts are pinned by
 * tests/golden/ fixtures produced from the reference's own code
 * (oracle/_ref, built by oracle/Makefile).
 */
#ifndef RLO_ORACLE_H_
#define RLO_ORACLE_H_

#include <stdint.h>

#include "../include/rlo.h"

#ifdef __cplusplus
extern "C" {
#endif

/* policy.cpp:116-122 on one row (fp64, max pass, ascending exp-sum, log).
 * entropy_out (nullable): H = sum_v p_v (lse - z_v), two-pass in fp64. */
void orc_logsoftmax_row(const double* z, int32_t V, double* lse_out, double* entropy_out);

/* policy.cpp:210-233 over a padded batch.  logits are host fp32 or bf16
 * (dtype per rlo_dtype), row (b*T+t) at logits + (b*T+t)*row_stride.
 * Scores every valid position regardless of mask.  Returns rlo_status. */
int32_t orc_forward_logprobs(const void* logits, int32_t dtype, int32_t V, int64_t row_stride,
                             int32_t B, int32_t T, const int32_t* lengths, const int32_t* tokens,
                             double* out_lp, double* out_entropy, double* out_tok_logit,
                             char* err, int32_t errlen);

/* policy.cpp:257-311 (REINFORCE) + GRPO + GAE.  rewards_tok [B*T] or
 * rewards_seq [B] (or both NULL -> InputError for non-empty samples). */
int32_t orc_compute_advantages(const rlo_train_config* cfg, int32_t B, int32_t T,
                               const int32_t* lengths, const uint8_t* mask,
                               const double* rewards_tok, const double* rewards_seq,
                               const double* values, double* out_adv, double* out_returns,
                               char* err, int32_t errlen);

/* policy.cpp:335-374 loss part, sequentially in token order.  ref_lp and
 * entropy nullable.  Writes per-token loss / dlogp (0 off-mask) and the
 * partial sums for the batch (one "rank"). */
int32_t orc_ppo_loss(const rlo_train_config* cfg, int32_t B, int32_t T, const int32_t* lengths,
                     const uint8_t* mask, const double* lp, const double* old_lp,
                     const double* ref_lp, const double* adv, const double* entropy,
                     double* out_loss_tok, double* out_dlogp, rlo_partials* out_partials,
                     char* err, int32_t errlen);

/* policy.cpp:421-450 scalar merge (rank order) + aggregation modes. */
int32_t orc_merge(const rlo_partials* parts, int32_t nranks, const rlo_train_config* cfg,
                  rlo_stats* out, char* err, int32_t errlen);

/* sample.cpp:99-105 */
void orc_split_sizes(int64_t n, int32_t parts, int64_t* out);

/* Aggregation weight of every loss-participating token (0 elsewhere): the
 * factor turning d(loss_t)/d(logp_t) into d(L)/d(logp_t) for cfg->loss_agg
 * (token-mean: 1/tokens, policy.cpp:438-440; seq-mean-token-mean:
 * 1/(seqs*m_b); seq-mean-token-sum: 1/seqs; group-mean: 1/(groups*M_g)). */
void orc_loss_weights(const rlo_train_config* cfg, int32_t B, int32_t T, const int32_t* lengths,
                      const uint8_t* mask, double* out_w);

/* Actor backward epilogue restated from policy.cpp:376-379:
 * dz[v] = scale * (1[v == tok] - exp(z_v - lse)), scale = w_t * dlogp_t. */
void orc_logits_backward_row(const double* z, int32_t V, int32_t tok, double scale, double* out);

/* Critic value loss, value_gradient restated (policy.cpp:500-512): per
 * loss-participating token err = v - target, loss 0.5*err^2, d/dv = err.
 * Extension: with old_values and value_clip > 0, the clipped PPO value loss
 * 0.5*max((v-R)^2, (v_old + clamp(v - v_old, +-c) - R)^2).
 * out4 = {loss_sum, tokens, clipped, sum of values}; out_dv per token (0 off-mask). */
void orc_value_loss(int32_t B, int32_t T, const int32_t* lengths, const uint8_t* mask, const double* values,
                    const double* old_values, const double* returns, double value_clip, double* out_dv,
                    double* out4);

/* decode_next restated (policy.cpp:143-169) on one logits row: tempered CDF
 * walk with u = keyed_double({seed, version, sample_key, position})
 * (rng.hpp:15-31, 82-85); returns the token, *logp = untempered log-prob. */
int32_t orc_decode_next(const double* z, int32_t V, double temperature, uint64_t seed, uint64_t version,
                        uint64_t sample_key, uint64_t position, double* logp);
uint64_t orc_hash_str(const char* s); /* rng.hpp:34-41 */

/* Synthetic row / token of include/rlo_synth.h, as doubles (bf16-rounded
 * when dtype is bf16). */
void orc_synth_row(double* out, int32_t dtype, int32_t V, uint64_t seed, int32_t model, uint64_t row_key);
void orc_synth_row_raw(void* out, int32_t dtype, int32_t V, uint64_t seed, int32_t model, uint64_t row_key);
int32_t orc_synth_token(uint64_t seed, uint64_t row_key, int32_t V);

/* CPU baseline ("port"): the restated path over a bounded sample, on
 * `threads` host threads (contiguous sequence ranges, thread-per-rank as in
 * the reference's cluster.cpp:146).  Synthetic logits are generated once into
 * `key_rows` resident rows per model; token row r reads row r % key_rows.
 * Returns elapsed seconds of the timed part; *checksum gets sum of losses. */
double orc_bench_objective(int32_t threads, const rlo_train_config* cfg, int32_t dtype, int32_t V,
                           int32_t B, int32_t T, int32_t key_rows, uint64_t seed, double* checksum);

#ifdef __cplusplus
}
#endif

#endif /* RLO_ORACLE_H_ */
