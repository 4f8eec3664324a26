// internal.h — declarations shared by the C-ABI host layer (api.cpp) and the
// sm_100a kernels (*.cu).  Not installed; the public surface is include/rlo.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <cmath>

#include "../../include/rlo.h"

#if defined(__CUDACC__)
#define RLO_HOST_DEVICE __host__ __device__
#else
#define RLO_HOST_DEVICE
#endif


namespace rlo {

extern std::atomic<uint64_t> g_launches;

// Records the calling thread's rlo_last_error() message and returns `code`.
rlo_status set_last_error(rlo_status code, const std::string& msg);

// Roles of the (up to 3) logits tensors a vocab pass reads.
enum Role : int32_t { ROLE_ACTOR = 0, ROLE_OLD = 1, ROLE_REF = 2 };

// Per-token flag bits written by the loss epilogue.
enum : uint8_t { TF_CLIPPED = 1, TF_DUAL = 2, TF_NONFINITE_GRAD = 4, TF_NONFINITE_LOSS = 8 };

// Device error slot.  The reference raises the FIRST failure in sample order
// (policy.cpp:223-225 walks samples, then positions), so the slot keeps the
// minimum of a 64-bit key over every failing row (atomicMin; no ordering
// between CTAs needed):  key = class:2 | position:30 | value:32, with class
// 0 = response length outside [0, T] (position = sequence, value = sequence),
// 1 = OOV token in forward_logprobs, 2 = OOV token in the loss pass
// (position = global row (seq_offset + b) * T + t, value = the token id).
// A length error therefore wins over any OOV token, and the earliest row wins
// among OOV tokens.  kDevErrNone (all ones) = no error; reset by memset 0xFF.
enum : int32_t { DE_NONE = 0, DE_OOV_LOGPROB = 1, DE_OOV_LOSS = 2, DE_BAD_LENGTH = 3 };
constexpr unsigned long long kDevErrNone = ~0ull;
struct DevError {
  unsigned long long key;
};
RLO_HOST_DEVICE inline unsigned long long dev_err_key(int32_t code, int64_t pos, int32_t value) {
  const unsigned long long cls = code == DE_BAD_LENGTH ? 0ull : code == DE_OOV_LOGPROB ? 1ull : 2ull;
  const unsigned long long p = pos < 0 ? 0ull : pos > 0x3FFFFFFF ? 0x3FFFFFFFull : (unsigned long long)pos;
  return (cls << 62) | (p << 32) | (unsigned long long)(uint32_t)value;
}
// Decoded slot: code DE_* (DE_NONE when empty) and its value.
RLO_HOST_DEVICE inline void dev_err_decode(unsigned long long key, int32_t* code, int32_t* value) {
  if (key == kDevErrNone) {
    *code = DE_NONE;
    *value = 0;
    return;
  }
  const unsigned long long cls = key >> 62;
  *code = cls == 0 ? DE_BAD_LENGTH : cls == 1 ? DE_OOV_LOGPROB : DE_OOV_LOSS;
  *value = (int32_t)(uint32_t)(key & 0xFFFFFFFFull);
}

// Per-sequence record of the loss pass (fp64 sums in a fixed order).
struct SeqRec {
  double loss, ratio, kl, entropy;
  double clipped, dual, tokens, nonfinite_grad, nonfinite_loss;
  double pad;
};

// Per-slot whitening statistics (slot = sequence, or group for GRPO).
struct WStat {
  double sum, sq, count, pad;
};


// Whitening parameters from rank-ordered statistics stats_all[r*4 + {0,1,2}] =
// (sum, sum of squares, count) over masked positions (policy.cpp:288-302):
// mean, var = max(0, E[x^2] - mean^2), inv = 1/(sqrt(var) + 1e-8).  Returns 0
// (no whitening) when the count is zero.  Shared by whiten_clip_kernel and the
// host (rlo_whiten_combine), so the CPU multi-rank tests exercise this code.
RLO_HOST_DEVICE inline int whiten_combine(const double* stats_all, int world, double* mean, double* inv) {
  double sum = 0.0, sq = 0.0, cnt = 0.0;
  for (int r = 0; r < world; ++r) {
    sum += stats_all[r * 4 + 0];
    sq += stats_all[r * 4 + 1];
    cnt += stats_all[r * 4 + 2];
  }
  if (!(cnt > 0.0)) return 0;
  const double m = sum / cnt;
  const double d = sq / cnt - m * m;
  *mean = m;
  *inv = 1.0 / (sqrt(d > 0.0 ? d : 0.0) + 1e-8);
  return 1;
}

// merge_gradients normalisation (policy.cpp:421-450) of rank-ordered
// partials parts[r*RLO_NPARTIAL + k]: returns 0, or the reason the reference
// aborts (1 no tokens, 2 non-finite gradient, 3 non-finite loss).  Shared by
// the host merge and the device finalize kernel (graph-capturable step).
RLO_HOST_DEVICE inline int32_t merge_stats(const double* parts, int32_t world, int32_t agg, rlo_stats* st) {
  double s[RLO_NPARTIAL];
  for (int k = 0; k < RLO_NPARTIAL; ++k) s[k] = 0.0;
  for (int32_t r = 0; r < world; ++r)
    for (int k = 0; k < RLO_NPARTIAL; ++k) s[k] += parts[r * RLO_NPARTIAL + k];
  if (s[RLO_P_TOKENS] == 0.0) return 1;
  if (s[RLO_P_NONFINITE_GRAD] > 0.0) return 2;
  const double inv = 1.0 / s[RLO_P_TOKENS];
  rlo_stats o;
  if (agg == RLO_AGG_SEQ_MEAN_TOKEN_MEAN)
    o.loss = s[RLO_P_SEQ_MEAN_SUM] * (1.0 / s[RLO_P_SEQS]);
  else if (agg == RLO_AGG_SEQ_MEAN_TOKEN_SUM)
    o.loss = s[RLO_P_LOSS_SUM] * (1.0 / s[RLO_P_SEQS]);
  else if (agg == RLO_AGG_GROUP_MEAN)
    o.loss = s[RLO_P_GROUP_MEAN_SUM] * (1.0 / s[RLO_P_GROUPS]);
  else
    o.loss = s[RLO_P_LOSS_SUM] * inv;
  o.mean_ratio = s[RLO_P_RATIO_SUM] * inv;
  o.clip_fraction = s[RLO_P_CLIPPED] * inv;
  o.mean_kl = s[RLO_P_KL_SUM] * inv;
  o.tokens = static_cast<uint64_t>(s[RLO_P_TOKENS]);
  o.mean_entropy = s[RLO_P_ENTROPY_SUM] * inv;
  o.dual_clip_fraction = s[RLO_P_DUAL_CLIPPED] * inv;
  o.seqs = static_cast<uint64_t>(s[RLO_P_SEQS]);
  o.groups = static_cast<uint64_t>(s[RLO_P_GROUPS]);
  *st = o;
  return isfinite(o.loss) ? 0 : 3;
}

// Diagnostic / experiment knobs, read ONCE from the environment when a
// handle is created (rlo_create) and never per launch.  None of them changes
// the numerics of the default path beyond its stated tolerance: they select
// the fused pass's slice budget and pipeline depth (or switch it off), and
// the decode screen's certificate margin.
//   RLO_FUSED_OFF=1          fused update pass -> two-pass form
//   RLO_FUSED_SLICE_KB=n     per-CTA actor slice budget (also enables bf16 rows)
//   RLO_FUSED_NB=3           three actor slices in flight instead of two
//   RLO_FUSED_DEBUG=1        print the fused launch shape
//   RLO_DECODE_MARGIN=x      fixed certificate margin (<= 0: fp64 path only)
//   RLO_DECODE_NOREDO=1      leave the screen's -1 marks (measures its fail rate)
struct Tuning {
  bool fused_off = false;
  int fused_slice_kb = 0;
  int fused_nb = 2;
  bool fused_debug = false;
  bool decode_fixed_margin = false;
  double decode_margin = -1.0;
  bool decode_noredo = false;
};
Tuning read_tuning();

struct VocabArgs {
  const void* logits[3];
  int64_t stride[3];
  const int64_t* seq_start[3];  // packed layout per tensor (rlo_logits.seq_start), NULL = padded
  int32_t role[3];
  int32_t ntens;
  int32_t dtype;  // rlo_dtype shared by all tensors of the pass
  int32_t V;
  int32_t B, T;
  int32_t seq_offset;  // first sequence of this view in the rank-local batch (error ordering)
  const int32_t* lengths;
  const int32_t* tokens;
  const uint8_t* mask;
  // forward_logprobs mode
  float* out_lp;
  float* out_ent;
  float* out_tok;
  // loss mode
  const float* old_lp_in;
  const float* ref_lp_in;
  const float* adv;
  double clip_eps, kl_coef, dual_c;
  int32_t kl_est;
  int32_t has_ref;  // KL term / kl_sum present (ref logits or ref_lp_in)
  float* o_logp;
  float* o_old;
  float* o_ref;
  float* o_ent;
  float* o_dlogp;
  float* o_loss;
  float* o_lse;
  double* o_lse64;
  // scratch consumed by the per-sequence reduction
  float* s_loss;
  float* s_ratio;
  float* s_kl;
  float* s_ent;
  uint8_t* s_flags;
  DevError* err;
};

struct AdvArgs {
  int32_t B, T;
  const int32_t* lengths;
  const uint8_t* mask;
  const float* rewards_tok;
  const float* rewards_seq;
  const float* values;
  float* out_adv;
  float* out_returns;
  int32_t estimator;
  double gamma, lambd, reward_clip, adv_clip;
  int32_t whiten;
  int32_t G, ddof;
  double grpo_eps;
  WStat* wstat;   // [B] (scan) or [B/G] (GRPO) when whiten
  double* raw64;  // [B*T] raw advantages in fp64 when whiten
};

// Launchers (return cudaGetLastError()).
cudaError_t launch_vocab_logprob(const VocabArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_vocab_loss(const VocabArgs& a, int num_sms, cudaStream_t s);
// Fused update pass (fused.cu): cluster size K (0 = not eligible) and the
// per-CTA slice length, then the launch.
int fused_cluster_size(const VocabArgs& a, const void* grad, int32_t gdtype, int64_t gstride, const Tuning& tu,
                       int32_t* slice);
cudaError_t launch_vocab_fused(const VocabArgs& a, const float* weight, void* grad, int32_t gdtype, int64_t gstride,
                               int K, int32_t slice, const Tuning& tu, cudaStream_t s);
cudaError_t launch_seq_reduce(int32_t B, int32_t T, int32_t seq_offset, const int32_t* lengths,
                              const uint8_t* mask, const float* s_loss, const float* s_ratio,
                              const float* s_kl, const float* s_ent, const uint8_t* s_flags, SeqRec* recs,
                              cudaStream_t s);
cudaError_t launch_merge_finalize(const double* parts, int32_t world, int32_t agg, DevError* err,
                                  rlo_step_result* out, cudaStream_t s);
cudaError_t launch_batch_reduce(const SeqRec* recs, int32_t nseq, int32_t G, double* partials,
                                cudaStream_t s);
cudaError_t launch_advantages(const AdvArgs& a, cudaStream_t s);
cudaError_t launch_wstat_reduce(const WStat* w, int32_t n, double* out4, cudaStream_t s);
cudaError_t launch_whiten_clip(const AdvArgs& a, const double* stats_all, int32_t world, cudaStream_t s);
cudaError_t launch_loss_weights(int32_t B, int32_t T, int32_t G, int32_t agg, double tokens, double seqs,
                                double groups, const int32_t* lengths, const uint8_t* mask, float* counts, float* w,
                                cudaStream_t s);
// Loss-participating tokens, non-empty sequences and non-empty groups of a
// batch -> out4[0..2] (fp64, exact integers); counts [B] scratch.
cudaError_t launch_batch_counts(int32_t B, int32_t T, int32_t G, const int32_t* lengths, const uint8_t* mask,
                                float* counts, double* out4, cudaStream_t s);
cudaError_t launch_logits_backward(const void* logits, int32_t dtype, int64_t stride, const int64_t* seq_start,
                                   int32_t V, int32_t B, int32_t T,
                                   const int32_t* lengths, const int32_t* tokens, const float* lse,
                                   const double* lse64, const float* dlogp,
                                   const float* weight, void* grad, int32_t gdtype, int64_t gstride, int num_sms,
                                   cudaStream_t s);
cudaError_t launch_value_loss(int32_t B, int32_t T, const int32_t* lengths, const uint8_t* mask, const float* values,
                              const float* old_values, const float* returns, double clip, float* dv,
                              double* seqsums, double* out4, cudaStream_t s);
cudaError_t launch_decode(const void* logits, int32_t dtype, int64_t stride, int32_t V, int32_t n, double temperature,
                          uint64_t seed, uint64_t version, const uint64_t* keys, const uint64_t* positions,
                          int32_t* out_tok, float* out_lp, int num_sms, const Tuning& tu, cudaStream_t s);
cudaError_t launch_synth_logits(void* dst, int32_t dtype, int64_t rows, int32_t V, int64_t row_stride,
                                uint64_t seed, int32_t model_id, int64_t row_key_offset, cudaStream_t s);
cudaError_t launch_synth_tokens(int32_t* dst, int64_t rows, int32_t V, uint64_t seed, int64_t row_key_offset,
                                int64_t key_rows, cudaStream_t s);

}  // namespace rlo
