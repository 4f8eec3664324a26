/*
 * oracle.c — CPU restatement of the reference RL-objective path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the checker for the CUDA path and
 * the "port" CPU baseline.  Never linked into or called by the product.
 *
 * Reference = /root/reference/proj/core/src/policy.cpp (cited per function).
 * fp64 throughout, fixed summation order ("All arithmetic in
 * 64-bit floating point with fixed reduction order").
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "../include/rlo_synth.h"

static int32_t fail(char* err, int32_t errlen, int32_t code, const char* fmt, ...) {
  if (err && errlen > 0) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, (size_t)errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

static inline double clampd(double v, double lo, double hi) {
  /* std::clamp semantics (NaN passes through), as used at policy.cpp:277/309/359. */
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

static inline int mask_at(const uint8_t* mask, int64_t i) { return mask == NULL || mask[i] != 0; }

/* ---- log-softmax: policy.cpp:116-122 --------------------------------------- */
void orc_logsoftmax_row(const double* z, int32_t V, double* lse_out, double* entropy_out) {
  double m = z[0];
  for (int32_t v = 1; v < V; ++v) m = (m < z[v]) ? z[v] : m; /* std::max(m, z[v]) */
  double s = 0.0;
  for (int32_t v = 0; v < V; ++v) s += exp(z[v] - m);
  const double lse = m + log(s);
  *lse_out = lse;
  if (entropy_out) {
    /* Extension (not in the reference): H = sum_v p_v * (lse - z_v), p_v = exp(z_v - lse). */
    double h = 0.0;
    for (int32_t v = 0; v < V; ++v) {
      const double lp = z[v] - lse;
      const double p = exp(lp);
      if (p > 0.0) h -= p * lp;
    }
    *entropy_out = h;
  }
}

static void load_row(const void* logits, int32_t dtype, int64_t off, int32_t V, double* out) {
  if (dtype == RLO_DTYPE_F32) {
    const float* p = (const float*)logits + off;
    for (int32_t v = 0; v < V; ++v) out[v] = (double)p[v];
  } else {
    const uint16_t* p = (const uint16_t*)logits + off;
    for (int32_t v = 0; v < V; ++v) out[v] = (double)rlo_bf16_to_f32(p[v]);
  }
}

/* ---- forward_logprobs: policy.cpp:210-233 --------------------------------- */
int32_t orc_forward_logprobs(const void* logits, int32_t dtype, int32_t V, int64_t row_stride,
                             int32_t B, int32_t T, const int32_t* lengths, const int32_t* tokens,
                             double* out_lp, double* out_entropy, double* out_tok_logit,
                             char* err, int32_t errlen) {
  double* z = (double*)malloc(sizeof(double) * (size_t)(V > 0 ? V : 1));
  for (int32_t b = 0; b < B; ++b) {
    const int32_t n = lengths[b];
    for (int32_t t = 0; t < T; ++t) {
      const int64_t i = (int64_t)b * T + t;
      if (out_lp) out_lp[i] = 0.0;
      if (out_entropy) out_entropy[i] = 0.0;
      if (out_tok_logit) out_tok_logit[i] = 0.0;
      if (t >= n) continue;
      const int32_t tok = tokens[i];
      if (tok < 0 || tok >= V) { /* policy.cpp:224-225 */
        free(z);
        return fail(err, errlen, RLO_ERR_INPUT, "forward_logprobs: out-of-vocabulary token %d", tok);
      }
      load_row(logits, dtype, i * row_stride, V, z);
      double lse, h;
      orc_logsoftmax_row(z, V, &lse, out_entropy ? &h : NULL);
      out_lp[i] = z[tok] - lse; /* ws.logp[tok] = logits[tok] - lse, policy.cpp:122/227 */
      if (out_entropy) out_entropy[i] = h;
      if (out_tok_logit) out_tok_logit[i] = z[tok];
    }
  }
  free(z);
  return RLO_OK;
}

/* ---- compute_advantages: policy.cpp:257-311 (+ GRPO, GAE) ------------------ */
int32_t orc_compute_advantages(const rlo_train_config* cfg, int32_t B, int32_t T,
                               const int32_t* lengths, const uint8_t* mask,
                               const double* rewards_tok, const double* rewards_seq,
                               const double* values, double* out_adv, double* out_returns,
                               char* err, int32_t errlen) {
  const int64_t N = (int64_t)B * T;
  for (int64_t i = 0; i < N; ++i) {
    out_adv[i] = 0.0;
    if (out_returns) out_returns[i] = 0.0;
  }
  const double rc = cfg->reward_clip;
  double* r = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1));

  if (cfg->adv_estimator == RLO_ADV_GRPO) {
    const int32_t G = cfg->group_size;
    if (G <= 0 || B % G != 0) {
      free(r);
      return fail(err, errlen, RLO_ERR_INPUT, "compute_advantages: batch of %d samples is not whole groups of %d", B, G);
    }
    if (!rewards_seq && !rewards_tok && B > 0) {
      free(r);
      return fail(err, errlen, RLO_ERR_INPUT, "compute_advantages: sample '0' has no rewards");
    }
    double* R = (double*)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1));
    for (int32_t b = 0; b < B; ++b) {
      double x;
      if (rewards_seq) {
        x = rewards_seq[b];
      } else {
        x = 0.0;
        for (int32_t t = 0; t < lengths[b]; ++t) x += rewards_tok[(int64_t)b * T + t];
      }
      R[b] = clampd(x, -rc, rc);
    }
    for (int32_t g0 = 0; g0 < B; g0 += G) {
      double mean = 0.0;
      for (int32_t k = 0; k < G; ++k) mean += R[g0 + k];
      mean /= (double)G;
      double ss = 0.0;
      for (int32_t k = 0; k < G; ++k) ss += (R[g0 + k] - mean) * (R[g0 + k] - mean);
      const int32_t dof = G - cfg->grpo_std_ddof;
      const double sd = dof > 0 ? sqrt(ss / (double)dof) : 0.0;
      for (int32_t k = 0; k < G; ++k) {
        const int32_t b = g0 + k;
        const double a = (R[b] - mean) / (sd + cfg->grpo_eps);
        for (int32_t t = 0; t < lengths[b]; ++t) {
          out_adv[(int64_t)b * T + t] = a;
          if (out_returns) out_returns[(int64_t)b * T + t] = R[b];
        }
      }
    }
    free(R);
  } else {
    for (int32_t b = 0; b < B; ++b) {
      const int32_t n = lengths[b];
      /* reward source, policy.cpp:265-276 */
      if (rewards_tok) {
        for (int32_t t = 0; t < n; ++t) r[t] = rewards_tok[(int64_t)b * T + t];
      } else if (rewards_seq && n > 0) {
        for (int32_t t = 0; t < n; ++t) r[t] = 0.0;
        r[n - 1] = rewards_seq[b];
      } else if (n == 0) {
        continue;
      } else {
        free(r);
        return fail(err, errlen, RLO_ERR_INPUT, "compute_advantages: sample '%d' has no rewards", b);
      }
      for (int32_t t = 0; t < n; ++t) r[t] = clampd(r[t], -rc, rc); /* policy.cpp:277 */
      double* a = out_adv + (int64_t)b * T;
      if (cfg->adv_estimator == RLO_ADV_REINFORCE) {
        double acc = 0.0; /* policy.cpp:279-283 */
        for (int32_t t = n; t-- > 0;) {
          acc = r[t] + cfg->gamma * acc;
          a[t] = acc;
          if (out_returns) out_returns[(int64_t)b * T + t] = acc;
        }
      } else { /* GAE */
        if (!values) {
          free(r);
          return fail(err, errlen, RLO_ERR_INPUT, "compute_advantages: GAE requires critic values");
        }
        const double* vv = values + (int64_t)b * T;
        const double gl = cfg->gamma * cfg->lambd;
        double acc = 0.0;
        for (int32_t t = n; t-- > 0;) {
          const double next_v = (t + 1 < n) ? vv[t + 1] : 0.0;
          const double delta = r[t] + cfg->gamma * next_v - vv[t];
          acc = delta + gl * acc;
          a[t] = acc;
          if (out_returns) out_returns[(int64_t)b * T + t] = acc + vv[t];
        }
      }
    }
  }
  free(r);

  if (cfg->whiten_advantages) { /* policy.cpp:287-306 */
    double sum = 0.0, sq = 0.0;
    int64_t count = 0;
    for (int32_t b = 0; b < B; ++b)
      for (int32_t t = 0; t < lengths[b]; ++t) {
        const int64_t i = (int64_t)b * T + t;
        if (!mask_at(mask, i)) continue;
        sum += out_adv[i];
        sq += out_adv[i] * out_adv[i];
        ++count;
      }
    if (count > 0) {
      const double mean = sum / (double)count;
      const double var = fmax(0.0, sq / (double)count - mean * mean);
      const double inv = 1.0 / (sqrt(var) + 1e-8);
      for (int32_t b = 0; b < B; ++b)
        for (int32_t t = 0; t < lengths[b]; ++t) {
          const int64_t i = (int64_t)b * T + t;
          out_adv[i] = (out_adv[i] - mean) * inv;
        }
    }
  }
  for (int32_t b = 0; b < B; ++b) /* policy.cpp:308-309 */
    for (int32_t t = 0; t < lengths[b]; ++t) {
      const int64_t i = (int64_t)b * T + t;
      out_adv[i] = clampd(out_adv[i], -cfg->advantage_clip, cfg->advantage_clip);
    }
  return RLO_OK;
}

/* ---- ppo_gradient loss part: policy.cpp:335-374 ---------------------------- */
int32_t orc_ppo_loss(const rlo_train_config* cfg, int32_t B, int32_t T, const int32_t* lengths,
                     const uint8_t* mask, const double* lp, const double* old_lp,
                     const double* ref_lp, const double* adv, const double* entropy,
                     double* out_loss_tok, double* out_dlogp, rlo_partials* out_partials,
                     char* err, int32_t errlen) {
  rlo_partials P;
  memset(&P, 0, sizeof(P));
  const double eps = cfg->clip_eps, kc = cfg->kl_coef;
  const int32_t G = cfg->group_size > 0 ? cfg->group_size : 1;
  double group_loss = 0.0;
  int64_t group_tokens = 0;
  const int64_t N = (int64_t)B * T;
  for (int64_t i = 0; i < N; ++i) {
    if (out_loss_tok) out_loss_tok[i] = 0.0;
    if (out_dlogp) out_dlogp[i] = 0.0;
  }
  for (int32_t b = 0; b < B; ++b) {
    const int32_t n = lengths[b];
    if (n > 0) { /* policy.cpp:336-343 */
      if (!adv) return fail(err, errlen, RLO_ERR_INPUT, "ppo_gradient: sample '%d' missing advantages", b);
      if (!old_lp) return fail(err, errlen, RLO_ERR_INPUT, "ppo_gradient: sample '%d' missing old logprobs", b);
      if (kc > 0.0 && !ref_lp) return fail(err, errlen, RLO_ERR_INPUT, "ppo_gradient: sample '%d' missing ref logprobs", b);
    }
    double seq_loss = 0.0;
    int64_t seq_tokens = 0;
    for (int32_t t = 0; t < n; ++t) {
      const int64_t i = (int64_t)b * T + t;
      if (!mask_at(mask, i)) continue; /* policy.cpp:348-351 */
      const double A = adv[i];
      const double ratio = exp(lp[i] - old_lp[i]);
      const double rcl = clampd(ratio, 1.0 - eps, 1.0 + eps);
      const double unclipped = ratio * A, clipped = rcl * A;
      const double surrogate = (clipped < unclipped) ? clipped : unclipped; /* std::min, :362 */
      double pg = -surrogate;
      int dual = 0;
      if (cfg->dual_clip_c > 1.0 && A < 0.0) { /* extension: dual-clip */
        const double cap = -cfg->dual_clip_c * A;
        if (pg > cap) {
          pg = cap;
          dual = 1;
        }
      }
      double k = 0.0, dk = 0.0;
      if (ref_lp) {
        const double rr = lp[i] - ref_lp[i];
        if (cfg->kl_estimator == RLO_KL_K2) {
          k = 0.5 * rr * rr;
          dk = rr;
        } else if (cfg->kl_estimator == RLO_KL_K3) {
          k = exp(-rr) - 1.0 + rr;
          dk = 1.0 - exp(-rr);
        } else {
          k = rr;
          dk = 1.0;
        }
      }
      const double kl_term = kc > 0.0 ? k : 0.0; /* policy.cpp:364-365 */
      const double loss_t = pg + kc * kl_term;   /* policy.cpp:366 */
      P.v[RLO_P_LOSS_SUM] += loss_t;
      P.v[RLO_P_RATIO_SUM] += ratio; /* :367 */
      if (ref_lp) P.v[RLO_P_KL_SUM] += k; /* :368 */
      if (unclipped > clipped) P.v[RLO_P_CLIPPED] += 1.0; /* :369 */
      P.v[RLO_P_DUAL_CLIPPED] += dual;
      P.v[RLO_P_TOKENS] += 1.0; /* :370 */
      if (entropy) P.v[RLO_P_ENTROPY_SUM] += entropy[i];
      /* :372-374 d(loss_t)/d(logp[a]) */
      const int flows = A >= 0.0 ? ratio <= 1.0 + eps : ratio >= 1.0 - eps;
      double dlp = (flows && !dual) ? -ratio * A : 0.0;
      dlp += kc > 0.0 ? kc * dk : 0.0;
      if (!isfinite(dlp)) P.v[RLO_P_NONFINITE_GRAD] += 1.0;
      if (!isfinite(loss_t)) P.v[RLO_P_NONFINITE_LOSS] += 1.0;
      if (out_loss_tok) out_loss_tok[i] = loss_t;
      if (out_dlogp) out_dlogp[i] = dlp;
      seq_loss += loss_t;
      ++seq_tokens;
    }
    if (seq_tokens > 0) {
      P.v[RLO_P_SEQ_MEAN_SUM] += seq_loss / (double)seq_tokens;
      P.v[RLO_P_SEQS] += 1.0;
    }
    group_loss += seq_loss;
    group_tokens += seq_tokens;
    if (b % G == G - 1 || b == B - 1) {
      if (group_tokens > 0) {
        P.v[RLO_P_GROUP_MEAN_SUM] += group_loss / (double)group_tokens;
        P.v[RLO_P_GROUPS] += 1.0;
      }
      group_loss = 0.0;
      group_tokens = 0;
    }
  }
  if (out_partials) *out_partials = P;
  return RLO_OK;
}

/* ---- merge_gradients: policy.cpp:421-450 ----------------------------------- */
int32_t orc_merge(const rlo_partials* parts, int32_t nranks, const rlo_train_config* cfg,
                  rlo_stats* out, char* err, int32_t errlen) {
  if (nranks <= 0) return fail(err, errlen, RLO_ERR_TRAINING, "merge_gradients: no gradient parts");
  double s[RLO_NPARTIAL];
  memset(s, 0, sizeof(s));
  for (int32_t r = 0; r < nranks; ++r) /* rank order, policy.cpp:428-436 */
    for (int k = 0; k < RLO_NPARTIAL; ++k) s[k] += parts[r].v[k];
  if (s[RLO_P_TOKENS] == 0.0) /* :437 */
    return fail(err, errlen, RLO_ERR_TRAINING, "merge_gradients: batch contains no loss-participating tokens");
  if (s[RLO_P_NONFINITE_GRAD] > 0.0) /* :439-442 */
    return fail(err, errlen, RLO_ERR_TRAINING, "training step aborted: non-finite gradient");
  const double inv = 1.0 / s[RLO_P_TOKENS];
  memset(out, 0, sizeof(*out));
  switch (cfg->loss_agg) {
    case RLO_AGG_SEQ_MEAN_TOKEN_MEAN: out->loss = s[RLO_P_SEQ_MEAN_SUM] * (1.0 / s[RLO_P_SEQS]); break;
    case RLO_AGG_SEQ_MEAN_TOKEN_SUM: out->loss = s[RLO_P_LOSS_SUM] * (1.0 / s[RLO_P_SEQS]); break;
    case RLO_AGG_GROUP_MEAN: out->loss = s[RLO_P_GROUP_MEAN_SUM] * (1.0 / s[RLO_P_GROUPS]); break;
    default: out->loss = s[RLO_P_LOSS_SUM] * inv; break; /* :443 */
  }
  out->mean_ratio = s[RLO_P_RATIO_SUM] * inv;                     /* :444 */
  out->clip_fraction = s[RLO_P_CLIPPED] * inv;                    /* :445 */
  out->mean_kl = s[RLO_P_KL_SUM] * inv;                           /* :446 */
  out->tokens = (uint64_t)s[RLO_P_TOKENS];                        /* :447 */
  out->mean_entropy = s[RLO_P_ENTROPY_SUM] * inv;
  out->dual_clip_fraction = s[RLO_P_DUAL_CLIPPED] * inv;
  out->seqs = (uint64_t)s[RLO_P_SEQS];
  out->groups = (uint64_t)s[RLO_P_GROUPS];
  if (!isfinite(out->loss)) /* :448 */
    return fail(err, errlen, RLO_ERR_TRAINING, "training step aborted: non-finite loss");
  return RLO_OK;
}

void orc_split_sizes(int64_t n, int32_t parts, int64_t* out) { /* sample.cpp:99-105 */
  for (int32_t p = 0; p < parts; ++p) out[p] = n / parts;
  for (int64_t i = 0; i < n % parts; ++i) ++out[i];
}

/* ---- aggregation weights, actor backward, value loss ------------------------ */
void orc_loss_weights(const rlo_train_config* cfg, int32_t B, int32_t T, const int32_t* lengths,
                      const uint8_t* mask, double* out_w) {
  const int32_t G = cfg->group_size > 0 ? cfg->group_size : 1;
  double tokens = 0.0, seqs = 0.0, groups = 0.0;
  double* m = (double*)calloc((size_t)(B > 0 ? B : 1), sizeof(double));
  for (int32_t b = 0; b < B; ++b) {
    for (int32_t t = 0; t < lengths[b]; ++t) m[b] += mask_at(mask, (int64_t)b * T + t) ? 1.0 : 0.0;
    tokens += m[b];
    seqs += m[b] > 0.0;
  }
  double* M = (double*)calloc((size_t)(B / G + 2), sizeof(double));
  for (int32_t b = 0; b < B; ++b) M[b / G] += m[b];
  for (int32_t g = 0; g * G < B; ++g) groups += M[g] > 0.0;
  for (int32_t b = 0; b < B; ++b)
    for (int32_t t = 0; t < T; ++t) {
      const int64_t i = (int64_t)b * T + t;
      double w = 0.0;
      if (t < lengths[b] && mask_at(mask, i)) {
        switch (cfg->loss_agg) {
          case RLO_AGG_SEQ_MEAN_TOKEN_MEAN: w = 1.0 / (seqs * m[b]); break;
          case RLO_AGG_SEQ_MEAN_TOKEN_SUM: w = 1.0 / seqs; break;
          case RLO_AGG_GROUP_MEAN: w = 1.0 / (groups * M[b / G]); break;
          default: w = 1.0 / tokens; break;
        }
      }
      out_w[i] = w;
    }
  free(m);
  free(M);
}

void orc_logits_backward_row(const double* z, int32_t V, int32_t tok, double scale, double* out) {
  double lse;
  orc_logsoftmax_row(z, V, &lse, NULL);
  for (int32_t v = 0; v < V; ++v) out[v] = scale * ((v == tok ? 1.0 : 0.0) - exp(z[v] - lse));
}

void orc_value_loss(int32_t B, int32_t T, const int32_t* lengths, const uint8_t* mask, const double* values,
                    const double* old_values, const double* returns, double value_clip, double* out_dv,
                    double* out4) {
  double loss = 0.0, tokens = 0.0, clipped = 0.0, vsum = 0.0;
  for (int64_t i = 0; i < (int64_t)B * T; ++i) out_dv[i] = 0.0;
  for (int32_t b = 0; b < B; ++b)
    for (int32_t t = 0; t < lengths[b]; ++t) {
      const int64_t i = (int64_t)b * T + t;
      if (!mask_at(mask, i)) continue; /* policy.cpp:501-504 */
      const double v = values[i], R = returns[i];
      const double err = v - R; /* :508 */
      double l = 0.5 * err * err, d = err;
      if (old_values && value_clip > 0.0) {
        const double dv = v - old_values[i];
        const double vc = old_values[i] + clampd(dv, -value_clip, value_clip);
        const double errc = vc - R;
        const double lc = 0.5 * errc * errc;
        if (lc > l) {
          l = lc;
          d = (dv > -value_clip && dv < value_clip) ? errc : 0.0;
          clipped += 1.0;
        }
      }
      loss += l; /* :509 */
      tokens += 1.0; /* :510 */
      vsum += v;
      out_dv[i] = d; /* :512 */
    }
  out4[0] = loss;
  out4[1] = tokens;
  out4[2] = clipped;
  out4[3] = vsum;
}

/* ---- decode_next: policy.cpp:143-169 --------------------------------------- */
static uint64_t orc_splitmix(uint64_t* state) { /* rng.hpp:15-20 */
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

int32_t orc_decode_next(const double* z, int32_t V, double temperature, uint64_t seed, uint64_t version,
                        uint64_t sample_key, uint64_t position, double* logp) {
  double m = z[0];
  for (int32_t v = 1; v < V; ++v) m = (m < z[v]) ? z[v] : m; /* :151-152 */
  double* probs = (double*)malloc(sizeof(double) * (size_t)V);
  double total = 0.0;
  for (int32_t v = 0; v < V; ++v) { /* :153-157 */
    probs[v] = exp((z[v] - m) / temperature);
    total += probs[v];
  }
  /* keyed_double({seed, version, sample_key, position}), rng.hpp:23-31, 83-85 */
  uint64_t state = 0x2545f4914f6cdd1dULL;
  uint64_t h = orc_splitmix(&state);
  const uint64_t keys[4] = {seed, version, sample_key, position};
  for (int k = 0; k < 4; ++k) {
    state ^= keys[k];
    h ^= orc_splitmix(&state);
  }
  const double u = (double)(h >> 11) * 0x1.0p-53;
  double acc = 0.0;
  int32_t chosen = V - 1; /* :159-167 */
  for (int32_t v = 0; v < V; ++v) {
    acc += probs[v] / total;
    if (u < acc) {
      chosen = v;
      break;
    }
  }
  free(probs);
  double lse;
  orc_logsoftmax_row(z, V, &lse, NULL);
  *logp = z[chosen] - lse; /* :168, untempered */
  return chosen;
}

uint64_t orc_hash_str(const char* s) { /* rng.hpp:34-41 */
  uint64_t h = 0xcbf29ce484222325ULL;
  for (const unsigned char* c = (const unsigned char*)s; *c; ++c) {
    h ^= *c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ---- synthetic inputs (include/rlo_synth.h) -------------------------------- */
static void synth_row_f(float* out, int32_t V, uint64_t seed, int32_t model, uint64_t row_key) {
  int32_t spikes[RLO_SYNTH_SPIKES];
  for (int k = 0; k < RLO_SYNTH_SPIKES; ++k) spikes[k] = rlo_synth_spike(seed, row_key, k, V);
  const uint64_t k0 = rlo_synth_model_key(seed, 0), km = rlo_synth_model_key(seed, model);
  for (int32_t v = 0; v < V; ++v) out[v] = rlo_synth_logit(k0, km, model, row_key, v, spikes);
}

void orc_synth_row_raw(void* out, int32_t dtype, int32_t V, uint64_t seed, int32_t model, uint64_t row_key) {
  if (dtype == RLO_DTYPE_F32) {
    synth_row_f((float*)out, V, seed, model, row_key);
  } else {
    float* tmp = (float*)malloc(sizeof(float) * (size_t)V);
    synth_row_f(tmp, V, seed, model, row_key);
    uint16_t* o = (uint16_t*)out;
    for (int32_t v = 0; v < V; ++v) o[v] = rlo_f32_to_bf16_rne(tmp[v]);
    free(tmp);
  }
}

void orc_synth_row(double* out, int32_t dtype, int32_t V, uint64_t seed, int32_t model, uint64_t row_key) {
  float* tmp = (float*)malloc(sizeof(float) * (size_t)V);
  synth_row_f(tmp, V, seed, model, row_key);
  for (int32_t v = 0; v < V; ++v)
    out[v] = dtype == RLO_DTYPE_F32 ? (double)tmp[v] : (double)rlo_bf16_to_f32(rlo_f32_to_bf16_rne(tmp[v]));
  free(tmp);
}

int32_t orc_synth_token(uint64_t seed, uint64_t row_key, int32_t V) { return rlo_synth_token(seed, row_key, V); }

/* ---- "port" CPU baseline ---------------------------------------------------- */
typedef struct {
  const rlo_train_config* cfg;
  int32_t dtype, V, T, key_rows, b0, b1;
  const int32_t* lengths;
  const int32_t* tokens;
  const void* rows[3];
  double *lp, *old, *ref, *ent;
} bench_job;

static void* bench_logprob_worker(void* arg) {
  bench_job* j = (bench_job*)arg;
  double* z = (double*)malloc(sizeof(double) * (size_t)j->V);
  const size_t esz = j->dtype == RLO_DTYPE_F32 ? 4 : 2;
  for (int32_t b = j->b0; b < j->b1; ++b)
    for (int32_t t = 0; t < j->lengths[b]; ++t) {
      const int64_t i = (int64_t)b * j->T + t;
      const int64_t key = i % j->key_rows;
      const int32_t tok = j->tokens[i];
      double* outs[3] = {j->lp, j->old, j->ref};
      for (int m = 0; m < 3; ++m) {
        const char* base = (const char*)j->rows[m] + (size_t)key * (size_t)j->V * esz;
        load_row(base, j->dtype, 0, j->V, z);
        double lse, h;
        orc_logsoftmax_row(z, j->V, &lse, m == 0 ? &h : NULL);
        outs[m][i] = z[tok] - lse;
        if (m == 0) j->ent[i] = h;
      }
    }
  free(z);
  return NULL;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

double orc_bench_objective(int32_t threads, const rlo_train_config* cfg, int32_t dtype, int32_t V,
                           int32_t B, int32_t T, int32_t key_rows, uint64_t seed, double* checksum) {
  const size_t esz = dtype == RLO_DTYPE_F32 ? 4 : 2;
  const int64_t N = (int64_t)B * T;
  void* rows[3];
  for (int m = 0; m < 3; ++m) {
    rows[m] = malloc((size_t)key_rows * (size_t)V * esz);
    for (int64_t k = 0; k < key_rows; ++k)
      orc_synth_row_raw((char*)rows[m] + (size_t)k * (size_t)V * esz, dtype, V, seed, m, (uint64_t)k);
  }
  int32_t* lengths = (int32_t*)malloc(sizeof(int32_t) * (size_t)B);
  int32_t* tokens = (int32_t*)malloc(sizeof(int32_t) * (size_t)N);
  double* rw = (double*)malloc(sizeof(double) * (size_t)B);
  double* vals = (double*)malloc(sizeof(double) * (size_t)N);
  for (int32_t b = 0; b < B; ++b) {
    lengths[b] = T;
    rw[b] = (double)(rlo_sm64(seed ^ (0xBEEF0000ULL + (uint64_t)b)) & 1u);
  }
  for (int64_t i = 0; i < N; ++i) {
    tokens[i] = rlo_synth_token(seed, (uint64_t)(i % key_rows), V);
    vals[i] = 0.5 * ((double)(rlo_sm64(seed ^ 0x7A1ULL ^ (uint64_t)i) >> 11) * 0x1.0p-53 - 0.5);
  }
  double* lp = (double*)calloc((size_t)N, sizeof(double));
  double* old = (double*)calloc((size_t)N, sizeof(double));
  double* ref = (double*)calloc((size_t)N, sizeof(double));
  double* ent = (double*)calloc((size_t)N, sizeof(double));
  double* adv = (double*)calloc((size_t)N, sizeof(double));
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  bench_job* jobs = (bench_job*)malloc(sizeof(bench_job) * (size_t)threads);
  int64_t* sizes = (int64_t*)malloc(sizeof(int64_t) * (size_t)threads);
  orc_split_sizes(B, threads, sizes);

  const double t0 = now_s();
  int32_t off = 0;
  for (int32_t k = 0; k < threads; ++k) {
    bench_job j = {cfg, dtype, V, T, key_rows, off, off + (int32_t)sizes[k], lengths, tokens,
                   {rows[0], rows[1], rows[2]}, lp, old, ref, ent};
    jobs[k] = j;
    off += (int32_t)sizes[k];
    pthread_create(&th[k], NULL, bench_logprob_worker, &jobs[k]);
  }
  for (int32_t k = 0; k < threads; ++k) pthread_join(th[k], NULL);
  const int gae = cfg->adv_estimator == RLO_ADV_GAE;
  orc_compute_advantages(cfg, B, T, lengths, NULL, NULL, rw, gae ? vals : NULL, adv, NULL, NULL, 0);
  rlo_partials part;
  orc_ppo_loss(cfg, B, T, lengths, NULL, lp, old, ref, adv, ent, NULL, NULL, &part, NULL, 0);
  rlo_stats st;
  orc_merge(&part, 1, cfg, &st, NULL, 0);
  const double elapsed = now_s() - t0;
  if (checksum) *checksum = st.loss;

  for (int m = 0; m < 3; ++m) free(rows[m]);
  free(lengths); free(tokens); free(rw); free(vals);
  free(lp); free(old); free(ref); free(ent); free(adv);
  free(th); free(jobs); free(sizes);
  return elapsed;
}
