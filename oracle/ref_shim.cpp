// ref_shim.cpp — extern "C" shim over the reference's OWN code (rollmini core,
// compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/librollmini_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used to (1) pin the oracle restatement and
// generate tests/golden/ fixtures (tests/golden/make_golden.py), and (2) time
// the reference's CPU path for bench.py --impl reference / cpu_baseline.
// No reference source is copied here; this file only calls the reference's
// public functions (include/rollmini/policy.hpp).
//
// The "b2 trick": PolicyLayout{V,1,1,1} with every parameter
// 0 except b2 := a logits row makes the reference's head produce exactly that
// row (trunk h = tanh(0) = 0, logits = b2 + 0*w2), so next_token_forward
// (policy.cpp:127-131) runs the reference log-softmax (policy.cpp:116-122) on
// an arbitrary row bit-for-bit.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rollmini/errors.hpp"
#include "rollmini/policy.hpp"
#include "rollmini/rng.hpp"
#include "rollmini/sample.hpp"

extern "C" {
#include "oracle.h"
}
#include "../include/rlo_synth.h"

using namespace rollmini;

namespace {

int32_t report(char* err, int32_t errlen, int32_t code, const std::string& msg) {
  if (err && errlen > 0) std::snprintf(err, static_cast<size_t>(errlen), "%s", msg.c_str());
  return code;
}

template <class F>
int32_t guarded(char* err, int32_t errlen, F&& f) {
  try {
    f();
    return RLO_OK;
  } catch (const InputError& e) {
    return report(err, errlen, RLO_ERR_INPUT, e.what());
  } catch (const ConfigError& e) {
    return report(err, errlen, RLO_ERR_CONFIG, e.what());
  } catch (const TrainingError& e) {
    return report(err, errlen, RLO_ERR_TRAINING, e.what());
  } catch (const std::exception& e) {
    return report(err, errlen, 99, e.what());
  }
}

PolicyParams b2_params(int32_t V) {
  PolicyParams p;
  p.layout = PolicyLayout{V, 1, 1, 1};
  p.version = 1;
  p.values.assign(p.layout.param_count(), 0.0);
  return p;
}

TrainConfig to_ref(const rlo_train_config* c) {
  TrainConfig t;
  t.clip_eps = c->clip_eps;
  t.kl_coef = c->kl_coef;
  t.learning_rate = c->learning_rate;
  t.advantage_clip = c->advantage_clip;
  t.reward_clip = c->reward_clip;
  t.gamma = c->gamma;
  t.whiten_advantages = c->whiten_advantages != 0;
  return t;
}

SampleBatch make_batch(int32_t B, int32_t T, const int32_t* lengths, const int32_t* tokens,
                       const uint8_t* mask, const double* rewards_tok, const double* rewards_seq,
                       const double* old_lp, const double* ref_lp, const double* adv) {
  SampleBatch batch;
  for (int32_t b = 0; b < B; ++b) {
    SampleRecord r;
    r.sample_id = std::to_string(b);
    r.prompt_tokens = {1};
    const int32_t n = lengths[b];
    const size_t base = static_cast<size_t>(b) * static_cast<size_t>(T);
    for (int32_t t = 0; t < n; ++t) r.response_tokens.push_back(tokens ? tokens[base + t] : 1);
    if (mask) r.action_mask.assign(mask + base, mask + base + n);
    if (rewards_tok) r.rewards.assign(rewards_tok + base, rewards_tok + base + n);
    if (rewards_seq) r.scalar_reward = rewards_seq[b];
    if (old_lp) r.response_logprobs.assign(old_lp + base, old_lp + base + n);
    if (ref_lp) r.ref_logprobs.assign(ref_lp + base, ref_lp + base + n);
    if (adv) r.advantages.assign(adv + base, adv + base + n);
    batch.push_back(std::move(r));
  }
  return batch;
}

}  // namespace

extern "C" {

// Reference log-softmax on arbitrary rows: logp of toks[i] under row i, and
// optionally the full logp vector (policy.cpp:116-122 via next_token_forward).
int32_t ref_logsoftmax_rows(const double* rows, int32_t n_rows, int32_t V, const int32_t* toks,
                            double* out_lp, double* out_logp_full, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    PolicyParams p = b2_params(V);
    PolicyWorkspace ws;
    ws.resize(p.layout);
    const int ctx[1] = {0};
    for (int32_t i = 0; i < n_rows; ++i) {
      std::memcpy(p.values.data() + p.layout.off_b2(), rows + static_cast<size_t>(i) * V, sizeof(double) * V);
      next_token_forward(p, std::span<const int>(ctx, 1), kWindowPadToken, ws);
      out_lp[i] = ws.logp[static_cast<size_t>(toks[i])];
      if (out_logp_full) std::memcpy(out_logp_full + static_cast<size_t>(i) * V, ws.logp.data(), sizeof(double) * V);
    }
  });
}

// forward_logprobs itself (policy.cpp:210-233) on a batch whose every position
// shares one logits row (b2 trick): exercises the OOV check and batch walk.
int32_t ref_forward_logprobs_b2(const double* row, int32_t V, int32_t B, int32_t T, const int32_t* lengths,
                                const int32_t* tokens, double* out_lp, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    PolicyParams p = b2_params(V);
    std::memcpy(p.values.data() + p.layout.off_b2(), row, sizeof(double) * V);
    SampleBatch batch = make_batch(B, T, lengths, tokens, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    auto lps = forward_logprobs(p, batch);
    for (int32_t b = 0; b < B; ++b)
      for (int32_t t = 0; t < T; ++t)
        out_lp[static_cast<size_t>(b) * T + t] = t < lengths[b] ? lps[b][t] : 0.0;
  });
}

// compute_advantages (policy.cpp:257-311) on a padded batch.
int32_t ref_compute_advantages(const rlo_train_config* cfg, int32_t B, int32_t T, const int32_t* lengths,
                               const uint8_t* mask, const double* rewards_tok, const double* rewards_seq,
                               double* out_adv, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    SampleBatch batch = make_batch(B, T, lengths, nullptr, mask, rewards_tok, rewards_seq, nullptr, nullptr, nullptr);
    auto advs = compute_advantages(batch, to_ref(cfg));
    for (int32_t b = 0; b < B; ++b)
      for (int32_t t = 0; t < T; ++t)
        out_adv[static_cast<size_t>(b) * T + t] =
            t < static_cast<int32_t>(advs[b].size()) ? advs[b][static_cast<size_t>(t)] : 0.0;
  });
}

// ppo_gradient -> merge_gradients over `world` split_batch shards
// (policy.cpp:313-450, ppo_update's sharding policy.cpp:462-472) with every
// position's logits = `row` (b2 trick).  out5 = {loss, mean_ratio,
// clip_fraction, mean_kl, tokens}.
int32_t ref_ppo_stats_b2(const double* row, int32_t V, int32_t B, int32_t T, const int32_t* lengths,
                         const int32_t* tokens, const uint8_t* mask, const double* old_lp,
                         const double* ref_lp, const double* adv, const rlo_train_config* cfg,
                         int32_t world, double* out5, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    PolicyParams p = b2_params(V);
    std::memcpy(p.values.data() + p.layout.off_b2(), row, sizeof(double) * V);
    SampleBatch batch = make_batch(B, T, lengths, tokens, mask, nullptr, nullptr, old_lp, ref_lp, adv);
    auto shards = split_batch(batch, static_cast<size_t>(world));
    std::vector<GradAccum> parts;
    for (const auto& s : shards) parts.push_back(ppo_gradient(p, s, to_ref(cfg)));
    auto [grad, stats] = merge_gradients(parts);
    out5[0] = stats.loss;
    out5[1] = stats.mean_ratio;
    out5[2] = stats.clip_fraction;
    out5[3] = stats.mean_kl;
    out5[4] = static_cast<double>(stats.tokens);
  });
}

// The same ppo_gradient -> merge_gradients run, returning the merged
// gradient's b2 segment: with every position's logits = b2, d(loss)/d(b2) is
// the token-mean sum over tokens of dz = dlp * (onehot - softmax)
// (policy.cpp:375-379, :391, :439-440) — the actor backward epilogue.
int32_t ref_ppo_grad_b2(const double* row, int32_t V, int32_t B, int32_t T, const int32_t* lengths,
                        const int32_t* tokens, const uint8_t* mask, const double* old_lp, const double* ref_lp,
                        const double* adv, const rlo_train_config* cfg, int32_t world, double* out_grad_b2,
                        char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    PolicyParams p = b2_params(V);
    std::memcpy(p.values.data() + p.layout.off_b2(), row, sizeof(double) * V);
    SampleBatch batch = make_batch(B, T, lengths, tokens, mask, nullptr, nullptr, old_lp, ref_lp, adv);
    auto shards = split_batch(batch, static_cast<size_t>(world));
    std::vector<GradAccum> parts;
    for (const auto& s : shards) parts.push_back(ppo_gradient(p, s, to_ref(cfg)));
    auto [grad, stats] = merge_gradients(parts);
    std::memcpy(out_grad_b2, grad.data() + p.layout.off_b2(), sizeof(double) * V);
  });
}

// value_gradient (policy.cpp:474-540) with every position's value = vb
// (all parameters 0 except the value-head bias vb): out3 = {loss_sum, tokens,
// d(loss_sum)/d(vb) = sum of err}.
int32_t ref_value_loss_b2(double vb, int32_t B, int32_t T, const int32_t* lengths, const uint8_t* mask,
                          const double* targets, double* out3, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    PolicyParams p = b2_params(4);
    p.values[p.layout.off_vb()] = vb;
    SampleBatch batch = make_batch(B, T, lengths, nullptr, mask, nullptr, nullptr, nullptr, nullptr, targets);
    GradAccum acc = value_gradient(p, batch);
    out3[0] = acc.loss_sum;
    out3[1] = static_cast<double>(acc.tokens);
    out3[2] = acc.grad[p.layout.off_vb()];
  });
}

// decode_next itself (policy.cpp:143-169) on an arbitrary row (b2 trick),
// with params.version = `version`.
int32_t ref_decode_b2(const double* row, int32_t V, double temperature, uint64_t seed, uint64_t version,
                      uint64_t sample_key, uint64_t position, int32_t* out_tok, double* out_lp, char* err,
                      int32_t errlen) {
  return guarded(err, errlen, [&] {
    PolicyParams p = b2_params(V);
    p.version = version;
    std::memcpy(p.values.data() + p.layout.off_b2(), row, sizeof(double) * V);
    PolicyWorkspace ws;
    ws.resize(p.layout);
    const int ctx[1] = {0};
    DecodeStep ds = decode_next(p, std::span<const int>(ctx, 1), temperature, seed, sample_key,
                                static_cast<size_t>(position), kWindowPadToken, ws);
    *out_tok = ds.token;
    *out_lp = ds.logprob;
  });
}

uint64_t ref_hash_str(const char* s) { return rng::hash_str(s); }

// SampleBatch::to_jsonl (sample.cpp:144-148) of a random batch exercising every
// field and presence pattern; returns the text length (writes up to cap bytes).
int64_t ref_batch_jsonl(uint64_t seed, int32_t n, char* out, int64_t cap) {
  rng::Stream s(seed);
  SampleBatch batch;
  for (int32_t i = 0; i < n; ++i) {
    SampleRecord r;
    r.sample_id = "s" + std::to_string(i) + (i % 5 == 0 ? "\"q\\u\t\xc3\xa9" : "");
    r.group_id = "g" + std::to_string(i / 3);
    r.domain_tag = i % 2 ? "math" : "code";
    const size_t np = 1 + s.next_below(4), nr = s.next_below(7);
    for (size_t t = 0; t < np; ++t) r.prompt_tokens.push_back(static_cast<int>(s.next_below(52)));
    for (size_t t = 0; t < nr; ++t) r.response_tokens.push_back(static_cast<int>(s.next_below(52)));
    const uint64_t pat = s.next_below(64);
    for (size_t t = 0; t < nr; ++t) {
      if (pat & 1) r.response_logprobs.push_back(-3.0 * s.next_double());
      if (pat & 2) r.ref_logprobs.push_back(-3.0 * s.next_double() - 1e-7);
      if (pat & 4) r.rewards.push_back(s.next_double() < 0.8 ? 0.0 : 2.0 * s.next_double() - 1.0);
      if (pat & 8) r.advantages.push_back(s.next_gaussian());
      if (pat & 16) r.action_mask.push_back(s.next_double() < 0.7 ? 1 : 0);
    }
    if (pat & 32) r.scalar_reward = s.next_double() * 3.0 - 1.0;
    r.done = (pat & 1) != 0;
    if (i % 4 == 0) r.meta["gold"] = std::to_string(i);
    batch.push_back(std::move(r));
  }
  const std::string text = batch.to_jsonl();
  if (out && cap > 0) std::memcpy(out, text.data(), std::min<size_t>(text.size(), static_cast<size_t>(cap)));
  return static_cast<int64_t>(text.size());
}

// SampleBatch::from_jsonl + validate (sample.cpp:85-102, 150-158) on `text`.
int32_t ref_parse_validate_jsonl(const char* text, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] { SampleBatch::from_jsonl(text).validate(); });
}

void ref_bucket_plan(uint64_t total, uint64_t bucket, uint64_t* out, int64_t* n) {
  auto p = bucket_plan(static_cast<size_t>(total), static_cast<size_t>(bucket));
  *n = static_cast<int64_t>(p.size());
  for (size_t i = 0; i < p.size(); ++i) out[i] = p[i];
}

// merge_gradients (policy.cpp:421-450) on scalar partials with empty grads.
int32_t ref_merge_scalars(const double* parts5, int32_t nranks, double* out5, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] {
    std::vector<GradAccum> parts(static_cast<size_t>(nranks));
    for (int32_t r = 0; r < nranks; ++r) {
      parts[r].loss_sum = parts5[r * 5 + 0];
      parts[r].ratio_sum = parts5[r * 5 + 1];
      parts[r].kl_sum = parts5[r * 5 + 2];
      parts[r].clipped = static_cast<size_t>(parts5[r * 5 + 3]);
      parts[r].tokens = static_cast<size_t>(parts5[r * 5 + 4]);
    }
    auto [grad, stats] = merge_gradients(parts);
    out5[0] = stats.loss;
    out5[1] = stats.mean_ratio;
    out5[2] = stats.clip_fraction;
    out5[3] = stats.mean_kl;
    out5[4] = static_cast<double>(stats.tokens);
  });
}

int32_t ref_train_config_validate(const rlo_train_config* cfg, char* err, int32_t errlen) {
  return guarded(err, errlen, [&] { to_ref(cfg).validate(); });
}

void ref_split_sizes(int64_t n, int32_t parts, int64_t* out) {
  auto s = split_sizes(static_cast<size_t>(n), static_cast<size_t>(parts));
  for (int32_t i = 0; i < parts; ++i) out[i] = static_cast<int64_t>(s[static_cast<size_t>(i)]);
}

// The reference's CPU path for the bench's --impl reference arm: per token,
// the reference log-softmax (next_token_forward, b2 trick) over the actor,
// old-policy and reference rows; advantages via the reference
// compute_advantages (REINFORCE; GRPO/GAE are absent from the reference and
// fall back to the oracle restatement); the loss arithmetic restated from
// policy.cpp:355-370; merge via the reference merge_gradients.  Threads:
// contiguous sequence ranges, one std::thread each (cluster.cpp:146).
// Synthetic rows are generated before the clock starts.
double ref_bench_objective(int32_t threads, const rlo_train_config* cfg, int32_t dtype, int32_t V, int32_t B,
                           int32_t T, int32_t key_rows, uint64_t seed, double* checksum) {
  const size_t N = static_cast<size_t>(B) * T;
  std::vector<std::vector<double>> rows(3, std::vector<double>(static_cast<size_t>(key_rows) * V));
  for (int m = 0; m < 3; ++m)
    for (int32_t k = 0; k < key_rows; ++k)
      orc_synth_row(rows[m].data() + static_cast<size_t>(k) * V, dtype, V, seed, m, static_cast<uint64_t>(k));
  std::vector<int32_t> lengths(static_cast<size_t>(B), T), tokens(N);
  std::vector<double> rw(static_cast<size_t>(B)), vals(N), lp(N), old(N), ref(N);
  for (int32_t b = 0; b < B; ++b) rw[b] = static_cast<double>(rlo_sm64(seed ^ (0xBEEF0000ULL + b)) & 1u);
  for (size_t i = 0; i < N; ++i) {
    tokens[i] = rlo_synth_token(seed, static_cast<uint64_t>(i % key_rows), V);
    vals[i] = 0.5 * (static_cast<double>(rlo_sm64(seed ^ 0x7A1ULL ^ i) >> 11) * 0x1.0p-53 - 0.5);
  }
  if (threads < 1) threads = 1;
  const auto sizes = split_sizes(static_cast<size_t>(B), static_cast<size_t>(threads));

  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  size_t off = 0;
  for (int32_t k = 0; k < threads; ++k) {
    const size_t b0 = off, b1 = off + sizes[static_cast<size_t>(k)];
    off = b1;
    pool.emplace_back([&, b0, b1] {
      PolicyParams p = b2_params(V);
      PolicyWorkspace ws;
      ws.resize(p.layout);
      const int ctx[1] = {0};
      double* outs[3] = {lp.data(), old.data(), ref.data()};
      for (size_t b = b0; b < b1; ++b)
        for (int32_t t = 0; t < T; ++t) {
          const size_t i = b * static_cast<size_t>(T) + t;
          const size_t key = i % static_cast<size_t>(key_rows);
          for (int m = 0; m < 3; ++m) {
            std::memcpy(p.values.data() + p.layout.off_b2(), rows[m].data() + key * V, sizeof(double) * V);
            next_token_forward(p, std::span<const int>(ctx, 1), kWindowPadToken, ws);
            outs[m][i] = ws.logp[static_cast<size_t>(tokens[i])];
          }
        }
    });
  }
  for (auto& th : pool) th.join();

  std::vector<double> adv(N);
  if (cfg->adv_estimator == RLO_ADV_REINFORCE) {
    SampleBatch batch = make_batch(B, T, lengths.data(), nullptr, nullptr, nullptr, rw.data(), nullptr, nullptr, nullptr);
    auto advs = compute_advantages(batch, to_ref(cfg));
    for (int32_t b = 0; b < B; ++b) std::memcpy(adv.data() + static_cast<size_t>(b) * T, advs[b].data(), sizeof(double) * T);
  } else {
    orc_compute_advantages(cfg, B, T, lengths.data(), nullptr, nullptr, rw.data(),
                           cfg->adv_estimator == RLO_ADV_GAE ? vals.data() : nullptr, adv.data(), nullptr, nullptr, 0);
  }
  GradAccum acc;  // policy.cpp:355-370 arithmetic, token order
  for (size_t i = 0; i < N; ++i) {
    const double ratio = std::exp(lp[i] - old[i]);
    const double rc = std::clamp(ratio, 1.0 - cfg->clip_eps, 1.0 + cfg->clip_eps);
    const double u = ratio * adv[i], c = rc * adv[i];
    const double kl = lp[i] - ref[i];
    acc.loss_sum += -std::min(u, c) + cfg->kl_coef * (cfg->kl_coef > 0.0 ? kl : 0.0);
    acc.ratio_sum += ratio;
    acc.kl_sum += kl;
    if (u > c) ++acc.clipped;
    ++acc.tokens;
  }
  auto merged = merge_gradients({acc});
  const double elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (checksum) *checksum = merged.second.loss;
  return elapsed;
}

}  // extern "C"
