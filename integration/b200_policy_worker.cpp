// b200_policy_worker.cpp — see b200_policy_worker.hpp.
#include "b200_policy_worker.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "rollmini/errors.hpp"

namespace rollmini_b200 {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw rollmini::Error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
auto translate(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const rlo::Error& e) {
    rethrow_as_rollmini(e);
  }
}

}  // namespace

[[noreturn]] void rethrow_as_rollmini(const rlo::Error& e) {
  if (dynamic_cast<const rlo::InputError*>(&e)) throw rollmini::InputError(e.what());
  if (dynamic_cast<const rlo::ConfigError*>(&e)) throw rollmini::ConfigError(e.what());
  if (dynamic_cast<const rlo::TrainingError*>(&e)) throw rollmini::TrainingError(e.what());
  if (dynamic_cast<const rlo::DispatchError*>(&e)) throw rollmini::DispatchError(e.what());
  if (dynamic_cast<const rlo::CollectError*>(&e)) throw rollmini::CollectError(e.what(), {});
  throw rollmini::Error(e.what());
}

rlo::TrainConfig to_rlo(const rollmini::TrainConfig& c) {
  rlo::TrainConfig t;  // extensions keep their reference-compatible defaults
  t.clip_eps = c.clip_eps;
  t.kl_coef = c.kl_coef;
  t.learning_rate = c.learning_rate;
  t.advantage_clip = c.advantage_clip;
  t.reward_clip = c.reward_clip;
  t.gamma = c.gamma;
  t.whiten_advantages = c.whiten_advantages ? 1 : 0;
  return t;
}

// ---- DeviceBatch --------------------------------------------------------------

DeviceBatch::~DeviceBatch() {
  for (void* p : owned_) cudaFree(p);
}

void* DeviceBatch::alloc(size_t bytes) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "DeviceBatch: cudaMalloc");
  owned_.push_back(p);
  return p;
}

float* DeviceBatch::scratch(size_t k) {
  if (!scratch_[k]) scratch_[k] = static_cast<float*>(alloc(sizeof(float) * static_cast<size_t>(B_) * T_));
  return scratch_[k];
}

void DeviceBatch::upload(const rollmini::SampleBatch& batch) {
  batch.validate();  // sample.cpp:85-102 invariants (InputError)
  B_ = static_cast<int32_t>(batch.size());
  T_ = 1;
  for (const auto& s : batch.samples) T_ = std::max<int32_t>(T_, static_cast<int32_t>(s.response_tokens.size()));
  const size_t N = static_cast<size_t>(B_) * T_;
  std::vector<int32_t> lengths(static_cast<size_t>(B_)), tokens(N, 0);
  std::vector<uint8_t> mask(N, 0);
  std::vector<float> old(N, 0.f), ref(N, 0.f), adv(N, 0.f), rtok(N, 0.f), rseq(static_cast<size_t>(B_), 0.f);
  for (int32_t b = 0; b < B_; ++b) {
    const auto& s = batch.samples[static_cast<size_t>(b)];
    const size_t n = s.response_tokens.size(), base = static_cast<size_t>(b) * T_;
    lengths[static_cast<size_t>(b)] = static_cast<int32_t>(n);
    for (size_t t = 0; t < n; ++t) {
      tokens[base + t] = s.response_tokens[t];
      mask[base + t] = s.mask_at(t) ? 1 : 0;
      if (!s.response_logprobs.empty()) old[base + t] = static_cast<float>(s.response_logprobs[t]);
      if (!s.ref_logprobs.empty()) ref[base + t] = static_cast<float>(s.ref_logprobs[t]);
      if (!s.advantages.empty()) adv[base + t] = static_cast<float>(s.advantages[t]);
      if (!s.rewards.empty()) rtok[base + t] = static_cast<float>(s.rewards[t]);
    }
    // policy.cpp:266-271: a sample without per-token rewards scores its
    // scalar_reward on the last response token
    if (s.rewards.empty() && s.scalar_reward && n > 0) rtok[base + n - 1] = static_cast<float>(*s.scalar_reward);
    if (s.scalar_reward) rseq[static_cast<size_t>(b)] = static_cast<float>(*s.scalar_reward);
    has_mask_ |= !s.action_mask.empty();
    has_old_ |= !s.response_logprobs.empty();
    has_ref_ |= !s.ref_logprobs.empty();
    has_adv_ |= !s.advantages.empty();
    has_rtok_ |= !s.rewards.empty();
    has_rseq_ |= s.scalar_reward.has_value();
  }
  auto up = [&](auto& dst, const auto& src) {
    using E = typename std::decay_t<decltype(src)>::value_type;
    dst = static_cast<std::remove_reference_t<decltype(dst)>>(alloc(sizeof(E) * src.size()));
    cuda_check(cudaMemcpy(dst, src.data(), sizeof(E) * src.size(), cudaMemcpyHostToDevice), "DeviceBatch: H2D");
  };
  up(lengths_, lengths);
  up(tokens_, tokens);
  up(mask_, mask);
  up(old_, old);
  up(ref_, ref);
  up(adv_, adv);
  up(rtok_, rtok);
  up(rseq_, rseq);
}

rlo_batch DeviceBatch::view() const { return rlo_batch{B_, T_, 0, 0, lengths_, tokens_, has_mask_ ? mask_ : nullptr}; }

std::vector<std::vector<double>> DeviceBatch::download(const float* dev, const rollmini::SampleBatch& batch) const {
  std::vector<float> host(static_cast<size_t>(B_) * T_);
  cuda_check(cudaMemcpy(host.data(), dev, sizeof(float) * host.size(), cudaMemcpyDeviceToHost), "DeviceBatch: D2H");
  std::vector<std::vector<double>> out;
  for (int32_t b = 0; b < B_; ++b) {
    const size_t n = batch.samples[static_cast<size_t>(b)].response_tokens.size();
    const float* p = host.data() + static_cast<size_t>(b) * T_;
    out.emplace_back(p, p + n);
  }
  return out;
}

// ---- free function ------------------------------------------------------------

std::vector<std::vector<double>> compute_advantages(rlo::Objective& obj, const rollmini::SampleBatch& batch,
                                                    const rollmini::TrainConfig& config) {
  return translate([&] {
    config.validate();  // policy.cpp:258
    DeviceBatch db;
    db.upload(batch);
    // Reference: per-token rewards win, else the scalar reward (policy.cpp:265-276)
    for (const auto& s : batch.samples)
      if (s.rewards.empty() && !s.scalar_reward && !s.response_tokens.empty())
        throw rollmini::InputError("compute_advantages: sample '" + s.sample_id + "' has no rewards");
    rlo::TrainConfig c = to_rlo(config);
    float* adv = db.scratch(0);
    // per-token rewards (with scalar-only samples resolved onto their last
    // token by upload) whenever any sample has them, else the scalar rewards
    obj.compute_advantages(c, db.view(), db.rewards(), db.rewards() ? nullptr : db.scalar_rewards(), nullptr, adv);
    obj.sync();
    return db.download(adv, batch);
  });
}

// ---- worker -------------------------------------------------------------------

B200PolicyWorker::B200PolicyWorker(int32_t device, const rollmini::TrainConfig& train_config, LogitsProvider logits,
                                   UpdateHook on_update)
    : obj_(device), train_config_(train_config), logits_(std::move(logits)), on_update_(std::move(on_update)),
      device_(device) {
  train_config_.validate();
  device_id = "cuda:" + std::to_string(device);
}

rollmini::Message B200PolicyWorker::call(const std::string& method, const rollmini::Message& input) {
  // Cluster workers run on their own threads (cluster.cpp:171-192): bind this
  // thread to the worker's GPU before any allocation or launch.
  cuda_check(cudaSetDevice(device_), "B200PolicyWorker: cudaSetDevice");
  // policy_workers.cpp:46-64 dispatch for the path's methods
  if (method == "forward_logprobs") return do_forward_logprobs(input);
  if (method == "compute_gradient") return do_compute_gradient(input);
  if (method == "apply_update") return do_apply_update(input);
  if (method == "get_version") {
    rollmini::Message out;
    out.fields["version"] = std::to_string(version_);
    return out;
  }
  throw rollmini::DispatchError("policy worker: unimplemented method '" + method + "'");
}

rollmini::Message B200PolicyWorker::do_forward_logprobs(const rollmini::Message& input) {
  // policy_workers.cpp:93-100: fills ref_logprobs with this replica's scores
  return translate([&] {
    DeviceBatch db;
    db.upload(input.batch);
    const rlo_logits L = logits_(input.batch, db.T());
    float* lp = db.scratch(0);
    obj_.forward_logprobs(db.view(), L, lp);
    obj_.sync();
    auto lps = db.download(lp, input.batch);
    rollmini::Message out;
    out.batch = input.batch;
    for (size_t s = 0; s < out.batch.size(); ++s) out.batch.samples[s].ref_logprobs = std::move(lps[s]);
    out.fields["version"] = std::to_string(version_);
    return out;
  });
}

rollmini::Message B200PolicyWorker::do_compute_gradient(const rollmini::Message& input) {
  // policy_workers.cpp:111-121: the per-rank GradAccum scalars and tensors["grad"].
  // The MLP parameter gradient of the reference has no counterpart here (the
  // model backward belongs to the trainer), so "grad" is 0-dim -- which
  // merge_gradients accepts (policy.cpp:421-430) and cluster_train_step
  // forwards to apply_update as grad_mean -- and "dlogp" carries
  // d(loss_t)/d(logp_t) per response token in sample order (policy.cpp:372-374).
  return translate([&] {
    const rollmini::SampleBatch& batch = input.batch;
    bool any_ref = false, any_noref = false;
    for (const auto& s : batch.samples) {  // policy.cpp:336-343, with the reference's sample ids
      const size_t n = s.response_tokens.size();
      if (n == 0) continue;
      if (s.advantages.size() != n)
        throw rollmini::InputError("ppo_gradient: sample '" + s.sample_id + "' missing advantages");
      if (s.response_logprobs.size() != n)
        throw rollmini::InputError("ppo_gradient: sample '" + s.sample_id + "' missing old logprobs");
      if (train_config_.kl_coef > 0.0 && s.ref_logprobs.size() != n)
        throw rollmini::InputError("ppo_gradient: sample '" + s.sample_id + "' missing ref logprobs");
      (s.ref_logprobs.empty() ? any_noref : any_ref) = true;
    }
    // kl_sum counts only samples that carry ref_logprobs (policy.cpp:368).
    // With kl_coef == 0 a batch may mix both kinds: the samples with ref go
    // first, as one view with ref log-probs, the others as a second view
    // without (seq_offset keeps their records apart); dlogp is put back in
    // sample order.
    std::vector<size_t> order(batch.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    size_t n_ref = batch.size();
    if (any_ref && any_noref) {
      std::stable_partition(order.begin(), order.end(),
                            [&](size_t i) { return !batch.samples[i].ref_logprobs.empty(); });
      n_ref = 0;
      for (size_t i : order) n_ref += batch.samples[i].ref_logprobs.empty() ? 0 : 1;
    } else if (!any_ref) {
      n_ref = 0;
    }
    rollmini::SampleBatch perm;
    for (size_t i : order) perm.push_back(batch.samples[i]);
    DeviceBatch db;
    db.upload(perm);
    const rlo_logits L = logits_(perm, db.T());
    rlo::TrainConfig c = to_rlo(train_config_);
    float* dlogp = db.scratch(1);
    const float* adv = db.advantages() ? db.advantages() : db.scratch(2);
    const int32_t T = db.T();
    const rlo_batch all = db.view();
    auto run = [&](int32_t b0, int32_t nb, bool with_ref) {
      if (nb == 0) return;
      const size_t off = static_cast<size_t>(b0) * static_cast<size_t>(T);
      rlo_batch v = all;
      v.B = nb;
      v.seq_offset = b0;
      v.lengths = all.lengths + b0;
      v.tokens = all.tokens + off;
      v.mask = all.mask ? all.mask + off : nullptr;
      rlo_logits lv = L;
      lv.data = static_cast<const char*>(L.data) +
                off * static_cast<size_t>(L.row_stride) * (L.dtype == RLO_DTYPE_BF16 ? 2 : 4);
      rlo_token_out out_tok{};
      out_tok.dlogp = dlogp + off;
      const float* old = db.old_logp();
      const float* ref = with_ref ? db.ref_logp() : nullptr;
      obj_.ppo_gradient(c, v, lv, nullptr, nullptr, old ? old + off : nullptr, ref ? ref + off : nullptr, adv + off,
                        &out_tok);
    };
    run(0, static_cast<int32_t>(n_ref), true);
    run(static_cast<int32_t>(n_ref), db.B() - static_cast<int32_t>(n_ref), false);
    // this rank's GradAccum scalars; zero tokens / non-finite values are the
    // controller's merge_gradients decision (policy.cpp:437-448)
    const rlo::Partials mine = obj_.rank_partials(c);
    auto dl = db.download(dlogp, perm);
    std::vector<std::vector<double>> by_sample(batch.size());
    for (size_t j = 0; j < order.size(); ++j) by_sample[order[j]] = std::move(dl[j]);
    std::vector<double> flat;
    for (auto& v : by_sample) flat.insert(flat.end(), v.begin(), v.end());
    rollmini::Message out;
    out.tensors["grad"] = {};
    out.tensors["dlogp"] = std::move(flat);
    out.scalars["loss_sum"] = mine.v[RLO_P_LOSS_SUM];
    out.scalars["ratio_sum"] = mine.v[RLO_P_RATIO_SUM];
    out.scalars["kl_sum"] = mine.v[RLO_P_KL_SUM];
    out.scalars["clipped"] = mine.v[RLO_P_CLIPPED];
    out.scalars["tokens"] = mine.v[RLO_P_TOKENS];
    return out;
  });
}

rollmini::Message B200PolicyWorker::do_apply_update(const rollmini::Message& input) {
  // policy_workers.cpp:123-128 / policy.cpp:452-460: a zero learning rate is
  // no update (the version stays); otherwise the trainer applies the step and
  // the version advances.
  const auto& grad_mean = input.tensor("grad_mean");
  const double lr = input.scalar("learning_rate");
  if (lr != 0.0) {
    ++version_;
    if (on_update_) on_update_(device_, lr, grad_mean, version_);
  }
  rollmini::Message out;
  out.fields["version"] = std::to_string(version_);
  return out;
}

rollmini::WorkerFactory b200_worker_factory(const rollmini::TrainConfig& train_config, LogitsProvider logits,
                                            UpdateHook on_update) {
  return [train_config, logits, on_update](int rank, int world_size, const std::string&) {
    auto w = std::make_unique<B200PolicyWorker>(rank, train_config, logits, on_update);
    w->rank = rank;
    w->world_size = world_size;
    return w;
  };
}

}  // namespace rollmini_b200
