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
    obj.compute_advantages(c, db.view(), db.rewards(), db.rewards() ? nullptr : db.scalar_rewards(), nullptr, adv);
    obj.sync();
    return db.download(adv, batch);
  });
}

// ---- worker -------------------------------------------------------------------

B200PolicyWorker::B200PolicyWorker(int32_t device, const rollmini::TrainConfig& train_config, LogitsProvider logits)
    : obj_(device), train_config_(train_config), logits_(std::move(logits)), device_(device) {
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
  // policy_workers.cpp:111-121: per-rank GradAccum scalars; "dlogp" replaces
  // the MLP parameter gradient (the model backward belongs to the trainer).
  return translate([&] {
    for (const auto& s : input.batch.samples) {  // policy.cpp:336-343, with the reference's sample ids
      const size_t n = s.response_tokens.size();
      if (n == 0) continue;
      if (s.advantages.size() != n)
        throw rollmini::InputError("ppo_gradient: sample '" + s.sample_id + "' missing advantages");
      if (s.response_logprobs.size() != n)
        throw rollmini::InputError("ppo_gradient: sample '" + s.sample_id + "' missing old logprobs");
      if (train_config_.kl_coef > 0.0 && s.ref_logprobs.size() != n)
        throw rollmini::InputError("ppo_gradient: sample '" + s.sample_id + "' missing ref logprobs");
    }
    DeviceBatch db;
    db.upload(input.batch);
    const rlo_logits L = logits_(input.batch, db.T());
    rlo::TrainConfig c = to_rlo(train_config_);
    rlo_token_out out_tok{};
    out_tok.dlogp = db.scratch(1);
    obj_.ppo_gradient(c, db.view(), L, nullptr, nullptr, db.old_logp(), db.ref_logp(),
                      db.advantages() ? db.advantages() : db.scratch(2), &out_tok);
    // this rank's GradAccum scalars; zero tokens / non-finite values are the
    // controller's merge_gradients decision (policy.cpp:437-448)
    const rlo::Partials mine = obj_.rank_partials(c);
    rollmini::Message out;
    auto dl = db.download(out_tok.dlogp, input.batch);
    std::vector<double> flat;
    for (auto& v : dl) flat.insert(flat.end(), v.begin(), v.end());
    out.tensors["dlogp"] = std::move(flat);
    out.scalars["loss_sum"] = mine.v[RLO_P_LOSS_SUM];
    out.scalars["ratio_sum"] = mine.v[RLO_P_RATIO_SUM];
    out.scalars["kl_sum"] = mine.v[RLO_P_KL_SUM];
    out.scalars["clipped"] = mine.v[RLO_P_CLIPPED];
    out.scalars["tokens"] = mine.v[RLO_P_TOKENS];
    return out;
  });
}

rollmini::WorkerFactory b200_worker_factory(const rollmini::TrainConfig& train_config, LogitsProvider logits) {
  return [train_config, logits](int rank, int world_size, const std::string&) {
    auto w = std::make_unique<B200PolicyWorker>(rank, train_config, logits);
    w->rank = rank;
    w->world_size = world_size;
    return w;
  };
}

}  // namespace rollmini_b200
