// b200_policy_worker.hpp — the reference-side binding a maintainer adds to
// rollmini to route the RL-objective path through the B200 library.
//
// It is a rollmini::Worker (include/rollmini/worker.hpp:37-45) answering the
// path's methods with the reference's Message schema
// (policy_workers.cpp:93-100 forward_logprobs, :111-121 compute_gradient), so
// Cluster::dispatch / cluster_forward_logprobs / controller code work
// unchanged.  The model's logits come from the trainer's own forward pass on
// the GPU through a LogitsProvider (the toy MLP of policy.cpp:74-123 is not
// part of the path).  Compiled against the reference headers; links
// librlo.so (include/rlo.h) and the CUDA runtime.
#pragma once

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "rlo.hpp"
#include "rollmini/policy.hpp"
#include "rollmini/sample.hpp"
#include "rollmini/worker.hpp"

namespace rollmini_b200 {

// Device logits for the rows of a padded view of `batch`: row (b, t) of the
// batch's b-th sample and t-th response position at data + (b*T + t)*row_stride.
using LogitsProvider = std::function<rlo_logits(const rollmini::SampleBatch& batch, int32_t T)>;

// apply_update (policy_workers.cpp:123-128, policy.cpp:452-460) on a B200
// worker: the model parameters and their backward live in the trainer (the
// path stops at dlogp / dlogits), so the worker hands the step to this hook:
// (worker device, learning rate, merged grad_mean -- 0-dim here, new version).
using UpdateHook = std::function<void(int32_t device, double learning_rate, const std::vector<double>& grad_mean,
                                      uint64_t version)>;

// Padded device copy of a SampleBatch (sample.hpp:16-60) for the C ABI.
class DeviceBatch {
 public:
  DeviceBatch() = default;
  ~DeviceBatch();
  DeviceBatch(const DeviceBatch&) = delete;
  DeviceBatch& operator=(const DeviceBatch&) = delete;

  // T = longest response; per-token arrays that are empty in every sample are
  // left null.  Rewards are resolved per sample as compute_advantages does
  // (policy.cpp:265-276): per-token rewards, else scalar_reward on the last
  // token -- so a batch mixing both kinds keeps every sample's reward.
  void upload(const rollmini::SampleBatch& batch);
  rlo_batch view() const;
  int32_t B() const { return B_; }
  int32_t T() const { return T_; }
  const float* old_logp() const { return has_old_ ? old_ : nullptr; }
  const float* ref_logp() const { return has_ref_ ? ref_ : nullptr; }
  const float* advantages() const { return has_adv_ ? adv_ : nullptr; }
  const float* rewards() const { return has_rtok_ ? rtok_ : nullptr; }
  const float* scalar_rewards() const { return has_rseq_ ? rseq_ : nullptr; }
  float* scratch(size_t k);  // [B*T] device float scratch k (0..3)
  // unpack a [B*T] device float array into per-sample vectors of the response lengths
  std::vector<std::vector<double>> download(const float* dev, const rollmini::SampleBatch& batch) const;

 private:
  void* alloc(size_t bytes);
  int32_t B_ = 0, T_ = 0;
  std::vector<void*> owned_;
  int32_t* lengths_ = nullptr;
  int32_t* tokens_ = nullptr;
  uint8_t* mask_ = nullptr;
  float *old_ = nullptr, *ref_ = nullptr, *adv_ = nullptr, *rtok_ = nullptr, *rseq_ = nullptr;
  bool has_mask_ = false, has_old_ = false, has_ref_ = false, has_adv_ = false, has_rtok_ = false, has_rseq_ = false;
  float* scratch_[4] = {nullptr, nullptr, nullptr, nullptr};
};

// Maps a rlo exception onto the same-named rollmini exception (errors.hpp).
[[noreturn]] void rethrow_as_rollmini(const rlo::Error& e);

rlo::TrainConfig to_rlo(const rollmini::TrainConfig& c);

// compute_advantages (policy.hpp:118) on the GPU; same return shape.
std::vector<std::vector<double>> compute_advantages(rlo::Objective& obj, const rollmini::SampleBatch& batch,
                                                    const rollmini::TrainConfig& config);

class B200PolicyWorker : public rollmini::Worker {
 public:
  B200PolicyWorker(int32_t device, const rollmini::TrainConfig& train_config, LogitsProvider logits,
                   UpdateHook on_update = nullptr);

  rollmini::Message call(const std::string& method, const rollmini::Message& input) override;

  rlo::Objective& objective() { return obj_; }

 private:
  rollmini::Message do_forward_logprobs(const rollmini::Message& input);
  rollmini::Message do_compute_gradient(const rollmini::Message& input);
  rollmini::Message do_apply_update(const rollmini::Message& input);

  rlo::Objective obj_;
  rollmini::TrainConfig train_config_;
  LogitsProvider logits_;
  UpdateHook on_update_;
  uint64_t version_ = 1;
  int32_t device_ = 0;
};

// WorkerFactory (worker.hpp:47-48) for a cluster of B200 workers, one GPU each.
rollmini::WorkerFactory b200_worker_factory(const rollmini::TrainConfig& train_config, LogitsProvider logits,
                                            UpdateHook on_update = nullptr);

}  // namespace rollmini_b200
