// rlo.hpp — C++ surface over the C ABI (rlo.h), shaped like the reference's
// include/rollmini/policy.hpp + errors.hpp so reference-side code can switch
// with minimal edits:
//
//   rollmini::TrainConfig        -> rlo::TrainConfig      (policy.hpp:57-67, same defaults)
//   rollmini::UpdateStats        -> rlo::UpdateStats      (policy.hpp:130-136, + extension stats)
//   rollmini::InputError, ...    -> rlo::InputError, ...  (errors.hpp:11-82, same messages)
//   compute_advantages / forward_logprobs / ppo_gradient / merge_gradients
//                                -> rlo::Objective methods (one object per GPU per worker
//                                   thread, like one PolicyWorkspace per worker)
//   split_sizes                  -> rlo::split_sizes      (sample.hpp:51-53)
//
// Header-only; link with -lrlo (paper_2506_06122_b200/lib/librlo.so).
// Streams are passed as void* (a cudaStream_t) so this header needs no CUDA
// headers.
#pragma once

#include <cstdint>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rlo.h"

namespace rlo {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class InputError : public Error {
 public:
  using Error::Error;
};
class TrainingError : public Error {
 public:
  using Error::Error;
};
class DispatchError : public Error {
 public:
  using Error::Error;
};
class CollectError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

inline void check(rlo_status s) {
  if (s == RLO_OK) return;
  const std::string msg = rlo_last_error();
  switch (s) {
    case RLO_ERR_INPUT: throw InputError(msg);
    case RLO_ERR_CONFIG: throw ConfigError(msg);
    case RLO_ERR_TRAINING: throw TrainingError(msg);
    case RLO_ERR_NCCL: throw CollectError(msg);
    case RLO_ERR_DISPATCH: throw DispatchError(msg);
    case RLO_ERR_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}

struct TrainConfig : rlo_train_config {
  TrainConfig() { rlo_train_config_default(this); }
  void validate() const { check(rlo_train_config_validate(this)); }
};

using UpdateStats = rlo_stats;
using Partials = rlo_partials;

inline std::vector<int64_t> split_sizes(int64_t n, int32_t parts) {
  std::vector<int64_t> out(static_cast<size_t>(parts > 0 ? parts : 0));
  check(rlo_split_sizes(n, parts, out.data()));
  return out;
}

inline std::pair<int32_t, int32_t> shard_plan(int32_t B, int32_t G, int32_t world, int32_t rank) {
  int32_t b = 0, n = 0;
  check(rlo_shard_plan(B, G, world, rank, &b, &n));
  return {b, n};
}

inline UpdateStats merge_partials(const std::vector<Partials>& parts, const TrainConfig& cfg) {
  UpdateStats st{};
  check(rlo_merge_partials(parts.data(), static_cast<int32_t>(parts.size()), &cfg, &st));
  return st;
}

// RAII owner of one rlo_handle (device workspace + optional NCCL group).
class Objective {
 public:
  explicit Objective(int32_t device) { check(rlo_create(device, &h_)); }
  ~Objective() { rlo_destroy(h_); }
  Objective(const Objective&) = delete;
  Objective& operator=(const Objective&) = delete;
  Objective(Objective&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }

  static std::vector<char> unique_id() {
    std::vector<char> id(128);
    check(rlo_comm_unique_id(id.data()));
    return id;
  }
  void init_comm(const std::vector<char>& id, int32_t rank, int32_t world) {
    check(rlo_comm_init(h_, id.data(), rank, world));
  }

  void forward_logprobs(const rlo_batch& batch, const rlo_logits& logits, float* logp, float* entropy = nullptr,
                        float* token_logit = nullptr, void* stream = nullptr) {
    check(rlo_forward_logprobs(h_, &batch, &logits, logp, entropy, token_logit, stream));
  }
  void compute_advantages(const TrainConfig& cfg, const rlo_batch& batch, const float* rewards_tok,
                          const float* rewards_seq, const float* values, float* adv, float* returns = nullptr,
                          void* stream = nullptr) {
    check(rlo_compute_advantages(h_, &cfg, &batch, rewards_tok, rewards_seq, values, adv, returns, stream));
  }
  void ppo_gradient(const TrainConfig& cfg, const rlo_batch& batch, const rlo_logits& actor,
                    const rlo_logits* old_logits, const rlo_logits* ref_logits, const float* old_logp,
                    const float* ref_logp, const float* adv, const rlo_token_out* out = nullptr,
                    void* stream = nullptr) {
    check(rlo_ppo_gradient(h_, &cfg, &batch, &actor, old_logits, ref_logits, old_logp, ref_logp, adv, out, stream));
  }
  UpdateStats merge_gradients(const TrainConfig& cfg, Partials* mine = nullptr, void* stream = nullptr) {
    UpdateStats st{};
    check(rlo_merge_gradients(h_, &cfg, &st, mine, stream));
    return st;
  }
  // merge_gradients without host synchronisation (CUDA-graph capturable):
  // `out` is device (or host-mapped) memory; read it with step_result().
  void merge_gradients_async(const TrainConfig& cfg, rlo_step_result* out, void* stream = nullptr) {
    check(rlo_merge_gradients_async(h_, &cfg, out, stream));
  }
  // UpdateStats of a host copy of a merge_gradients_async result; throws what
  // the synchronous merge_gradients would have thrown.
  static UpdateStats step_result(const rlo_step_result& host_copy) {
    check(rlo_step_result_check(&host_copy));
    return host_copy.stats;
  }
  Partials rank_partials(const TrainConfig& cfg, void* stream = nullptr) {
    Partials p{};
    check(rlo_rank_partials(h_, &cfg, &p, stream));
    return p;
  }
  // Actor update (policy.cpp:375-379): counts ahead of the pass -> weights ->
  // loss + backward epilogue in one read of the actor logits.
  UpdateStats batch_counts(const TrainConfig& cfg, const rlo_batch& batch, void* stream = nullptr) {
    UpdateStats st{};
    check(rlo_batch_counts(h_, &cfg, &batch, &st, stream));
    return st;
  }
  void loss_weights(const TrainConfig& cfg, const rlo_batch& batch, const UpdateStats& counts, float* w,
                    void* stream = nullptr) {
    check(rlo_loss_weights(h_, &cfg, &batch, &counts, w, stream));
  }
  void ppo_gradient_fused(const TrainConfig& cfg, const rlo_batch& batch, const rlo_logits& actor,
                          const rlo_logits* old_logits, const rlo_logits* ref_logits, const float* old_logp,
                          const float* ref_logp, const float* adv, const float* weight, void* grad,
                          int32_t grad_dtype, int64_t grad_row_stride, const rlo_token_out* out = nullptr,
                          void* stream = nullptr) {
    check(rlo_ppo_gradient_fused(h_, &cfg, &batch, &actor, old_logits, ref_logits, old_logp, ref_logp, adv, weight,
                                 grad, grad_dtype, grad_row_stride, out, stream));
  }
  void logits_backward(const rlo_batch& batch, const rlo_logits& logits, const float* lse, const float* dlogp,
                       const float* weight, void* grad, int32_t grad_dtype, int64_t grad_row_stride,
                       void* stream = nullptr) {
    check(rlo_logits_backward(h_, &batch, &logits, lse, dlogp, weight, grad, grad_dtype, grad_row_stride, stream));
  }
  // The whole step from host SampleBatch arrays (rlo_objective_step_host).
  UpdateStats step_host(const TrainConfig& cfg, int32_t B, int32_t T, const int32_t* lengths, const int32_t* tokens,
                        const uint8_t* mask, const float* rewards_tok, const float* rewards_seq, const float* values,
                        const rlo_logits& actor, const rlo_logits* old_logits, const rlo_logits* ref_logits,
                        const float* old_logp, const float* ref_logp, float* adv_out, float* logp_out,
                        void* stream = nullptr) {
    UpdateStats st{};
    check(rlo_objective_step_host(h_, &cfg, B, T, lengths, tokens, mask, rewards_tok, rewards_seq, values, &actor,
                                  old_logits, ref_logits, old_logp, ref_logp, adv_out, logp_out, &st, stream));
    return st;
  }
  // Micro-batched form (rlo_objective_step_host_mb): `logits(mb, seq_begin,
  // n_seqs, actor, old, ref)` names each micro-batch's device logits (run the
  // model forward there); an exception thrown by it aborts the step and is
  // rethrown here.
  using LogitsFn = std::function<void(int32_t mb, int32_t seq_begin, int32_t n_seqs, rlo_logits* actor,
                                      rlo_logits* old_logits, rlo_logits* ref_logits)>;
  UpdateStats step_host_mb(const TrainConfig& cfg, int32_t B, int32_t T, int32_t mb_seqs, const int32_t* lengths,
                           const int32_t* tokens, const uint8_t* mask, const float* rewards_tok,
                           const float* rewards_seq, const float* values, const LogitsFn& logits,
                           const float* old_logp, const float* ref_logp, float* adv_out, float* logp_out,
                           void* stream = nullptr) {
    struct Ctx {
      const LogitsFn* fn;
      std::exception_ptr err;
    } ctx{&logits, nullptr};
    auto tramp = [](void* user, int32_t mb, int32_t b0, int32_t nb, rlo_logits* a, rlo_logits* o,
                    rlo_logits* r) -> rlo_status {
      auto* c = static_cast<Ctx*>(user);
      try {
        (*c->fn)(mb, b0, nb, a, o, r);
        return RLO_OK;
      } catch (...) {
        c->err = std::current_exception();
        return RLO_ERR_INPUT;
      }
    };
    UpdateStats st{};
    const rlo_status rc = rlo_objective_step_host_mb(h_, &cfg, B, T, mb_seqs, lengths, tokens, mask, rewards_tok,
                                                     rewards_seq, values, tramp, &ctx, old_logp, ref_logp, adv_out,
                                                     logp_out, &st, stream);
    if (ctx.err) std::rethrow_exception(ctx.err);
    check(rc);
    return st;
  }
  void sync(void* stream = nullptr) { check(rlo_sync(h_, stream)); }
  rlo_handle* get() const { return h_; }

 private:
  rlo_handle* h_ = nullptr;
};

}  // namespace rlo
