// trainer_step.cpp — a C++ trainer's use of the B200 RL-objective library
// through include/rlo.hpp only (no Python, no PyTorch): one GRPO update step
// over micro-batches, then the fused loss + dlogits pass for the actor
// backward, then sampling-time log-probs for the next rollout.  The logits
// stand in for the model's forward output (counter-hash synthetic rows,
// include/rlo_synth.h).  Prints the UpdateStats and a gradient checksum, and
// exits non-zero on any library error.
//
//   make -C examples && ./build/trainer_step
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rlo.hpp"

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      std::exit(2);                                                                        \
    }                                                                                      \
  } while (0)

template <class T>
T* to_device(const std::vector<T>& h) {
  T* d = nullptr;
  CK(cudaMalloc(&d, sizeof(T) * (h.empty() ? 1 : h.size())));
  if (!h.empty()) CK(cudaMemcpy(d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
  return d;
}

int main() {
  try {
    const int32_t G = 8, B = 64, T = 256, V = 32000, MB = 16;  // 8 prompts x 8 responses, 4 micro-batches
    rlo::Objective obj(0);
    cudaStream_t s;
    CK(cudaStreamCreate(&s));

    // ---- the rollout's SampleBatch (host), ragged lengths, binary rewards
    std::vector<int32_t> lengths(B);
    std::vector<float> rewards(B);
    for (int b = 0; b < B; ++b) {
      lengths[b] = T / 2 + (b * 37) % (T / 2 + 1);
      rewards[b] = (b * 7919 % 5) < 2 ? 1.f : 0.f;
    }
    int32_t* d_len = to_device(lengths);
    float* d_rew = to_device(rewards);
    int32_t* d_tok = nullptr;
    CK(cudaMalloc(&d_tok, sizeof(int32_t) * B * T));
    rlo::check(rlo_synth_tokens(d_tok, (int64_t)B * T, V, 42, 0, (int64_t)B * T, s));

    // ---- logits of the actor / old-policy / reference models (the forward pass's output)
    float* logits[3];
    for (int m = 0; m < 3; ++m) {
      CK(cudaMalloc(&logits[m], sizeof(float) * (size_t)B * T * V));
      rlo::check(rlo_synth_logits(logits[m], RLO_DTYPE_F32, (int64_t)B * T, V, V, 42, m, 0, s));
    }
    auto view = [&](int m, int b0) { return rlo_logits{logits[m] + (size_t)b0 * T * V, RLO_DTYPE_F32, V, V, nullptr}; };

    rlo::TrainConfig cfg;  // reference defaults (policy.hpp:58-64) + extensions below
    cfg.adv_estimator = RLO_ADV_GRPO;
    cfg.group_size = G;
    cfg.kl_coef = 1e-3;
    cfg.kl_estimator = RLO_KL_K3;
    cfg.validate();

    // ---- advantages for the whole batch, then the loss over micro-batches of whole groups
    float* d_adv = nullptr;
    CK(cudaMalloc(&d_adv, sizeof(float) * B * T));
    rlo_batch full{B, T, 0, 0, d_len, d_tok, nullptr};
    obj.compute_advantages(cfg, full, nullptr, d_rew, nullptr, d_adv, nullptr, s);
    for (int b0 = 0; b0 < B; b0 += MB) {
      rlo_batch mb{MB, T, b0, 0, d_len + b0, d_tok + (size_t)b0 * T, nullptr};
      const rlo_logits a = view(0, b0), o = view(1, b0), r = view(2, b0);
      obj.ppo_gradient(cfg, mb, a, &o, &r, nullptr, nullptr, d_adv + (size_t)b0 * T, nullptr, s);
    }
    const rlo::UpdateStats st = obj.merge_gradients(cfg, nullptr, s);
    std::printf("update: loss %.9f mean_ratio %.9f clip_fraction %.6f mean_kl %.3e entropy %.6f tokens %llu\n",
                st.loss, st.mean_ratio, st.clip_fraction, st.mean_kl, st.mean_entropy,
                (unsigned long long)st.tokens);

    // ---- actor backward: dL/dlogits in the same read of the actor logits as the loss
    float *d_w = nullptr, *d_grad = nullptr;
    CK(cudaMalloc(&d_w, sizeof(float) * B * T));
    CK(cudaMalloc(&d_grad, sizeof(float) * (size_t)B * T * V));
    const rlo::UpdateStats counts = obj.batch_counts(cfg, full, s);
    obj.loss_weights(cfg, full, counts, d_w, s);
    for (int b0 = 0; b0 < B; b0 += MB) {
      rlo_batch mb{MB, T, b0, 0, d_len + b0, d_tok + (size_t)b0 * T, nullptr};
      const rlo_logits a = view(0, b0), o = view(1, b0), r = view(2, b0);
      obj.ppo_gradient_fused(cfg, mb, a, &o, &r, nullptr, nullptr, d_adv + (size_t)b0 * T, d_w + (size_t)b0 * T,
                             d_grad + (size_t)b0 * T * V, RLO_DTYPE_F32, V, nullptr, s);
    }
    const rlo::UpdateStats st2 = obj.merge_gradients(cfg, nullptr, s);
    std::vector<float> g((size_t)T * V);
    CK(cudaMemcpy(g.data(), d_grad, sizeof(float) * g.size(), cudaMemcpyDeviceToHost));  // sequence 0's rows
    double gsum = 0.0, gabs = 0.0;
    for (float x : g) gsum += x, gabs += std::fabs(x);
    std::printf("fused: loss %.9f (same step) grad[seq 0] sum %.3e |sum| %.6e\n", st2.loss, gsum, gabs);
    if (std::fabs(st2.loss - st.loss) > 1e-6 * std::fmax(1.0, std::fabs(st.loss)) || st2.tokens != st.tokens) {
      std::fprintf(stderr, "fused pass disagrees with the two-pass loss\n");
      return 1;
    }
    if (std::fabs(gsum) > 1e-4 * gabs + 1e-9) {  // every gradient row sums to zero (onehot - softmax)
      std::fprintf(stderr, "gradient rows do not sum to zero\n");
      return 1;
    }

    // ---- the same step from host SampleBatch arrays (the reference-facing call):
    //      one copy in, advantages over the whole batch, a callback per
    //      micro-batch that names its logits (where the model forward would run)
    std::vector<int32_t> htok((size_t)B * T);
    CK(cudaMemcpy(htok.data(), d_tok, sizeof(int32_t) * htok.size(), cudaMemcpyDeviceToHost));
    std::vector<float> hadv((size_t)B * T), hlp((size_t)B * T);
    int calls = 0;
    const rlo::UpdateStats st3 = obj.step_host_mb(
        cfg, B, T, MB, lengths.data(), htok.data(), nullptr, nullptr, rewards.data(), nullptr,
        [&](int32_t mb, int32_t b0, int32_t nb, rlo_logits* a, rlo_logits* o, rlo_logits* r) {
          ++calls;
          (void)mb;
          (void)nb;
          *a = view(0, b0);
          *o = view(1, b0);
          *r = view(2, b0);
        },
        nullptr, nullptr, hadv.data(), hlp.data(), s);
    std::printf("host step: loss %.9f tokens %llu (%d micro-batch callbacks)\n", st3.loss,
                (unsigned long long)st3.tokens, calls);
    if (st3.loss != st.loss || st3.tokens != st.tokens || calls != B / MB) {
      std::fprintf(stderr, "host-buffer step disagrees with the device step\n");
      return 1;
    }

    // ---- next rollout: sample one token per sequence with its untempered log-prob
    std::vector<uint64_t> keys(B), pos(B, 0);
    for (int b = 0; b < B; ++b) keys[b] = rlo_sample_key(("sample-" + std::to_string(b)).c_str());
    uint64_t *d_keys = to_device(keys), *d_pos = to_device(pos);
    int32_t* d_next = nullptr;
    float* d_lp = nullptr;
    CK(cudaMalloc(&d_next, sizeof(int32_t) * B));
    CK(cudaMalloc(&d_lp, sizeof(float) * B));
    const rlo_logits last{logits[0], RLO_DTYPE_F32, V, (int64_t)T * V, nullptr};  // row t = 0 of each sequence
    rlo::check(rlo_decode_sample(obj.get(), &last, B, 0.8, 42, 1, d_keys, d_pos, d_next, d_lp, s));
    std::vector<int32_t> next(B);
    std::vector<float> lp(B);
    CK(cudaMemcpy(next.data(), d_next, sizeof(int32_t) * B, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(lp.data(), d_lp, sizeof(float) * B, cudaMemcpyDeviceToHost));
    std::printf("decode: token[0] %d logp %.6f token[1] %d logp %.6f\n", next[0], lp[0], next[1], lp[1]);
    for (int b = 0; b < B; ++b)
      if (next[b] < 0 || next[b] >= V || !(lp[b] <= 0.f)) {
        std::fprintf(stderr, "bad draw %d\n", b);
        return 1;
      }
    std::printf("launches %llu\nOK\n", (unsigned long long)rlo_launch_count());
  } catch (const rlo::Error& e) {
    std::fprintf(stderr, "rlo error: %s\n", e.what());
    return 1;
  }
  return 0;
}
