// integration_main.cpp — drop-in check at the reference's own API level.
//
// Runs the reference's PolicyWorker (policy_workers.cpp, compiled from
// /root/reference into oracle/_ref) and the B200PolicyWorker
// (integration/b200_policy_worker.cpp -> librlo.so) on the same Messages and
// compares their replies, then drives B200 workers through the reference's
// own Cluster + cluster_forward_logprobs (cluster.cpp, policy_workers.cpp:298-303).
// Both see identical logits: the reference through the "b2 trick"
// (PolicyLayout{V,1,1,1}, all parameters 0 except b2 := row, so every
// position's logits equal `row`), the B200 worker through a LogitsProvider
// that tiles the same row into device memory.
//
// Exit code 0 = all checks passed.  Built by tests/cpp/Makefile (needs the
// reference headers); run by tests/test_gpu_integration.py on a B200.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "b200_policy_worker.hpp"
#include "rollmini/cluster.hpp"
#include "rollmini/errors.hpp"
#include "rollmini/policy.hpp"
#include "rollmini/policy_workers.hpp"
#include "rollmini/rng.hpp"
#include "rollmini/vocab.hpp"

using namespace rollmini;

namespace {

int g_fail = 0;

void check(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++g_fail;
}

bool close(double g, double r, double tol = 1e-5) { return std::fabs(g - r) <= tol * std::max(1.0, std::fabs(r)); }

// Device logits provider: every row of the padded view equals `row`.  Called
// from several worker threads (one per rank / GPU): one buffer per device.
struct TiledRow {
  std::vector<float> row;
  std::mutex mu;
  std::map<int, std::pair<float*, size_t>> bufs;  // device -> (buffer, capacity)
  rlo_logits operator()(const SampleBatch& batch, int32_t T) {
    const size_t V = row.size(), rows = batch.size() * static_cast<size_t>(T);
    int dev = 0;
    cudaGetDevice(&dev);  // the calling worker bound its GPU
    std::lock_guard<std::mutex> lock(mu);
    auto& [ptr, cap] = bufs[dev];
    if (rows * V > cap) {
      if (ptr) cudaFree(ptr);
      cap = rows * V;
      cudaMalloc(&ptr, sizeof(float) * cap);
    }
    std::vector<float> host(rows * V);
    for (size_t r = 0; r < rows; ++r) std::memcpy(host.data() + r * V, row.data(), sizeof(float) * V);
    cudaMemcpy(ptr, host.data(), sizeof(float) * host.size(), cudaMemcpyHostToDevice);
    return rlo_logits{ptr, RLO_DTYPE_F32, static_cast<int32_t>(V), static_cast<int64_t>(V)};
  }
};

}  // namespace

int main() {
  const int V = 37;
  rng::Stream s(2506);
  std::vector<float> row(V);
  for (auto& z : row) z = static_cast<float>(1.5 * s.next_gaussian());
  PolicyParams params;
  params.layout = PolicyLayout{V, 1, 1, 1};
  params.version = 1;
  params.values.assign(params.layout.param_count(), 0.0);
  for (int v = 0; v < V; ++v) params.values[params.layout.off_b2() + v] = row[static_cast<size_t>(v)];

  // A batch in the reference's own currency (sample.hpp:16-33).
  SampleBatch batch;
  for (int i = 0; i < 7; ++i) {
    SampleRecord r;
    r.sample_id = "s" + std::to_string(i);
    r.prompt_tokens = {1, 2};
    const size_t n = 1 + s.next_below(9);
    for (size_t t = 0; t < n; ++t) r.response_tokens.push_back(static_cast<int>(s.next_below(V)));
    if (i % 2) {
      for (size_t t = 0; t < n; ++t) r.action_mask.push_back(s.next_double() < 0.75 ? 1 : 0);
      r.action_mask[0] = 1;
    }
    batch.push_back(r);
  }
  const auto lps = forward_logprobs(params, batch);
  for (size_t i = 0; i < batch.size(); ++i) {
    auto& r = batch.samples[i];
    for (size_t t = 0; t < r.response_tokens.size(); ++t) {
      r.response_logprobs.push_back(lps[i][t] + 0.4 * (2.0 * s.next_double() - 1.0));
      r.ref_logprobs.push_back(lps[i][t] + 0.2 * (2.0 * s.next_double() - 1.0));
      r.advantages.push_back(2.0 * s.next_double() - 1.0);
      r.rewards.push_back(t + 1 == r.response_tokens.size() ? s.next_double() : 0.0);
    }
  }

  TrainConfig cfg;
  cfg.kl_coef = 0.1;
  const Vocabulary& vocab = Vocabulary::standard();
  (void)vocab;
  TiledRow tiles;
  tiles.row = row;
  auto provider = [&tiles](const SampleBatch& b, int32_t T) { return tiles(b, T); };

  PolicyWorker ref_worker(params, Vocabulary::standard(), cfg);
  rollmini_b200::B200PolicyWorker b200(0, cfg, provider);

  Message in;
  in.batch = batch;
  in.fields["version"] = "1";

  // 1) forward_logprobs (policy_workers.cpp:93-100)
  {
    Message a = ref_worker.call("forward_logprobs", in);
    Message b = b200.call("forward_logprobs", in);
    double worst = 0.0;
    for (size_t i = 0; i < batch.size(); ++i)
      for (size_t t = 0; t < a.batch.samples[i].ref_logprobs.size(); ++t) {
        const double g = b.batch.samples[i].ref_logprobs[t], r = a.batch.samples[i].ref_logprobs[t];
        worst = std::max(worst, std::fabs(g - r) / std::max(1.0, std::fabs(r)));
      }
    check(worst <= 1e-5, "forward_logprobs reply matches the reference worker (max scaled err " +
                             std::to_string(worst) + ")");
  }

  // 2) compute_gradient scalars (policy_workers.cpp:111-121) and the controller merge (policy.cpp:421-450)
  {
    Message a = ref_worker.call("compute_gradient", in);
    Message b = b200.call("compute_gradient", in);
    bool ok = true;
    for (const char* k : {"loss_sum", "ratio_sum", "kl_sum"}) ok &= close(b.scalar(k), a.scalar(k));
    ok &= b.scalar("clipped") == a.scalar("clipped") && b.scalar("tokens") == a.scalar("tokens");
    check(ok, "compute_gradient scalars match (loss_sum " + std::to_string(b.scalar("loss_sum")) + " vs " +
                  std::to_string(a.scalar("loss_sum")) + ", tokens " + std::to_string(b.scalar("tokens")) + ")");
    GradAccum pa, pb;
    pa.loss_sum = a.scalar("loss_sum");
    pa.ratio_sum = a.scalar("ratio_sum");
    pa.kl_sum = a.scalar("kl_sum");
    pa.clipped = static_cast<size_t>(a.scalar("clipped"));
    pa.tokens = static_cast<size_t>(a.scalar("tokens"));
    pb.loss_sum = b.scalar("loss_sum");
    pb.ratio_sum = b.scalar("ratio_sum");
    pb.kl_sum = b.scalar("kl_sum");
    pb.clipped = static_cast<size_t>(b.scalar("clipped"));
    pb.tokens = static_cast<size_t>(b.scalar("tokens"));
    const auto sa = merge_gradients({pa}).second, sb = merge_gradients({pb}).second;
    check(close(sb.loss, sa.loss) && close(sb.mean_ratio, sa.mean_ratio) && close(sb.mean_kl, sa.mean_kl) &&
              sb.tokens == sa.tokens,
          "reference merge_gradients over B200 partials == over reference partials");
    check(b.tensors.count("dlogp") == 1, "compute_gradient returns per-token dlogp");
  }

  // 3) compute_advantages (policy.cpp:257-311), whitening on
  {
    TrainConfig c2 = cfg;
    c2.whiten_advantages = true;
    c2.gamma = 0.95;
    const auto ra = compute_advantages(batch, c2);
    const auto ga = rollmini_b200::compute_advantages(b200.objective(), batch, c2);
    double worst = 0.0;
    for (size_t i = 0; i < ra.size(); ++i)
      for (size_t t = 0; t < ra[i].size(); ++t)
        worst = std::max(worst, std::fabs(ga[i][t] - ra[i][t]) / std::max(1.0, std::fabs(ra[i][t])));
    check(worst <= 2e-5, "compute_advantages matches the reference (max scaled err " + std::to_string(worst) + ")");
  }

  // 4) error contracts: same exception classes and messages
  {
    Message bad = in;
    bad.batch.samples[2].advantages.clear();
    std::string ra, rb;
    try {
      ref_worker.call("compute_gradient", bad);
    } catch (const InputError& e) {
      ra = e.what();
    }
    try {
      b200.call("compute_gradient", bad);
    } catch (const InputError& e) {
      rb = e.what();
    }
    check(!ra.empty() && ra == rb, "missing advantages -> InputError '" + rb + "'");
    bool dispatch = false;
    try {
      b200.call("generate", in);
    } catch (const DispatchError&) {
      dispatch = true;
    }
    check(dispatch, "unknown method -> DispatchError");
    Message oov = in;
    oov.batch.samples[0].response_tokens[0] = V + 3;
    std::string ea, eb;
    try {
      ref_worker.call("forward_logprobs", oov);
    } catch (const InputError& e) {
      ea = e.what();
    }
    try {
      b200.call("forward_logprobs", oov);
    } catch (const InputError& e) {
      eb = e.what();
    }
    check(!ea.empty() && ea == eb, "OOV token -> InputError '" + eb + "'");
  }

  // 5) the reference's own Cluster driving B200 workers (thread per rank)
  {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    std::vector<BindingAssignment> assign = {{0, "g0"}, {1, "g1"}};
    auto factory = [&provider, &cfg, ndev](int rank, int world, const std::string&) -> std::unique_ptr<Worker> {
      auto w = std::make_unique<rollmini_b200::B200PolicyWorker>(rank % std::max(ndev, 1), cfg, provider);
      w->rank = rank;
      w->world_size = world;
      return w;
    };
    Cluster cluster(Role::reference, 2, assign, factory);
    SampleBatch out = cluster_forward_logprobs(cluster, batch);
    double worst = 0.0;
    for (size_t i = 0; i < batch.size(); ++i)
      for (size_t t = 0; t < lps[i].size(); ++t)
        worst = std::max(worst, std::fabs(out.samples[i].ref_logprobs[t] - lps[i][t]) / std::max(1.0, std::fabs(lps[i][t])));
    check(out.size() == batch.size() && worst <= 1e-5,
          "reference Cluster + cluster_forward_logprobs over 2 B200 workers == reference forward_logprobs");
  }

  // 6) compute_advantages on a batch MIXING per-token and scalar-only rewards
  //    (policy.cpp:265-276 resolves the source per sample)
  {
    SampleBatch mixed = batch;
    for (size_t i = 1; i < mixed.size(); i += 2) {
      auto& r = mixed.samples[i];
      r.rewards.clear();
      r.scalar_reward = 0.25 + 0.5 * static_cast<double>(i);
    }
    TrainConfig c2 = cfg;
    c2.gamma = 0.9;
    for (bool whiten : {false, true}) {
      c2.whiten_advantages = whiten;
      const auto ra = compute_advantages(mixed, c2);
      const auto ga = rollmini_b200::compute_advantages(b200.objective(), mixed, c2);
      double worst = 0.0;
      for (size_t i = 0; i < ra.size(); ++i)
        for (size_t t = 0; t < ra[i].size(); ++t)
          worst = std::max(worst, std::fabs(ga[i][t] - ra[i][t]) / std::max(1.0, std::fabs(ra[i][t])));
      check(worst <= 2e-5, std::string("mixed per-token / scalar rewards: compute_advantages matches (whiten ") +
                               (whiten ? "on" : "off") + ", max scaled err " + std::to_string(worst) + ")");
    }
  }

  // 7) compute_gradient with kl_coef = 0 on a batch where some samples carry
  //    no ref_logprobs: kl_sum counts only the samples that do (policy.cpp:368)
  {
    TrainConfig c0 = cfg;
    c0.kl_coef = 0.0;
    PolicyWorker ref0(params, Vocabulary::standard(), c0);
    rollmini_b200::B200PolicyWorker b0(0, c0, provider);
    Message mix = in;
    mix.batch.samples[1].ref_logprobs.clear();
    mix.batch.samples[4].ref_logprobs.clear();
    Message a = ref0.call("compute_gradient", mix);
    Message b = b0.call("compute_gradient", mix);
    bool ok = true;
    for (const char* k : {"loss_sum", "ratio_sum", "kl_sum"}) ok &= close(b.scalar(k), a.scalar(k));
    ok &= b.scalar("clipped") == a.scalar("clipped") && b.scalar("tokens") == a.scalar("tokens");
    size_t ntok = 0;
    for (const auto& r : mix.batch.samples) ntok += r.response_tokens.size();
    ok &= b.tensor("dlogp").size() == ntok;
    check(ok, "mixed ref_logprobs presence (kl_coef 0): scalars match (kl_sum " + std::to_string(b.scalar("kl_sum")) +
                  " vs " + std::to_string(a.scalar("kl_sum")) + ")");
    // dlogp is returned in sample order: equal to a batch without the
    // permutation when every sample carries ref (kl_coef 0: ref does not enter
    // dlogp) -- up to fp32 rounding, since permuting the samples moves these
    // 148-byte rows to other 16-byte alignments (another summation split)
    Message full = b0.call("compute_gradient", in);
    const auto& dm = b.tensor("dlogp");
    const auto& df = full.tensor("dlogp");
    size_t first_bad = dm.size() == df.size() ? dm.size() : 0;
    for (size_t i = 0; i < std::min(dm.size(), df.size()); ++i)
      if (!close(dm[i], df[i], 1e-6)) {
        first_bad = i;
        break;
      }
    check(first_bad == dm.size(), "mixed-ref dlogp is returned in sample order" +
                                      (first_bad < dm.size() ? " (first difference at " + std::to_string(first_bad) +
                                                                   ": " + std::to_string(dm[first_bad]) + " vs " +
                                                                   std::to_string(df[first_bad]) + ")"
                                                             : std::string()));
  }

  // 8) the reference's own training controller, cluster_train_step
  //    (policy_workers.cpp:208-232: compute_gradient over shards ->
  //    merge_gradients -> apply_update broadcast), unchanged, over 2 B200
  //    workers vs over 2 reference PolicyWorkers
  {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    std::vector<BindingAssignment> assign = {{0, "g0"}, {1, "g1"}};
    std::mutex mu;
    std::vector<std::pair<int, double>> updates;
    size_t grad_dim = 99;
    rollmini_b200::UpdateHook hook = [&](int32_t device, double lr, const std::vector<double>& g, uint64_t ver) {
      std::lock_guard<std::mutex> lock(mu);
      updates.emplace_back(device, lr);
      grad_dim = g.size();
      (void)ver;
    };
    auto bfac = [&provider, &cfg, &hook, ndev](int rank, int world, const std::string&) -> std::unique_ptr<Worker> {
      auto w = std::make_unique<rollmini_b200::B200PolicyWorker>(rank % std::max(ndev, 1), cfg, provider, hook);
      w->rank = rank;
      w->world_size = world;
      return w;
    };
    Cluster b200_train(Role::actor_train, 2, assign, bfac);
    Cluster ref_train(Role::actor_train, 2, assign, policy_worker_factory(params, Vocabulary::standard(), cfg));
    const UpdateStats sb = cluster_train_step(b200_train, batch, cfg);
    const UpdateStats sa = cluster_train_step(ref_train, batch, cfg);
    check(close(sb.loss, sa.loss) && close(sb.mean_ratio, sa.mean_ratio) && close(sb.mean_kl, sa.mean_kl) &&
              close(sb.clip_fraction, sa.clip_fraction) && sb.tokens == sa.tokens,
          "cluster_train_step over 2 B200 workers == over 2 reference PolicyWorkers (loss " +
              std::to_string(sb.loss) + " vs " + std::to_string(sa.loss) + ", tokens " + std::to_string(sb.tokens) +
              ")");
    const Message v0 = b200_train.call_rank(0, "get_version", {});
    const Message r0 = ref_train.call_rank(0, "get_version", {});
    check(updates.size() == 2 && grad_dim == 0 && updates[0].second == cfg.learning_rate &&
              v0.field("version") == r0.field("version"),
          "apply_update reached every B200 rank (lr " + std::to_string(cfg.learning_rate) + "), version " +
              v0.field("version") + " == reference " + r0.field("version"));
  }

  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
