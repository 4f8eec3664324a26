// api.cpp — the C ABI (include/rlo.h): validation with the reference's error
// messages, the per-GPU handle and its workspace, the NCCL data-parallel
// group, and the stream-ordered orchestration of the sm_100a kernels.
//
// Host-side counterparts of the reference (proj/core/src/):
//   TrainConfig::validate      policy.cpp:29-37    -> rlo_train_config_validate
//   split_sizes                sample.cpp:99-105   -> rlo_split_sizes / rlo_shard_plan
//   merge_gradients            policy.cpp:421-450  -> rlo_merge_partials / rlo_merge_gradients
//   forward_logprobs           policy.cpp:210-233  -> rlo_forward_logprobs
//   compute_advantages         policy.cpp:257-311  -> rlo_compute_advantages
//   ppo_gradient (loss part)   policy.cpp:313-374  -> rlo_ppo_gradient
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is bound at run time (see nccl_api())

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace rlo {
std::atomic<uint64_t> g_launches{0};
}

using namespace rlo;

namespace {
thread_local std::string g_last_error;
}  // namespace

rlo_status rlo::set_last_error(rlo_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

namespace {

rlo_status fail(rlo_status code, const std::string& msg) { return set_last_error(code, msg); }

rlo_status cuda_fail(cudaError_t e, const char* where) {
  return fail(RLO_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define RLO_CUDA(call)                                       \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);      \
  } while (0)

// NCCL is resolved with dlopen on first use instead of being linked: the
// process may already hold a libnccl.so.2 (torch bundles NCCL 2.28 while the
// system copy is 2.27), and two different copies of one SONAME in one process
// break the one loaded second.  RTLD_NOLOAD picks the copy already resident;
// RLO_NCCL_LIBRARY overrides; otherwise the default search path is used.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
  bool ok() const { return GetUniqueId && CommInitRank && AllGather && Broadcast && CommDestroy && GetErrorString; }
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) {
      const char* env = std::getenv("RLO_NCCL_LIBRARY");
      h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      a.error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(h, "ncclBroadcast"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!a.ok()) a.error = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

#define RLO_NCCL(call)                                                                                  \
  do {                                                                                                  \
    if (!nccl_api().ok()) return fail(RLO_ERR_NCCL, nccl_api().error);                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess)                                                                              \
      return fail(RLO_ERR_NCCL, std::string(#call) + ": " + nccl_api().GetErrorString(r_));             \
  } while (0)

#define RLO_TRY(call)                    \
  do {                                   \
    rlo_status s_ = (call);              \
    if (s_ != RLO_OK) return s_;         \
  } while (0)

bool getenv_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && *e && *e != '0';
}

int getenv_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

struct DeviceGuard {
  int prev = -1, dev;
  explicit DeviceGuard(int d) : dev(d) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n, bool zero = false) {
    if (n <= cap) return cudaSuccess;
    if (p) {
      cudaError_t e = cudaFree(p);
      if (e != cudaSuccess) return e;
    }
    p = nullptr;
    cap = 0;
    cudaError_t e = cudaMalloc(&p, sizeof(T) * n);
    if (e != cudaSuccess) return e;
    cap = n;
    if (zero) return cudaMemset(p, 0, sizeof(T) * n);
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

}  // namespace

Tuning rlo::read_tuning() {
  Tuning t;
  t.fused_off = getenv_flag("RLO_FUSED_OFF");
  t.fused_slice_kb = getenv_int("RLO_FUSED_SLICE_KB", 0);
  t.fused_nb = getenv_int("RLO_FUSED_NB", 2) == 3 ? 3 : 2;
  t.fused_debug = getenv_flag("RLO_FUSED_DEBUG");
  const char* me = std::getenv("RLO_DECODE_MARGIN");
  t.decode_fixed_margin = me && *me;
  t.decode_margin = t.decode_fixed_margin ? std::atof(me) : -1.0;
  t.decode_noredo = getenv_flag("RLO_DECODE_NOREDO");
  return t;
}

struct rlo_handle {
  int device = 0;
  int num_sms = 148;
  Tuning tuning;  // environment knobs, read once here (internal.h)
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  // accumulator of the loss pass (per sequence), reset by merge
  DevBuf<SeqRec> recs;
  int32_t acc_nseq = 0;
  // per-token scratch of the loss pass
  DevBuf<float> s_loss, s_ratio, s_kl, s_ent;
  DevBuf<float> s_dlogp;  // two-pass fallback of the fused update pass
  DevBuf<double> s_lse64;
  DevBuf<uint8_t> s_flags;
  // whitening
  DevBuf<WStat> wstat;
  DevBuf<double> raw64;
  // next-row callers: loss weights, value loss
  DevBuf<float> counts;
  DevBuf<double> vseq, vout, vgath;
  DevBuf<double> stats4, stats_all, partials, gathered;
  DevBuf<DevError> err;
  // staging for rlo_objective_step_host and internal advantages
  DevBuf<int32_t> h_lengths, h_tokens;
  DevBuf<uint8_t> h_mask;
  DevBuf<float> h_rtok, h_rseq, h_values, h_old, h_ref, h_adv, h_logp;
  // pinned host mirrors
  double* host_gathered = nullptr;
  DevError* host_err = nullptr;
};

// ---------------------------------------------------------------------------
// library / config (host only)
// ---------------------------------------------------------------------------
extern "C" {

int rlo_abi_version(void) { return RLO_ABI_VERSION; }

const char* rlo_last_error(void) { return g_last_error.c_str(); }

uint64_t rlo_launch_count(void) { return g_launches.load(); }

void rlo_train_config_default(rlo_train_config* c) {
  // policy.hpp:58-64 defaults; extensions default to the reference behaviour.
  c->clip_eps = 0.2;
  c->kl_coef = 0.0;
  c->learning_rate = 0.05;
  c->advantage_clip = 10.0;
  c->reward_clip = 20.0;
  c->gamma = 1.0;
  c->whiten_advantages = 0;
  c->adv_estimator = RLO_ADV_REINFORCE;
  c->lambd = 0.95;
  c->kl_estimator = RLO_KL_K1;
  c->dual_clip_c = 0.0;
  c->loss_agg = RLO_AGG_TOKEN_MEAN;
  c->group_size = 1;
  c->grpo_std_ddof = 0;
  c->grpo_eps = 1e-6;
}

rlo_status rlo_train_config_validate(const rlo_train_config* c) {
  if (!c) return fail(RLO_ERR_CONFIG, "train config: null");
  // TrainConfig::validate, policy.cpp:29-37 (same order, same messages)
  if (!(c->clip_eps > 0.0 && c->clip_eps < 1.0)) return fail(RLO_ERR_CONFIG, "train config: clip_eps must be in (0,1)");
  if (c->kl_coef < 0.0) return fail(RLO_ERR_CONFIG, "train config: kl_coef must be non-negative");
  if (c->learning_rate < 0.0) return fail(RLO_ERR_CONFIG, "train config: learning_rate must be non-negative");
  if (!(c->advantage_clip > 0.0)) return fail(RLO_ERR_CONFIG, "train config: advantage_clip must be positive");
  if (!(c->reward_clip > 0.0)) return fail(RLO_ERR_CONFIG, "train config: reward_clip must be positive");
  if (!(c->gamma > 0.0 && c->gamma <= 1.0)) return fail(RLO_ERR_CONFIG, "train config: gamma must be in (0,1]");
  // extensions
  if (c->adv_estimator < RLO_ADV_REINFORCE || c->adv_estimator > RLO_ADV_GAE)
    return fail(RLO_ERR_CONFIG, "train config: adv_estimator must be reinforce, grpo or gae");
  if (!(c->lambd >= 0.0 && c->lambd <= 1.0)) return fail(RLO_ERR_CONFIG, "train config: lambda must be in [0,1]");
  if (c->kl_estimator < RLO_KL_K1 || c->kl_estimator > RLO_KL_K3)
    return fail(RLO_ERR_CONFIG, "train config: kl_estimator must be k1, k2 or k3");
  if (!(c->dual_clip_c == 0.0 || c->dual_clip_c > 1.0))
    return fail(RLO_ERR_CONFIG, "train config: dual_clip_c must be 0 (off) or > 1");
  if (c->loss_agg < RLO_AGG_TOKEN_MEAN || c->loss_agg > RLO_AGG_GROUP_MEAN)
    return fail(RLO_ERR_CONFIG, "train config: loss_agg must be token-mean, seq-mean-token-mean, "
                                "seq-mean-token-sum or group-mean");
  if (c->group_size < 1) return fail(RLO_ERR_CONFIG, "train config: group_size must be >= 1");
  if (c->grpo_std_ddof != 0 && c->grpo_std_ddof != 1)
    return fail(RLO_ERR_CONFIG, "train config: grpo_std_ddof must be 0 or 1");
  if (!(c->grpo_eps >= 0.0)) return fail(RLO_ERR_CONFIG, "train config: grpo_eps must be non-negative");
  return RLO_OK;
}

rlo_status rlo_split_sizes(int64_t n, int32_t parts, int64_t* out) {
  // sample.cpp:99-105: contiguous, sizes differ by at most one, larger first
  if (parts <= 0) return fail(RLO_ERR_CONFIG, "split: partition count must be positive");
  if (n < 0) return fail(RLO_ERR_INPUT, "split: negative item count");
  for (int32_t p = 0; p < parts; ++p) out[p] = n / parts;
  for (int64_t i = 0; i < n % parts; ++i) ++out[i];
  return RLO_OK;
}

rlo_status rlo_shard_plan(int32_t B, int32_t G, int32_t world, int32_t rank, int32_t* out_begin, int32_t* out_count) {
  if (world <= 0) return fail(RLO_ERR_CONFIG, "split: partition count must be positive");
  if (rank < 0 || rank >= world) return fail(RLO_ERR_CONFIG, "shard plan: rank out of range");
  if (G < 1) return fail(RLO_ERR_CONFIG, "train config: group_size must be >= 1");
  if (B < 0 || B % G != 0)
    return fail(RLO_ERR_INPUT, "shard plan: batch of " + std::to_string(B) + " samples is not whole groups of " +
                                   std::to_string(G));
  std::vector<int64_t> sizes(static_cast<size_t>(world));
  RLO_TRY(rlo_split_sizes(B / G, world, sizes.data()));
  int64_t begin = 0;
  for (int32_t r = 0; r < rank; ++r) begin += sizes[static_cast<size_t>(r)];
  *out_begin = static_cast<int32_t>(begin * G);
  *out_count = static_cast<int32_t>(sizes[static_cast<size_t>(rank)] * G);
  return RLO_OK;
}

rlo_status rlo_merge_partials(const rlo_partials* parts, int32_t nranks, const rlo_train_config* cfg, rlo_stats* out) {
  // merge_gradients, policy.cpp:421-450: rank-ordered sums, then normalisation.
  if (nranks <= 0 || !parts) return fail(RLO_ERR_TRAINING, "merge_gradients: no gradient parts");
  std::vector<double> flat(static_cast<size_t>(nranks) * RLO_NPARTIAL);
  for (int32_t r = 0; r < nranks; ++r) std::memcpy(&flat[static_cast<size_t>(r) * RLO_NPARTIAL], parts[r].v,
                                                   sizeof(double) * RLO_NPARTIAL);
  rlo_stats st;
  std::memset(&st, 0, sizeof(st));
  switch (merge_stats(flat.data(), nranks, cfg ? cfg->loss_agg : RLO_AGG_TOKEN_MEAN, &st)) {
    case 1: return fail(RLO_ERR_TRAINING, "merge_gradients: batch contains no loss-participating tokens");
    case 2: return fail(RLO_ERR_TRAINING, "training step aborted: non-finite gradient");
    case 3: return fail(RLO_ERR_TRAINING, "training step aborted: non-finite loss");
    default: break;
  }
  if (out) *out = st;
  return RLO_OK;
}

int32_t rlo_whiten_combine(const double* stats_all, int32_t world, double* mean, double* inv) {
  if (!stats_all || world <= 0 || !mean || !inv) return 0;
  return whiten_combine(stats_all, world, mean, inv);
}

// ---------------------------------------------------------------------------
// handle
// ---------------------------------------------------------------------------

rlo_status rlo_create(int32_t device, rlo_handle** out) {
  if (!out) return fail(RLO_ERR_INPUT, "rlo_create: null output");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(RLO_ERR_CUDA, std::string("rlo_create: no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(RLO_ERR_CUDA, "rlo_create: device ordinal out of range");
  DeviceGuard g(device);
  cudaDeviceProp prop;
  RLO_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(RLO_ERR_CUDA, std::string("rlo_create: built for sm_100a (B200); device is ") + prop.name);
  auto* h = new rlo_handle();
  h->device = device;
  h->num_sms = prop.multiProcessorCount;
  h->tuning = read_tuning();
  if (h->err.ensure(1) != cudaSuccess || cudaMemset(h->err.p, 0xFF, sizeof(DevError)) != cudaSuccess || h->stats4.ensure(4, true) != cudaSuccess ||
      h->partials.ensure(RLO_NPARTIAL, true) != cudaSuccess || h->stats_all.ensure(4, true) != cudaSuccess ||
      h->gathered.ensure(RLO_NPARTIAL, true) != cudaSuccess ||
      cudaMallocHost(&h->host_gathered, sizeof(double) * RLO_NPARTIAL) != cudaSuccess ||
      cudaMallocHost(&h->host_err, sizeof(DevError)) != cudaSuccess) {
    rlo_destroy(h);
    return fail(RLO_ERR_CUDA, "rlo_create: workspace allocation failed");
  }
  *out = h;
  return RLO_OK;
}

rlo_status rlo_destroy(rlo_handle* h) {
  if (!h) return RLO_OK;
  DeviceGuard g(h->device);
  if (h->comm && nccl_api().ok()) nccl_api().CommDestroy(h->comm);
  h->recs.release();
  h->s_loss.release();
  h->s_ratio.release();
  h->s_kl.release();
  h->s_ent.release();
  h->s_dlogp.release();
  h->s_lse64.release();
  h->s_flags.release();
  h->wstat.release();
  h->raw64.release();
  h->counts.release();
  h->vseq.release();
  h->vout.release();
  h->vgath.release();
  h->stats4.release();
  h->stats_all.release();
  h->partials.release();
  h->gathered.release();
  h->err.release();
  h->h_lengths.release();
  h->h_tokens.release();
  h->h_mask.release();
  h->h_rtok.release();
  h->h_rseq.release();
  h->h_values.release();
  h->h_old.release();
  h->h_ref.release();
  h->h_adv.release();
  h->h_logp.release();
  if (h->host_gathered) cudaFreeHost(h->host_gathered);
  if (h->host_err) cudaFreeHost(h->host_err);
  delete h;
  return RLO_OK;
}

rlo_status rlo_comm_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  RLO_NCCL(nccl_api().GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return RLO_OK;
}

rlo_status rlo_comm_init(rlo_handle* h, const void* id128, int32_t rank, int32_t world) {
  if (!h) return fail(RLO_ERR_INPUT, "rlo_comm_init: null handle");
  if (world < 1 || rank < 0 || rank >= world) return fail(RLO_ERR_CONFIG, "rlo_comm_init: bad rank/world");
  DeviceGuard g(h->device);
  if (world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    RLO_NCCL(nccl_api().CommInitRank(&h->comm, world, id, rank));
  }
  h->rank = rank;
  h->world = world;
  RLO_CUDA(h->stats_all.ensure(static_cast<size_t>(4 * world), true));
  RLO_CUDA(h->gathered.ensure(static_cast<size_t>(RLO_NPARTIAL * world), true));
  if (h->host_gathered) cudaFreeHost(h->host_gathered);
  RLO_CUDA(cudaMallocHost(&h->host_gathered, sizeof(double) * RLO_NPARTIAL * world));
  return RLO_OK;
}

// ---------------------------------------------------------------------------
// the path
// ---------------------------------------------------------------------------

namespace {

rlo_status check_batch(const rlo_batch* b, const char* op, bool need_tokens) {
  if (!b) return fail(RLO_ERR_INPUT, std::string(op) + ": null batch");
  if (b->B < 0 || b->T < 0 || b->seq_offset < 0) return fail(RLO_ERR_INPUT, std::string(op) + ": negative batch shape");
  if ((int64_t)b->B * b->T > 0 && (!b->lengths || (need_tokens && !b->tokens)))
    return fail(RLO_ERR_INPUT, std::string(op) + ": batch lengths/tokens missing");
  return RLO_OK;
}

rlo_status check_logits(const rlo_logits* l, const char* op, const char* which) {
  if (!l || !l->data) return fail(RLO_ERR_INPUT, std::string(op) + ": missing " + which + " logits");
  if (l->dtype != RLO_DTYPE_F32 && l->dtype != RLO_DTYPE_BF16)
    return fail(RLO_ERR_INPUT, std::string(op) + ": unsupported logits dtype");
  if (l->V <= 0 || l->row_stride < l->V)
    return fail(RLO_ERR_INPUT, std::string(op) + ": bad vocab size / row stride for " + which + " logits");
  return RLO_OK;
}

rlo_status device_error_status(int32_t code, int32_t value) {
  if (code == DE_NONE) return RLO_OK;
  switch (code) {
    case DE_OOV_LOGPROB:  // policy.cpp:224-225
      return fail(RLO_ERR_INPUT, "forward_logprobs: out-of-vocabulary token " + std::to_string(value));
    case DE_OOV_LOSS:
      return fail(RLO_ERR_INPUT, "ppo_gradient: out-of-vocabulary token " + std::to_string(value));
    default:
      return fail(RLO_ERR_INPUT, "sample batch: response length of sample '" + std::to_string(value) +
                                     "' is outside [0, T]");
  }
}

rlo_status collect_device_error(rlo_handle* h, cudaStream_t s) {
  // h->host_err was filled by an async copy already synchronised by the caller
  (void)s;
  int32_t code = DE_NONE, value = 0;
  dev_err_decode(h->host_err->key, &code, &value);
  return device_error_status(code, value);
}

}  // namespace

rlo_status rlo_sync(rlo_handle* h, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "rlo_sync: null handle");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RLO_CUDA(cudaMemcpyAsync(h->host_err, h->err.p, sizeof(DevError), cudaMemcpyDeviceToHost, s));
  RLO_CUDA(cudaMemsetAsync(h->err.p, 0xFF, sizeof(DevError), s));
  RLO_CUDA(cudaStreamSynchronize(s));
  return collect_device_error(h, s);
}

rlo_status rlo_forward_logprobs(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits, float* out_logp,
                                float* out_entropy, float* out_token_logit, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "forward_logprobs: null handle");
  RLO_TRY(check_batch(batch, "forward_logprobs", true));
  if ((int64_t)batch->B * batch->T == 0) return RLO_OK;  // an empty batch scores nothing (policy.cpp:219-231)
  RLO_TRY(check_logits(logits, "forward_logprobs", "policy"));
  if (!out_logp) return fail(RLO_ERR_INPUT, "forward_logprobs: out_logp required");
  DeviceGuard g(h->device);
  VocabArgs a;
  std::memset(&a, 0, sizeof(a));
  a.logits[0] = logits->data;
  a.stride[0] = logits->row_stride;
  a.seq_start[0] = logits->seq_start;
  a.role[0] = ROLE_ACTOR;
  a.ntens = 1;
  a.dtype = logits->dtype;
  a.V = logits->V;
  a.B = batch->B;
  a.T = batch->T;
  a.seq_offset = batch->seq_offset;
  a.lengths = batch->lengths;
  a.tokens = batch->tokens;
  a.mask = nullptr;  // forward_logprobs scores every response position (policy.cpp:223-229)
  a.out_lp = out_logp;
  a.out_ent = out_entropy;
  a.out_tok = out_token_logit;
  a.err = h->err.p;
  RLO_CUDA(launch_vocab_logprob(a, h->num_sms, static_cast<cudaStream_t>(stream)));
  return RLO_OK;
}

rlo_status rlo_compute_advantages(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                                  const float* rewards_tok, const float* rewards_seq, const float* values,
                                  float* out_adv, float* out_returns, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "compute_advantages: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));  // policy.cpp:258
  RLO_TRY(check_batch(batch, "compute_advantages", false));
  const int32_t B = batch->B, T = batch->T;
  if ((int64_t)B * T == 0) return RLO_OK;
  if (!out_adv) return fail(RLO_ERR_INPUT, "compute_advantages: out_adv required");
  if (!rewards_tok && !rewards_seq)  // policy.cpp:274-275
    return fail(RLO_ERR_INPUT, "compute_advantages: sample '0' has no rewards");
  if (cfg->adv_estimator == RLO_ADV_GAE && !values)
    return fail(RLO_ERR_INPUT, "compute_advantages: GAE requires critic values");
  if (cfg->adv_estimator == RLO_ADV_GRPO && B % cfg->group_size != 0)
    return fail(RLO_ERR_INPUT, "compute_advantages: batch of " + std::to_string(B) +
                                   " samples is not whole groups of " + std::to_string(cfg->group_size));
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  AdvArgs a;
  std::memset(&a, 0, sizeof(a));
  a.B = B;
  a.T = T;
  a.lengths = batch->lengths;
  a.mask = batch->mask;
  a.rewards_tok = rewards_tok;
  a.rewards_seq = rewards_seq;
  a.values = values;
  a.out_adv = out_adv;
  a.out_returns = out_returns;
  a.estimator = cfg->adv_estimator;
  a.gamma = cfg->gamma;
  a.lambd = cfg->lambd;
  a.reward_clip = cfg->reward_clip;
  a.adv_clip = cfg->advantage_clip;
  a.whiten = cfg->whiten_advantages != 0;
  a.G = cfg->group_size;
  a.ddof = cfg->grpo_std_ddof;
  a.grpo_eps = cfg->grpo_eps;
  const int32_t nslots = cfg->adv_estimator == RLO_ADV_GRPO ? B / cfg->group_size : B;
  if (a.whiten) {
    RLO_CUDA(h->wstat.ensure(static_cast<size_t>(nslots)));
    a.wstat = h->wstat.p;
    RLO_CUDA(h->raw64.ensure(static_cast<size_t>((int64_t)B * T)));
    a.raw64 = h->raw64.p;
  }
  RLO_CUDA(launch_advantages(a, s));
  if (a.whiten) {
    RLO_CUDA(launch_wstat_reduce(h->wstat.p, nslots, h->stats4.p, s));
    const double* stats = h->stats4.p;
    if (h->comm) {  // global whitening: all-gather (sum, sq, count), rank-ordered sum in the kernel
      RLO_NCCL(nccl_api().AllGather(h->stats4.p, h->stats_all.p, 4, ncclFloat64, h->comm, s));
      stats = h->stats_all.p;
    }
    RLO_CUDA(launch_whiten_clip(a, stats, h->comm ? h->world : 1, s));
  }
  return RLO_OK;
}

}  // extern "C"

namespace {

// Validation (policy.cpp:315, :338-343, same order and messages) and the
// VocabArgs of one loss pass; shared by rlo_ppo_gradient and the fused
// update pass.  *empty = true for a batch without positions (nothing to do).
rlo_status ppo_setup(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch, const rlo_logits* actor,
                     const rlo_logits* old_logits, const rlo_logits* ref_logits, const float* old_logp,
                     const float* ref_logp, const float* advantages, const rlo_token_out* out, cudaStream_t s,
                     VocabArgs& a, bool* empty) {
  *empty = true;
  if (!h) return fail(RLO_ERR_INPUT, "ppo_gradient: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));  // policy.cpp:315
  RLO_TRY(check_batch(batch, "ppo_gradient", true));
  const int32_t B = batch->B, T = batch->T;
  const int64_t N = (int64_t)B * T;
  if (N == 0) return RLO_OK;
  *empty = false;
  // policy.cpp:338-343, same order
  if (!advantages) return fail(RLO_ERR_INPUT, "ppo_gradient: sample '0' missing advantages");
  if (!old_logits && !old_logp) return fail(RLO_ERR_INPUT, "ppo_gradient: sample '0' missing old logprobs");
  if (cfg->kl_coef > 0.0 && !ref_logits && !ref_logp)
    return fail(RLO_ERR_INPUT, "ppo_gradient: sample '0' missing ref logprobs");
  RLO_TRY(check_logits(actor, "ppo_gradient", "actor"));
  if (old_logits) RLO_TRY(check_logits(old_logits, "ppo_gradient", "old-policy"));
  if (ref_logits) RLO_TRY(check_logits(ref_logits, "ppo_gradient", "reference"));
  for (const rlo_logits* l : {old_logits, ref_logits})
    if (l && (l->dtype != actor->dtype || l->V != actor->V))
      return fail(RLO_ERR_INPUT, "ppo_gradient: actor/old/ref logits must share dtype and vocab size");
  RLO_CUDA(h->s_loss.ensure(N));
  RLO_CUDA(h->s_ratio.ensure(N));
  RLO_CUDA(h->s_kl.ensure(N));
  RLO_CUDA(h->s_ent.ensure(N));
  RLO_CUDA(h->s_flags.ensure(N));
  const size_t need = static_cast<size_t>(batch->seq_offset) + static_cast<size_t>(B);
  if (need > h->recs.cap) {
    // growing drops accumulated records only if none are pending
    if (h->acc_nseq > 0) {
      std::vector<SeqRec> keep(static_cast<size_t>(h->acc_nseq));
      RLO_CUDA(cudaStreamSynchronize(s));
      RLO_CUDA(cudaMemcpy(keep.data(), h->recs.p, sizeof(SeqRec) * keep.size(), cudaMemcpyDeviceToHost));
      RLO_CUDA(h->recs.ensure(std::max(need, h->recs.cap * 2), true));
      RLO_CUDA(cudaMemcpy(h->recs.p, keep.data(), sizeof(SeqRec) * keep.size(), cudaMemcpyHostToDevice));
    } else {
      RLO_CUDA(h->recs.ensure(std::max(need, h->recs.cap * 2), true));
    }
  }
  h->acc_nseq = std::max<int32_t>(h->acc_nseq, static_cast<int32_t>(need));

  std::memset(&a, 0, sizeof(a));
  int nt = 0;
  auto add = [&](const rlo_logits* l, int role) {
    a.logits[nt] = l->data;
    a.stride[nt] = l->row_stride;
    a.seq_start[nt] = l->seq_start;
    a.role[nt] = role;
    ++nt;
  };
  add(actor, ROLE_ACTOR);
  if (old_logits) add(old_logits, ROLE_OLD);
  if (ref_logits) add(ref_logits, ROLE_REF);
  a.ntens = nt;
  a.dtype = actor->dtype;
  a.V = actor->V;
  a.B = B;
  a.T = T;
  a.seq_offset = batch->seq_offset;
  a.lengths = batch->lengths;
  a.tokens = batch->tokens;
  a.mask = batch->mask;
  a.old_lp_in = old_logits ? nullptr : old_logp;
  a.ref_lp_in = ref_logits ? nullptr : ref_logp;
  a.adv = advantages;
  a.clip_eps = cfg->clip_eps;
  a.kl_coef = cfg->kl_coef;
  a.dual_c = cfg->dual_clip_c;
  a.kl_est = cfg->kl_estimator;
  a.has_ref = (ref_logits || ref_logp) ? 1 : 0;
  if (out) {
    a.o_logp = out->logp;
    a.o_old = out->old_logp;
    a.o_ref = out->ref_logp;
    a.o_ent = out->entropy;
    a.o_dlogp = out->dlogp;
    a.o_loss = out->loss;
    a.o_lse = out->lse;
    a.o_lse64 = out->lse64;
  }
  a.s_loss = h->s_loss.p;
  a.s_ratio = h->s_ratio.p;
  a.s_kl = h->s_kl.p;
  a.s_ent = h->s_ent.p;
  a.s_flags = h->s_flags.p;
  a.err = h->err.p;
  return RLO_OK;
}

}  // namespace

extern "C" {

rlo_status rlo_ppo_gradient(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                            const rlo_logits* actor, const rlo_logits* old_logits, const rlo_logits* ref_logits,
                            const float* old_logp, const float* ref_logp, const float* advantages,
                            const rlo_token_out* out, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "ppo_gradient: null handle");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VocabArgs a;
  bool empty = true;
  RLO_TRY(ppo_setup(h, cfg, batch, actor, old_logits, ref_logits, old_logp, ref_logp, advantages, out, s, a, &empty));
  if (empty) return RLO_OK;
  RLO_CUDA(launch_vocab_loss(a, h->num_sms, s));
  RLO_CUDA(launch_seq_reduce(batch->B, batch->T, batch->seq_offset, batch->lengths, batch->mask, h->s_loss.p,
                             h->s_ratio.p, h->s_kl.p, h->s_ent.p, h->s_flags.p, h->recs.p, s));
  return RLO_OK;
}

rlo_status rlo_ppo_gradient_fused(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                                  const rlo_logits* actor, const rlo_logits* old_logits, const rlo_logits* ref_logits,
                                  const float* old_logp, const float* ref_logp, const float* advantages,
                                  const float* weight, void* grad, int32_t grad_dtype, int64_t grad_row_stride,
                                  const rlo_token_out* out, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "ppo_gradient: null handle");
  if (batch && (int64_t)batch->B * batch->T > 0) {  // before any accumulator state changes
    if (!weight || !grad) return fail(RLO_ERR_INPUT, "ppo_gradient_fused: weight and grad required");
    if (grad_dtype != RLO_DTYPE_F32 && grad_dtype != RLO_DTYPE_BF16)
      return fail(RLO_ERR_INPUT, "ppo_gradient_fused: unsupported grad dtype");
    if (actor && grad_row_stride < actor->V) return fail(RLO_ERR_INPUT, "ppo_gradient_fused: grad row stride < V");
  }
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VocabArgs a;
  bool empty = true;
  RLO_TRY(ppo_setup(h, cfg, batch, actor, old_logits, ref_logits, old_logp, ref_logp, advantages, out, s, a, &empty));
  if (empty) return RLO_OK;
  const int32_t B = batch->B, T = batch->T;
  int32_t slice = 0;
  const int K = fused_cluster_size(a, grad, grad_dtype, grad_row_stride, h->tuning, &slice);
  cudaError_t e = K > 0 ? launch_vocab_fused(a, weight, grad, grad_dtype, grad_row_stride, K, slice, h->tuning, s)
                        : cudaErrorNotSupported;
  if (e != cudaSuccess) {
    // not eligible (unaligned rows, vocab too large for a cluster's shared
    // memory): the two-pass form, loss pass then backward epilogue
    cudaGetLastError();
    const int64_t N = (int64_t)B * T;
    RLO_CUDA(h->s_lse64.ensure(N));
    RLO_CUDA(h->s_dlogp.ensure(N));
    if (!a.o_lse64) a.o_lse64 = h->s_lse64.p;
    if (!a.o_dlogp) a.o_dlogp = h->s_dlogp.p;
    RLO_CUDA(launch_vocab_loss(a, h->num_sms, s));
    RLO_CUDA(launch_logits_backward(actor->data, actor->dtype, actor->row_stride, actor->seq_start, actor->V, B, T,
                                    batch->lengths, batch->tokens, nullptr, a.o_lse64, a.o_dlogp, weight, grad,
                                    grad_dtype, grad_row_stride, h->num_sms, s));
  }
  RLO_CUDA(launch_seq_reduce(B, T, batch->seq_offset, batch->lengths, batch->mask, h->s_loss.p, h->s_ratio.p,
                             h->s_kl.p, h->s_ent.p, h->s_flags.p, h->recs.p, s));
  return RLO_OK;
}

rlo_status rlo_merge_gradients(rlo_handle* h, const rlo_train_config* cfg, rlo_stats* out, rlo_partials* out_partials,
                               void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "merge_gradients: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int32_t nseq = h->acc_nseq;
  if (nseq > 0) {
    RLO_CUDA(launch_batch_reduce(h->recs.p, nseq, cfg->group_size, h->partials.p, s));
  } else {
    RLO_CUDA(cudaMemsetAsync(h->partials.p, 0, sizeof(double) * RLO_NPARTIAL, s));
  }
  const int world = h->comm ? h->world : 1;
  if (h->comm) {
    // all-gather of the per-rank partials, merged below in rank order (policy.cpp:428-436)
    RLO_NCCL(nccl_api().AllGather(h->partials.p, h->gathered.p, RLO_NPARTIAL, ncclFloat64, h->comm, s));
    RLO_CUDA(cudaMemcpyAsync(h->host_gathered, h->gathered.p, sizeof(double) * RLO_NPARTIAL * world,
                             cudaMemcpyDeviceToHost, s));
  } else {
    RLO_CUDA(cudaMemcpyAsync(h->host_gathered, h->partials.p, sizeof(double) * RLO_NPARTIAL, cudaMemcpyDeviceToHost, s));
  }
  RLO_CUDA(cudaMemcpyAsync(h->host_err, h->err.p, sizeof(DevError), cudaMemcpyDeviceToHost, s));
  RLO_CUDA(cudaMemsetAsync(h->err.p, 0xFF, sizeof(DevError), s));
  if (nseq > 0) RLO_CUDA(cudaMemsetAsync(h->recs.p, 0, sizeof(SeqRec) * static_cast<size_t>(nseq), s));
  h->acc_nseq = 0;
  RLO_CUDA(cudaStreamSynchronize(s));
  RLO_TRY(collect_device_error(h, s));
  std::vector<rlo_partials> parts(static_cast<size_t>(world));
  for (int r = 0; r < world; ++r)
    std::memcpy(parts[static_cast<size_t>(r)].v, h->host_gathered + r * RLO_NPARTIAL, sizeof(double) * RLO_NPARTIAL);
  if (out_partials) *out_partials = parts[static_cast<size_t>(h->comm ? h->rank : 0)];
  return rlo_merge_partials(parts.data(), world, cfg, out);
}

rlo_status rlo_merge_gradients_async(rlo_handle* h, const rlo_train_config* cfg, rlo_step_result* out,
                                     void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "merge_gradients: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));
  if (!out) return fail(RLO_ERR_INPUT, "merge_gradients_async: out required");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int32_t nseq = h->acc_nseq;
  if (nseq > 0) {
    RLO_CUDA(launch_batch_reduce(h->recs.p, nseq, cfg->group_size, h->partials.p, s));
  } else {
    RLO_CUDA(cudaMemsetAsync(h->partials.p, 0, sizeof(double) * RLO_NPARTIAL, s));
  }
  const double* parts = h->partials.p;
  int world = 1;
  if (h->comm) {  // all-gather of the per-rank partials, merged in rank order on the device
    RLO_NCCL(nccl_api().AllGather(h->partials.p, h->gathered.p, RLO_NPARTIAL, ncclFloat64, h->comm, s));
    parts = h->gathered.p;
    world = h->world;
  }
  RLO_CUDA(launch_merge_finalize(parts, world, cfg->loss_agg, h->err.p, out, s));
  if (nseq > 0) RLO_CUDA(cudaMemsetAsync(h->recs.p, 0, sizeof(SeqRec) * static_cast<size_t>(nseq), s));
  h->acc_nseq = 0;
  return RLO_OK;
}

rlo_status rlo_step_result_check(const rlo_step_result* r) {
  if (!r) return fail(RLO_ERR_INPUT, "step_result_check: null result");
  switch (r->reason) {
    case 0: return RLO_OK;
    case 1: return fail(RLO_ERR_TRAINING, "merge_gradients: batch contains no loss-participating tokens");
    case 2: return fail(RLO_ERR_TRAINING, "training step aborted: non-finite gradient");
    case 3: return fail(RLO_ERR_TRAINING, "training step aborted: non-finite loss");
    default: {
      return device_error_status(r->dev_error, r->dev_error_value);
    }
  }
}

rlo_status rlo_rank_partials(rlo_handle* h, const rlo_train_config* cfg, rlo_partials* out, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "rank_partials: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int32_t nseq = h->acc_nseq;
  if (nseq > 0) {
    RLO_CUDA(launch_batch_reduce(h->recs.p, nseq, cfg->group_size, h->partials.p, s));
  } else {
    RLO_CUDA(cudaMemsetAsync(h->partials.p, 0, sizeof(double) * RLO_NPARTIAL, s));
  }
  RLO_CUDA(cudaMemcpyAsync(h->host_gathered, h->partials.p, sizeof(double) * RLO_NPARTIAL, cudaMemcpyDeviceToHost, s));
  RLO_CUDA(cudaMemcpyAsync(h->host_err, h->err.p, sizeof(DevError), cudaMemcpyDeviceToHost, s));
  RLO_CUDA(cudaMemsetAsync(h->err.p, 0xFF, sizeof(DevError), s));
  if (nseq > 0) RLO_CUDA(cudaMemsetAsync(h->recs.p, 0, sizeof(SeqRec) * static_cast<size_t>(nseq), s));
  h->acc_nseq = 0;
  RLO_CUDA(cudaStreamSynchronize(s));
  RLO_TRY(collect_device_error(h, s));
  if (out) std::memcpy(out->v, h->host_gathered, sizeof(double) * RLO_NPARTIAL);
  return RLO_OK;
}

rlo_status rlo_objective_step(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch,
                              const float* rewards_tok, const float* rewards_seq, const float* values,
                              const rlo_logits* actor_logits, const rlo_logits* old_logits,
                              const rlo_logits* ref_logits, const float* old_logp, const float* ref_logp,
                              float* out_adv, const rlo_token_out* out, rlo_stats* stats, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "objective_step: null handle");
  RLO_TRY(check_batch(batch, "objective_step", true));
  DeviceGuard g(h->device);
  if (!out_adv) {
    RLO_CUDA(h->h_adv.ensure(static_cast<size_t>((int64_t)batch->B * batch->T)));
    out_adv = h->h_adv.p;
  }
  RLO_TRY(rlo_compute_advantages(h, cfg, batch, rewards_tok, rewards_seq, values, out_adv, nullptr, stream));
  RLO_TRY(rlo_ppo_gradient(h, cfg, batch, actor_logits, old_logits, ref_logits, old_logp, ref_logp, out_adv, out,
                           stream));
  return rlo_merge_gradients(h, cfg, stats, nullptr, stream);
}

rlo_status rlo_objective_step_host(rlo_handle* h, const rlo_train_config* cfg, int32_t B, int32_t T,
                                   const int32_t* lengths, const int32_t* tokens, const uint8_t* mask,
                                   const float* rewards_tok, const float* rewards_seq, const float* values,
                                   const rlo_logits* actor_logits, const rlo_logits* old_logits,
                                   const rlo_logits* ref_logits, const float* old_logp, const float* ref_logp,
                                   float* host_adv_out, float* host_logp_out, rlo_stats* stats, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "objective_step: null handle");
  if (B < 0 || T < 0) return fail(RLO_ERR_INPUT, "objective_step: negative batch shape");
  if ((int64_t)B * T > 0 && (!lengths || !tokens)) return fail(RLO_ERR_INPUT, "objective_step: lengths/tokens missing");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t N = static_cast<size_t>(B) * static_cast<size_t>(T);
  const size_t nB = static_cast<size_t>(B);
  auto up = [&](auto& buf, const auto* src, size_t n) -> cudaError_t {
    using E = std::remove_pointer_t<decltype(buf.p)>;
    if (!src || n == 0) return cudaSuccess;
    cudaError_t e = buf.ensure(n);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(buf.p, src, sizeof(E) * n, cudaMemcpyHostToDevice, s);
  };
  RLO_CUDA(up(h->h_lengths, lengths, nB));
  RLO_CUDA(up(h->h_tokens, tokens, N));
  RLO_CUDA(up(h->h_mask, mask, N));
  RLO_CUDA(up(h->h_rtok, rewards_tok, N));
  RLO_CUDA(up(h->h_rseq, rewards_seq, nB));
  RLO_CUDA(up(h->h_values, values, N));
  RLO_CUDA(up(h->h_old, old_logp, N));
  RLO_CUDA(up(h->h_ref, ref_logp, N));
  RLO_CUDA(h->h_adv.ensure(N));
  RLO_CUDA(h->h_logp.ensure(N));
  rlo_batch batch{B, T, 0, 0, h->h_lengths.p, h->h_tokens.p, mask ? h->h_mask.p : nullptr};
  rlo_token_out out;
  std::memset(&out, 0, sizeof(out));
  out.logp = host_logp_out ? h->h_logp.p : nullptr;
  RLO_TRY(rlo_compute_advantages(h, cfg, &batch, rewards_tok ? h->h_rtok.p : nullptr,
                                 rewards_seq ? h->h_rseq.p : nullptr, values ? h->h_values.p : nullptr, h->h_adv.p,
                                 nullptr, stream));
  RLO_TRY(rlo_ppo_gradient(h, cfg, &batch, actor_logits, old_logits, ref_logits, old_logp ? h->h_old.p : nullptr,
                           ref_logp ? h->h_ref.p : nullptr, h->h_adv.p, &out, stream));
  if (host_adv_out && N) RLO_CUDA(cudaMemcpyAsync(host_adv_out, h->h_adv.p, sizeof(float) * N, cudaMemcpyDeviceToHost, s));
  if (host_logp_out && N)
    RLO_CUDA(cudaMemcpyAsync(host_logp_out, h->h_logp.p, sizeof(float) * N, cudaMemcpyDeviceToHost, s));
  return rlo_merge_gradients(h, cfg, stats, nullptr, stream);  // synchronises the stream
}

rlo_status rlo_objective_step_host_mb(rlo_handle* h, const rlo_train_config* cfg, int32_t B, int32_t T,
                                      int32_t mb_seqs, const int32_t* lengths, const int32_t* tokens,
                                      const uint8_t* mask, const float* rewards_tok, const float* rewards_seq,
                                      const float* values, rlo_logits_fn logits_fn, void* user,
                                      const float* old_logp, const float* ref_logp, float* host_adv_out,
                                      float* host_logp_out, rlo_stats* stats, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "objective_step: null handle");
  if (B < 0 || T < 0) return fail(RLO_ERR_INPUT, "objective_step: negative batch shape");
  if ((int64_t)B * T > 0 && (!lengths || !tokens)) return fail(RLO_ERR_INPUT, "objective_step: lengths/tokens missing");
  if (mb_seqs <= 0) return fail(RLO_ERR_CONFIG, "objective_step: micro-batch size must be positive");
  if (!logits_fn) return fail(RLO_ERR_INPUT, "objective_step: logits callback required");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t N = static_cast<size_t>(B) * static_cast<size_t>(T);
  const size_t nB = static_cast<size_t>(B);
  auto up = [&](auto& buf, const auto* src, size_t n) -> cudaError_t {
    using E = std::remove_pointer_t<decltype(buf.p)>;
    if (!src || n == 0) return cudaSuccess;
    cudaError_t e = buf.ensure(n);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(buf.p, src, sizeof(E) * n, cudaMemcpyHostToDevice, s);
  };
  RLO_CUDA(up(h->h_lengths, lengths, nB));
  RLO_CUDA(up(h->h_tokens, tokens, N));
  RLO_CUDA(up(h->h_mask, mask, N));
  RLO_CUDA(up(h->h_rtok, rewards_tok, N));
  RLO_CUDA(up(h->h_rseq, rewards_seq, nB));
  RLO_CUDA(up(h->h_values, values, N));
  RLO_CUDA(up(h->h_old, old_logp, N));
  RLO_CUDA(up(h->h_ref, ref_logp, N));
  RLO_CUDA(h->h_adv.ensure(N));
  RLO_CUDA(h->h_logp.ensure(N));
  rlo_batch all{B, T, 0, 0, h->h_lengths.p, h->h_tokens.p, mask ? h->h_mask.p : nullptr};
  RLO_TRY(rlo_compute_advantages(h, cfg, &all, rewards_tok ? h->h_rtok.p : nullptr,
                                 rewards_seq ? h->h_rseq.p : nullptr, values ? h->h_values.p : nullptr, h->h_adv.p,
                                 nullptr, stream));
  // a failed micro-batch aborts the step: drop what the earlier ones accumulated
  auto abort_step = [&](rlo_status st) {
    if (h->acc_nseq > 0) cudaMemsetAsync(h->recs.p, 0, sizeof(SeqRec) * static_cast<size_t>(h->acc_nseq), s);
    h->acc_nseq = 0;
    cudaStreamSynchronize(s);
    return st;
  };
  for (int32_t b0 = 0, i = 0; b0 < B; b0 += mb_seqs, ++i) {
    const int32_t nb = std::min(mb_seqs, B - b0);
    const size_t off = static_cast<size_t>(b0) * static_cast<size_t>(T);
    rlo_logits la, lo, lr;
    std::memset(&la, 0, sizeof(la));
    std::memset(&lo, 0, sizeof(lo));
    std::memset(&lr, 0, sizeof(lr));
    const rlo_status cb = logits_fn(user, i, b0, nb, &la, &lo, &lr);
    if (cb != RLO_OK)
      return abort_step(fail(cb, "objective_step: logits callback failed for micro-batch " + std::to_string(i)));
    rlo_batch mb{nb, T, b0, 0, h->h_lengths.p + b0, h->h_tokens.p + off, mask ? h->h_mask.p + off : nullptr};
    rlo_token_out out;
    std::memset(&out, 0, sizeof(out));
    out.logp = host_logp_out ? h->h_logp.p + off : nullptr;
    const rlo_status st = rlo_ppo_gradient(h, cfg, &mb, &la, lo.data ? &lo : nullptr, lr.data ? &lr : nullptr,
                                           old_logp ? h->h_old.p + off : nullptr,
                                           ref_logp ? h->h_ref.p + off : nullptr, h->h_adv.p + off, &out, stream);
    if (st != RLO_OK) return abort_step(st);
  }
  if (host_adv_out && N) RLO_CUDA(cudaMemcpyAsync(host_adv_out, h->h_adv.p, sizeof(float) * N, cudaMemcpyDeviceToHost, s));
  if (host_logp_out && N)
    RLO_CUDA(cudaMemcpyAsync(host_logp_out, h->h_logp.p, sizeof(float) * N, cudaMemcpyDeviceToHost, s));
  return rlo_merge_gradients(h, cfg, stats, nullptr, stream);  // synchronises the stream
}

rlo_status rlo_batch_counts(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch, rlo_stats* out,
                            void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "batch_counts: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));
  RLO_TRY(check_batch(batch, "batch_counts", false));
  if (!out) return fail(RLO_ERR_INPUT, "batch_counts: out required");
  std::memset(out, 0, sizeof(*out));
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RLO_CUDA(h->counts.ensure(static_cast<size_t>(batch->B > 0 ? batch->B : 1)));
  RLO_CUDA(launch_batch_counts(batch->B, batch->T, cfg->group_size, batch->lengths, batch->mask, h->counts.p,
                               h->stats4.p, s));
  const double* src = h->stats4.p;
  int world = 1;
  if (h->comm) {  // global normalisers: all-gather, rank-ordered sum
    RLO_NCCL(nccl_api().AllGather(h->stats4.p, h->stats_all.p, 4, ncclFloat64, h->comm, s));
    src = h->stats_all.p;
    world = h->world;
  }
  std::vector<double> host(static_cast<size_t>(4 * world));
  RLO_CUDA(cudaMemcpyAsync(host.data(), src, sizeof(double) * host.size(), cudaMemcpyDeviceToHost, s));
  RLO_CUDA(cudaStreamSynchronize(s));
  double t = 0.0, q = 0.0, gr = 0.0;
  for (int r = 0; r < world; ++r) {
    t += host[4 * r + 0];
    q += host[4 * r + 1];
    gr += host[4 * r + 2];
  }
  out->tokens = static_cast<uint64_t>(t);
  out->seqs = static_cast<uint64_t>(q);
  out->groups = static_cast<uint64_t>(gr);
  return RLO_OK;
}

rlo_status rlo_loss_weights(rlo_handle* h, const rlo_train_config* cfg, const rlo_batch* batch, const rlo_stats* stats,
                            float* out_w, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "loss_weights: null handle");
  RLO_TRY(rlo_train_config_validate(cfg));
  RLO_TRY(check_batch(batch, "loss_weights", false));
  if (!stats || !out_w) return fail(RLO_ERR_INPUT, "loss_weights: stats and out_w required");
  if (stats->tokens == 0) return fail(RLO_ERR_TRAINING, "merge_gradients: batch contains no loss-participating tokens");
  DeviceGuard g(h->device);
  RLO_CUDA(h->counts.ensure(static_cast<size_t>(batch->B > 0 ? batch->B : 1)));
  RLO_CUDA(launch_loss_weights(batch->B, batch->T, cfg->group_size, cfg->loss_agg, (double)stats->tokens,
                               (double)stats->seqs, (double)stats->groups, batch->lengths, batch->mask, h->counts.p,
                               out_w, static_cast<cudaStream_t>(stream)));
  return RLO_OK;
}

namespace {
rlo_status logits_backward_impl(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits, const float* lse,
                                const double* lse64, const float* dlogp, const float* weight, void* grad,
                                int32_t grad_dtype, int64_t grad_row_stride, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "logits_backward: null handle");
  RLO_TRY(check_batch(batch, "logits_backward", true));
  RLO_TRY(check_logits(logits, "logits_backward", "actor"));
  if ((int64_t)batch->B * batch->T == 0) return RLO_OK;
  if ((!lse && !lse64) || !dlogp || !weight || !grad)
    return fail(RLO_ERR_INPUT, "logits_backward: lse, dlogp, weight, grad required");
  if (grad_dtype != RLO_DTYPE_F32 && grad_dtype != RLO_DTYPE_BF16)
    return fail(RLO_ERR_INPUT, "logits_backward: unsupported grad dtype");
  if (grad_row_stride < logits->V) return fail(RLO_ERR_INPUT, "logits_backward: grad row stride < V");
  DeviceGuard g(h->device);
  RLO_CUDA(launch_logits_backward(logits->data, logits->dtype, logits->row_stride, logits->seq_start, logits->V,
                                  batch->B, batch->T, batch->lengths, batch->tokens, lse, lse64, dlogp, weight, grad,
                                  grad_dtype, grad_row_stride, h->num_sms, static_cast<cudaStream_t>(stream)));
  return RLO_OK;
}
}  // namespace

rlo_status rlo_logits_backward(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits, const float* lse,
                               const float* dlogp, const float* weight, void* grad, int32_t grad_dtype,
                               int64_t grad_row_stride, void* stream) {
  return logits_backward_impl(h, batch, logits, lse, nullptr, dlogp, weight, grad, grad_dtype, grad_row_stride,
                              stream);
}

rlo_status rlo_logits_backward64(rlo_handle* h, const rlo_batch* batch, const rlo_logits* logits,
                                 const double* lse64, const float* dlogp, const float* weight, void* grad,
                                 int32_t grad_dtype, int64_t grad_row_stride, void* stream) {
  return logits_backward_impl(h, batch, logits, nullptr, lse64, dlogp, weight, grad, grad_dtype, grad_row_stride,
                              stream);
}

rlo_status rlo_value_loss(rlo_handle* h, const rlo_batch* batch, const float* values, const float* old_values,
                          const float* returns, double value_clip, float* out_dvalue, rlo_value_stats* out,
                          void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "value_loss: null handle");
  RLO_TRY(check_batch(batch, "value_loss", false));
  const int32_t B = batch->B, T = batch->T;
  if ((int64_t)B * T > 0 && (!values || !returns))  // policy.cpp:497-498
    return fail(RLO_ERR_INPUT, "value_gradient: sample '0' missing targets");
  if (!(value_clip >= 0.0)) return fail(RLO_ERR_CONFIG, "value_loss: value_clip must be non-negative");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  RLO_CUDA(h->vseq.ensure(static_cast<size_t>(4 * (B > 0 ? B : 1))));
  RLO_CUDA(h->vout.ensure(4));
  RLO_CUDA(launch_value_loss(B, T, batch->lengths, batch->mask, values, old_values, returns, value_clip, out_dvalue,
                             h->vseq.p, h->vout.p, s));
  const int world = h->comm ? h->world : 1;
  if (h->comm) {
    RLO_CUDA(h->vgath.ensure(static_cast<size_t>(4 * world)));
    RLO_NCCL(nccl_api().AllGather(h->vout.p, h->vgath.p, 4, ncclFloat64, h->comm, s));
    RLO_CUDA(cudaMemcpyAsync(h->host_gathered, h->vgath.p, sizeof(double) * 4 * world, cudaMemcpyDeviceToHost, s));
  } else {
    RLO_CUDA(cudaMemcpyAsync(h->host_gathered, h->vout.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
  }
  RLO_CUDA(cudaStreamSynchronize(s));
  double sum[4] = {0, 0, 0, 0};
  for (int r = 0; r < world; ++r)  // rank order
    for (int k = 0; k < 4; ++k) sum[k] += h->host_gathered[4 * r + k];
  if (sum[1] == 0.0) return fail(RLO_ERR_TRAINING, "value_loss: batch contains no loss-participating tokens");
  const double inv = 1.0 / sum[1];
  rlo_value_stats st{sum[0] * inv, sum[2] * inv, sum[3] * inv, static_cast<uint64_t>(sum[1])};
  if (!std::isfinite(st.loss)) return fail(RLO_ERR_TRAINING, "value_loss: non-finite loss");
  if (out) *out = st;
  return RLO_OK;
}

rlo_status rlo_decode_sample(rlo_handle* h, const rlo_logits* logits, int32_t n_rows, double temperature,
                             uint64_t seed, uint64_t version, const uint64_t* sample_keys, const uint64_t* positions,
                             int32_t* out_tokens, float* out_logp, void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "decode: null handle");
  if (!(temperature > 0.0)) return fail(RLO_ERR_CONFIG, "decode: temperature must be positive");  // policy.cpp:146
  if (n_rows < 0) return fail(RLO_ERR_INPUT, "decode: negative row count");
  if (n_rows == 0) return RLO_OK;
  RLO_TRY(check_logits(logits, "decode", "policy"));
  if (logits->seq_start) return fail(RLO_ERR_INPUT, "decode: rows are consecutive (seq_start must be NULL)");
  if (!sample_keys || !positions || !out_tokens || !out_logp)
    return fail(RLO_ERR_INPUT, "decode: sample_keys, positions, out_tokens and out_logp are required");
  DeviceGuard g(h->device);
  RLO_CUDA(launch_decode(logits->data, logits->dtype, logits->row_stride, logits->V, n_rows, temperature, seed, version,
                         sample_keys, positions, out_tokens, out_logp, h->num_sms, h->tuning,
                         static_cast<cudaStream_t>(stream)));
  return RLO_OK;
}

rlo_status rlo_bucket_plan(uint64_t total, uint64_t bucket, uint64_t* out, int64_t* n_buckets) {
  // bucket_plan, policy.cpp:542-548
  if (bucket == 0) return fail(RLO_ERR_CONFIG, "bucket_plan: bucket_size must be positive");
  if (!n_buckets) return fail(RLO_ERR_INPUT, "bucket_plan: null count");
  const int64_t need = total == 0 ? 1 : static_cast<int64_t>((total + bucket - 1) / bucket);
  const int64_t room = *n_buckets;
  *n_buckets = need;
  if (!out || room < need) return fail(RLO_ERR_INPUT, "bucket_plan: output has room for fewer buckets than needed");
  if (total == 0) {
    out[0] = 0;
    return RLO_OK;
  }
  int64_t i = 0;
  for (uint64_t off = 0; off < total; off += bucket) out[i++] = std::min(bucket, total - off);
  return RLO_OK;
}

rlo_status rlo_broadcast_params(rlo_handle* h, void* buffer, uint64_t bytes, uint64_t bucket_bytes, int32_t root,
                                void* stream) {
  if (!h) return fail(RLO_ERR_INPUT, "broadcast_params: null handle");
  if (bucket_bytes == 0) return fail(RLO_ERR_CONFIG, "sync_params: bucket_size must be positive");  // policy_workers.cpp:235
  if (root < 0 || root >= (h->comm ? h->world : 1)) return fail(RLO_ERR_CONFIG, "broadcast_params: root out of range");
  if (!h->comm || bytes == 0) return RLO_OK;  // a group of one already holds the parameters
  if (!buffer) return fail(RLO_ERR_INPUT, "broadcast_params: null buffer");
  DeviceGuard g(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* p = static_cast<char*>(buffer);
  for (uint64_t off = 0; off < bytes; off += bucket_bytes) {  // contiguous buckets, bucket_plan order
    const uint64_t n = std::min(bucket_bytes, bytes - off);
    RLO_NCCL(nccl_api().Broadcast(p + off, p + off, n, ncclUint8, root, h->comm, s));
  }
  return RLO_OK;
}

uint64_t rlo_sample_key(const char* sample_id) {  // rng::hash_str, FNV-1a 64
  uint64_t hsh = 0xcbf29ce484222325ULL;
  for (const unsigned char* c = reinterpret_cast<const unsigned char*>(sample_id); c && *c; ++c) {
    hsh ^= *c;
    hsh *= 0x100000001b3ULL;
  }
  return hsh;
}

rlo_status rlo_synth_logits(void* dst, int32_t dtype, int64_t rows, int32_t V, int64_t row_stride, uint64_t seed,
                            int32_t model_id, int64_t row_key_offset, void* stream) {
  if (!dst && rows > 0) return fail(RLO_ERR_INPUT, "synth_logits: null destination");
  if (V <= 0 || V > 262144 || row_stride < V) return fail(RLO_ERR_INPUT, "synth_logits: V must be in [1, 2^18]");
  if (dtype != RLO_DTYPE_F32 && dtype != RLO_DTYPE_BF16) return fail(RLO_ERR_INPUT, "synth_logits: bad dtype");
  RLO_CUDA(launch_synth_logits(dst, dtype, rows, V, row_stride, seed, model_id, row_key_offset,
                               static_cast<cudaStream_t>(stream)));
  return RLO_OK;
}

rlo_status rlo_synth_tokens(int32_t* dst, int64_t rows, int32_t V, uint64_t seed, int64_t row_key_offset,
                            int64_t key_rows, void* stream) {
  if (!dst && rows > 0) return fail(RLO_ERR_INPUT, "synth_tokens: null destination");
  if (V <= 0 || key_rows <= 0) return fail(RLO_ERR_INPUT, "synth_tokens: V and key_rows must be positive");
  RLO_CUDA(launch_synth_tokens(dst, rows, V, seed, row_key_offset, key_rows, static_cast<cudaStream_t>(stream)));
  return RLO_OK;
}

}  // extern "C"
