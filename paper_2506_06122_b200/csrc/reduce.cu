// reduce.cu — K4: deterministic reductions of the loss pass.
//
// The reference accumulates GradAccum scalars in token order and merges
// ranks in rank order (policy.cpp:366-370, :428-436; SPEC.md:278 fixed
// reduction order).  Here: per-token results (vocab.cu) -> one CTA per
// sequence sums its tokens in fp64 (thread-strided, butterfly, warps in
// order: a fixed order) -> one CTA reduces the sequence records into the
// rank's partials, including
// the sequence- and group-level aggregation sums.  No floating-point atomics
// anywhere, so results are bitwise reproducible run to run.
#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

constexpr int kSeqThreads = 256;  // one CTA per sequence: long responses (T up to 16384) stay parallel

__global__ void __launch_bounds__(kSeqThreads)
    seq_reduce_kernel(int B, int T, int seq_offset, const int32_t* __restrict__ lengths,
                      const uint8_t* __restrict__ mask, const float* __restrict__ s_loss,
                      const float* __restrict__ s_ratio, const float* __restrict__ s_kl,
                      const float* __restrict__ s_ent, const uint8_t* __restrict__ s_flags, SeqRec* recs) {
  __shared__ double sm[9][kSeqThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x;
  const int n = seq_len(lengths, b, T);
  double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // loss ratio kl ent | clipped dual tokens nfg nfl
  int c[5] = {0, 0, 0, 0, 0};
  for (int t = threadIdx.x; t < n; t += kSeqThreads) {
    const int64_t i = (int64_t)b * T + t;
    if (mask && !mask[i]) continue;
    const uint8_t f = s_flags[i];
    v[0] += (double)s_loss[i];
    v[1] += (double)s_ratio[i];
    v[2] += (double)s_kl[i];
    v[3] += (double)s_ent[i];
    c[0] += (f & TF_CLIPPED) ? 1 : 0;
    c[1] += (f & TF_DUAL) ? 1 : 0;
    c[2] += 1;
    c[3] += (f & TF_NONFINITE_GRAD) ? 1 : 0;
    c[4] += (f & TF_NONFINITE_LOSS) ? 1 : 0;
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) v[4 + k] = (double)c[k];
#pragma unroll
  for (int k = 0; k < 9; ++k) {  // fixed shuffle tree, then warps in order: deterministic
    v[k] = warp_sum(v[k]);
    if (lane == 0) sm[k][warp] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r[9];
    for (int k = 0; k < 9; ++k) {
      r[k] = 0.0;
      for (int w = 0; w < kSeqThreads / 32; ++w) r[k] += sm[k][w];
    }
    recs[seq_offset + b] = SeqRec{r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8], 0.0};
  }
}

constexpr int kBR = 1024;
constexpr int kNV = 13;

__global__ void __launch_bounds__(kBR) batch_reduce_kernel(const SeqRec* __restrict__ recs, int nseq, int G,
                                                           double* partials) {
  __shared__ double sm[kNV][32];
  double v[kNV];
#pragma unroll
  for (int k = 0; k < kNV; ++k) v[k] = 0.0;
  for (int b = threadIdx.x; b < nseq; b += kBR) {
    const SeqRec r = recs[b];
    v[RLO_P_LOSS_SUM] += r.loss;
    v[RLO_P_RATIO_SUM] += r.ratio;
    v[RLO_P_KL_SUM] += r.kl;
    v[RLO_P_ENTROPY_SUM] += r.entropy;
    v[RLO_P_CLIPPED] += r.clipped;
    v[RLO_P_DUAL_CLIPPED] += r.dual;
    v[RLO_P_TOKENS] += r.tokens;
    v[RLO_P_NONFINITE_GRAD] += r.nonfinite_grad;
    v[RLO_P_NONFINITE_LOSS] += r.nonfinite_loss;
    if (r.tokens > 0.0) {
      v[RLO_P_SEQ_MEAN_SUM] += r.loss / r.tokens;
      v[RLO_P_SEQS] += 1.0;
    }
  }
  const int ngroups = (nseq + G - 1) / G;
  for (int g = threadIdx.x; g < ngroups; g += kBR) {
    double gl = 0.0, gt = 0.0;
    const int e = min(nseq, (g + 1) * G);
    for (int b = g * G; b < e; ++b) {
      gl += recs[b].loss;
      gt += recs[b].tokens;
    }
    if (gt > 0.0) {
      v[RLO_P_GROUP_MEAN_SUM] += gl / gt;
      v[RLO_P_GROUPS] += 1.0;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kNV; ++k) {
    v[k] = warp_sum(v[k]);
    if (lane == 0) sm[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < kNV; ++k) {
      double x = sm[k][lane];
      x = warp_sum(x);
      if (lane == 0) partials[k] = x;
    }
    if (lane < RLO_NPARTIAL - kNV) partials[kNV + lane] = 0.0;
  }
}

// One thread: rank-ordered merge of the all-gathered partials into the step
// result (rlo_merge_gradients_async), plus the device error slot, which it
// then clears for the next step.
__global__ void merge_finalize_kernel(const double* __restrict__ parts, int world, int agg, DevError* err,
                                      rlo_step_result* out) {
  rlo_step_result r;
  r.stats = rlo_stats{};
  dev_err_decode(err->key, &r.dev_error, &r.dev_error_value);
  r.reason = r.dev_error ? 4 : merge_stats(parts, world, agg, &r.stats);
  r.status = r.reason == 0 ? RLO_OK : r.reason == 4 ? RLO_ERR_INPUT : RLO_ERR_TRAINING;
  *out = r;
  err->key = kDevErrNone;
}

}  // namespace

cudaError_t launch_merge_finalize(const double* parts, int32_t world, int32_t agg, DevError* err,
                                  rlo_step_result* out, cudaStream_t s) {
  merge_finalize_kernel<<<1, 1, 0, s>>>(parts, world, agg, err, out);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_seq_reduce(int32_t B, int32_t T, int32_t seq_offset, const int32_t* lengths,
                              const uint8_t* mask, const float* s_loss, const float* s_ratio,
                              const float* s_kl, const float* s_ent, const uint8_t* s_flags, SeqRec* recs,
                              cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  seq_reduce_kernel<<<B, kSeqThreads, 0, s>>>(
      B, T, seq_offset, lengths, mask, s_loss, s_ratio, s_kl, s_ent, s_flags, recs);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_batch_reduce(const SeqRec* recs, int32_t nseq, int32_t G, double* partials, cudaStream_t s) {
  batch_reduce_kernel<<<1, kBR, 0, s>>>(recs, nseq, G < 1 ? 1 : G, partials);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace rlo
