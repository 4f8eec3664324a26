// advantages.cu — K2: advantage estimators over the padded [B, T] batch.
//
// Replaces compute_advantages (policy.cpp:257-311) and adds the ROLL GRPO and
// GAE estimators.  O(N) work in fp64:
//   * REINFORCE / GAE: one CTA per sequence; each thread owns a contiguous
//     chunk, computes its chunk's reverse discounted sum assuming a zero
//     carry, the CTA scans the (sum, c^len) affine maps right-to-left with
//     warp shuffles + shared memory, then each thread replays its chunk from
//     its carry-in.  c = gamma (REINFORCE) or gamma*lambda (GAE).  The
//     reference's semantics are kept: every position t < length is scanned,
//     including mask-0 (environment) positions (policy.cpp:280-283).
//   * GRPO: one CTA per group of G contiguous sequences (scheduler.cpp:460-469).
//   * whitening: per-slot fp64 (sum, sum^2, count) over masked positions
//     (policy.cpp:288-298); a one-CTA fixed-order reduction; then a
//     normalise+clip pass that combines the world's statistics in rank order.
#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

constexpr int kScanThreads = 256;

__device__ __forceinline__ double reward_at(const AdvArgs& a, int b, int t, int n) {
  double r;
  if (a.rewards_tok)
    r = (double)a.rewards_tok[(int64_t)b * a.T + t];
  else
    r = (t == n - 1) ? (double)a.rewards_seq[b] : 0.0;  // scalar reward on the last token, policy.cpp:268-270
  return clampd(r, -a.reward_clip, a.reward_clip);     // policy.cpp:277
}

__device__ __forceinline__ double delta_at(const AdvArgs& a, int b, int t, int n, bool gae) {
  const double r = reward_at(a, b, t, n);
  if (!gae) return r;
  const float* v = a.values + (int64_t)b * a.T;
  const double next_v = (t + 1 < n) ? (double)v[t + 1] : 0.0;
  return r + a.gamma * next_v - (double)v[t];
}

// Block-wide reduction of 3 doubles (fixed shuffle/smem order: deterministic).
__device__ void block_sum3(double& x, double& y, double& z, double* sm /*[3*32]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  x = warp_sum(x);
  y = warp_sum(y);
  z = warp_sum(z);
  __syncthreads();
  if (lane == 0) {
    sm[warp] = x;
    sm[32 + warp] = y;
    sm[64 + warp] = z;
  }
  __syncthreads();
  if (warp == 0) {
    x = lane < nw ? sm[lane] : 0.0;
    y = lane < nw ? sm[32 + lane] : 0.0;
    z = lane < nw ? sm[64 + lane] : 0.0;
    x = warp_sum(x);
    y = warp_sum(y);
    z = warp_sum(z);
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_kernel(const AdvArgs a) {
  __shared__ double s_sum[kScanThreads / 32], s_pow[kScanThreads / 32];
  __shared__ double s_red[96];
  const int b = blockIdx.x;
  const int n = seq_len(a.lengths, b, a.T);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool gae = a.estimator == RLO_ADV_GAE;
  const double c = gae ? a.gamma * a.lambd : a.gamma;
  const int L = (n + kScanThreads - 1) / kScanThreads;
  const int t0 = min(n, tid * L), t1 = min(n, t0 + L);
  // 1) local reverse sum with zero carry, and c^len
  double acc = 0.0, pw = 1.0;
  for (int t = t1 - 1; t >= t0; --t) {
    acc = delta_at(a, b, t, n, gae) + c * acc;
    pw *= c;
  }
  // 2) right-to-left exclusive scan of affine maps x -> acc + pw * x
  //    carry_i = sum_{j>i} (prod_{i<k<j} pw_k) acc_j
  double S = acc, P = pw;  // inclusive suffix composition within the warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double S2 = __shfl_down_sync(0xffffffffu, S, o);
    const double P2 = __shfl_down_sync(0xffffffffu, P, o);
    if (lane + o < 32) {
      S = S + P * S2;
      P = P * P2;
    }
  }
  if (lane == 0) {
    s_sum[warp] = S;
    s_pow[warp] = P;
  }
  __syncthreads();
  // carry from warps to the right of this one
  double wc = 0.0;
  for (int w = kScanThreads / 32 - 1; w > warp; --w) wc = s_sum[w] + s_pow[w] * wc;
  // exclusive within warp: the composition of lanes > lane applied to wc
  double Sx = __shfl_down_sync(0xffffffffu, S, 1);
  double Px = __shfl_down_sync(0xffffffffu, P, 1);
  if (lane == 31) {
    Sx = 0.0;
    Px = 1.0;
  }
  double carry = Sx + Px * wc;
  // 3) replay the chunk from its carry-in
  double ssum = 0.0, ssq = 0.0, scnt = 0.0;
  acc = carry;
  const float* vv = a.values ? a.values + (int64_t)b * a.T : nullptr;
  for (int t = t1 - 1; t >= t0; --t) {
    acc = delta_at(a, b, t, n, gae) + c * acc;
    const int64_t i = (int64_t)b * a.T + t;
    if (a.out_returns) a.out_returns[i] = (float)(gae ? acc + (double)vv[t] : acc);
    if (a.whiten) {
      a.raw64[i] = acc;  // raw fp64; normalised + clipped by whiten_clip_kernel (fp32 storage would
                         // amplify rounding by 1/std when the masked variance is tiny)
      if (!a.mask || a.mask[i]) {
        ssum += acc;
        ssq += acc * acc;
        scnt += 1.0;
      }
    } else {
      a.out_adv[i] = (float)clampd(acc, -a.adv_clip, a.adv_clip);  // policy.cpp:308-309
    }
  }
  // padding positions are written as 0
  for (int t = n + tid; t < a.T; t += kScanThreads) {
    a.out_adv[(int64_t)b * a.T + t] = 0.f;
    if (a.out_returns) a.out_returns[(int64_t)b * a.T + t] = 0.f;
  }
  if (a.whiten) {
    block_sum3(ssum, ssq, scnt, s_red);
    if (tid == 0) a.wstat[b] = WStat{ssum, ssq, scnt, 0.0};
  }
}

__global__ void __launch_bounds__(kScanThreads) grpo_kernel(const AdvArgs a) {
  extern __shared__ double R[];  // [G]
  __shared__ double s_red[96];
  __shared__ double s_mean, s_sd;
  const int g = blockIdx.x;
  const int G = a.G;
  const int tid = threadIdx.x;
  for (int k = 0; k < G; ++k) {
    const int b = g * G + k;
    double x;
    if (a.rewards_seq) {
      x = (double)a.rewards_seq[b];
    } else {
      x = 0.0;
      double y = 0.0, z = 0.0;
      for (int t = tid; t < seq_len(a.lengths, b, a.T); t += kScanThreads) x += (double)a.rewards_tok[(int64_t)b * a.T + t];
      block_sum3(x, y, z, s_red);
    }
    if (tid == 0) R[k] = clampd(x, -a.reward_clip, a.reward_clip);
  }
  __syncthreads();
  if (tid == 0) {
    double mean = 0.0;
    for (int k = 0; k < G; ++k) mean += R[k];
    mean /= (double)G;
    double ss = 0.0;
    for (int k = 0; k < G; ++k) ss += (R[k] - mean) * (R[k] - mean);
    const int dof = G - a.ddof;
    s_mean = mean;
    s_sd = dof > 0 ? sqrt(ss / (double)dof) : 0.0;
  }
  __syncthreads();
  double ssum = 0.0, ssq = 0.0, scnt = 0.0;
  for (int k = 0; k < G; ++k) {
    const int b = g * G + k;
    const int n = seq_len(a.lengths, b, a.T);
    const double adv = (R[k] - s_mean) / (s_sd + a.grpo_eps);
    const float outv = a.whiten ? (float)adv : (float)clampd(adv, -a.adv_clip, a.adv_clip);
    for (int t = tid; t < a.T; t += kScanThreads) {
      const int64_t i = (int64_t)b * a.T + t;
      const bool valid = t < n;
      a.out_adv[i] = valid ? outv : 0.f;
      if (a.whiten) a.raw64[i] = valid ? adv : 0.0;
      if (a.out_returns) a.out_returns[i] = valid ? (float)R[k] : 0.f;
      if (a.whiten && valid && (!a.mask || a.mask[i])) {
        ssum += adv;
        ssq += adv * adv;
        scnt += 1.0;
      }
    }
  }
  if (a.whiten) {
    block_sum3(ssum, ssq, scnt, s_red);
    if (tid == 0) a.wstat[g] = WStat{ssum, ssq, scnt, 0.0};
  }
}

__global__ void __launch_bounds__(1024) wstat_reduce_kernel(const WStat* __restrict__ w, int n, double* out4) {
  __shared__ double s_red[96];
  double x = 0.0, y = 0.0, z = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    x += w[i].sum;
    y += w[i].sq;
    z += w[i].count;
  }
  block_sum3(x, y, z, s_red);
  if (threadIdx.x == 0) {
    out4[0] = x;
    out4[1] = y;
    out4[2] = z;
    out4[3] = 0.0;
  }
}

// Whitening over the world's statistics (rank-ordered sum of stats_all[r*4..]),
// policy.cpp:299-305, then the advantage clip, policy.cpp:308-309.
__global__ void whiten_clip_kernel(const AdvArgs a, const double* __restrict__ stats_all, int world) {
  __shared__ double s_mean, s_inv;
  __shared__ int s_apply;
  if (threadIdx.x == 0) {
    double mean = 0.0, inv = 1.0;
    s_apply = whiten_combine(stats_all, world, &mean, &inv);
    s_mean = mean;
    s_inv = inv;
  }
  __syncthreads();
  const int64_t N = (int64_t)a.B * a.T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / a.T), t = (int)(i - (int64_t)b * a.T);
    if (t >= seq_len(a.lengths, b, a.T)) continue;
    double v = a.raw64[i];
    if (s_apply) v = (v - s_mean) * s_inv;
    a.out_adv[i] = (float)clampd(v, -a.adv_clip, a.adv_clip);
  }
}

}  // namespace

cudaError_t launch_advantages(const AdvArgs& a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  if (a.estimator == RLO_ADV_GRPO) {
    const int groups = a.B / a.G;
    grpo_kernel<<<groups, kScanThreads, sizeof(double) * (size_t)a.G, s>>>(a);
  } else {
    scan_kernel<<<a.B, kScanThreads, 0, s>>>(a);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_wstat_reduce(const WStat* w, int32_t n, double* out4, cudaStream_t s) {
  wstat_reduce_kernel<<<1, 1024, 0, s>>>(w, n, out4);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_whiten_clip(const AdvArgs& a, const double* stats_all, int32_t world, cudaStream_t s) {
  const int64_t N = (int64_t)a.B * a.T;
  if (N == 0) return cudaSuccess;
  int64_t blocks = (N + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  whiten_clip_kernel<<<(int)blocks, 256, 0, s>>>(a, stats_all, world);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace rlo
