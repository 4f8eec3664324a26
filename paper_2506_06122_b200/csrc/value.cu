// value.cu — critic value loss: value_gradient
// (policy.cpp:474-540) per loss-participating token, err = v - return,
// loss 0.5*err^2, d/dv = err; optionally the clipped PPO value loss.  One warp
// per sequence (fp64 sums, fixed order), one CTA for the batch; the ranks'
// partials are merged in rank order by the host (api.cpp).
#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

__global__ void value_seq_kernel(int B, int T, const int32_t* __restrict__ lengths, const uint8_t* __restrict__ mask,
                                 const float* __restrict__ values, const float* __restrict__ old_values,
                                 const float* __restrict__ returns, double clip, float* __restrict__ dv,
                                 double* __restrict__ seqsums /*[B][4]*/) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (b >= B) return;
  const int n = seq_len(lengths, b, T);
  double loss = 0.0, tokens = 0.0, clipped = 0.0, vsum = 0.0;
  for (int t = lane; t < T; t += 32) {
    const int64_t i = (int64_t)b * T + t;
    float d = 0.f;
    if (t < n && (!mask || mask[i])) {  // policy.cpp:501-504
      const double v = (double)values[i], R = (double)returns[i];
      const double err = v - R;  // :508
      double l = 0.5 * err * err, g = err;
      if (old_values && clip > 0.0) {
        const double dvv = v - (double)old_values[i];
        const double vc = (double)old_values[i] + clampd(dvv, -clip, clip);
        const double lc = 0.5 * (vc - R) * (vc - R);
        if (lc > l) {
          l = lc;
          g = (dvv > -clip && dvv < clip) ? vc - R : 0.0;
          clipped += 1.0;
        }
      }
      loss += l;      // :509
      tokens += 1.0;  // :510
      vsum += v;
      d = (float)g;   // :512
    }
    if (dv) dv[i] = d;
  }
  loss = warp_sum(loss);
  tokens = warp_sum(tokens);
  clipped = warp_sum(clipped);
  vsum = warp_sum(vsum);
  if (lane == 0) {
    seqsums[4 * b + 0] = loss;
    seqsums[4 * b + 1] = tokens;
    seqsums[4 * b + 2] = clipped;
    seqsums[4 * b + 3] = vsum;
  }
}

__global__ void __launch_bounds__(1024) value_batch_kernel(int B, const double* __restrict__ seqsums, double* out4) {
  __shared__ double sm[4][32];
  double v[4] = {0, 0, 0, 0};
  for (int b = threadIdx.x; b < B; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] += seqsums[4 * b + k];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = warp_sum(v[k]);
    if (lane == 0) sm[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double x = lane < (int)(blockDim.x >> 5) ? sm[k][lane] : 0.0;
      x = warp_sum(x);
      if (lane == 0) out4[k] = x;
    }
  }
}

}  // namespace

cudaError_t launch_value_loss(int32_t B, int32_t T, const int32_t* lengths, const uint8_t* mask, const float* values,
                              const float* old_values, const float* returns, double clip, float* dv,
                              double* seqsums, double* out4, cudaStream_t s) {
  if (B > 0) value_seq_kernel<<<(B + 7) / 8, 256, 0, s>>>(B, T, lengths, mask, values, old_values, returns, clip, dv,
                                                        seqsums);
  value_batch_kernel<<<1, 1024, 0, s>>>(B, seqsums, out4);
  g_launches.fetch_add(B > 0 ? 2 : 1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace rlo
