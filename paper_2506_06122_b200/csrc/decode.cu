// decode.cu — sampling-time log-probs: decode_next
// (policy.cpp:143-169) for a batch of rows.  The reference draws a token by a
// CDF walk in token-id order over the tempered softmax with the keyed uniform
// u = keyed_double({seed, version, sample_key, position}) (rng.hpp:22-31,
// 82-85) and returns the token with its UNtempered log-prob (:168) — the
// "old" log-prob of the PPO ratio, so emitting it here removes the separate
// old-policy logits pass (P = 3 -> 2).
//
// One CTA per row, 8 warps; warp j owns the contiguous token range
// [j*W, (j+1)*W) (lane-strided inside, so loads stay coalesced).
//   pass 1: per warp, online max + fp64 tempered sum sum exp((z-m)/T) and
//           untempered sum sum exp(z-m) (fp64 exp: the reference's precision);
//   combine: thread 0 rescales the warp sums to the row max in warp order,
//           forms the row totals and the warp prefix, and finds the warp whose
//           range holds the crossing of u * total;
//   pass 2: that warp re-reads its range in 32-element chunks, warp prefix
//           sums (shfl), and takes the first token whose cumulative tempered
//           mass exceeds the threshold — the reference's first `u < acc`.
// Traffic per row ~ (1 + 1/8) x V x s; latency-bound at decode batch sizes.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

constexpr int kDecWarps = 8;

// rng::mix / keyed_double (rng.hpp:15-31, 82-85), restated bit-for-bit.
__device__ __forceinline__ uint64_t splitmix(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double keyed_double4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t state = 0x2545f4914f6cdd1dULL;
  uint64_t h = splitmix(state);
  const uint64_t keys[4] = {a, b, c, d};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    state ^= keys[k];
    h ^= splitmix(state);
  }
  return (double)(h >> 11) * 0x1.0p-53;
}

template <typename ET>
__device__ __forceinline__ double logit(const ET* p, int v);
template <>
__device__ __forceinline__ double logit<float>(const float* p, int v) {
  return (double)__ldg(p + v);
}
template <>
__device__ __forceinline__ double logit<__nv_bfloat16>(const __nv_bfloat16* p, int v) {
  return (double)__bfloat162float(p[v]);
}

template <typename ET>
__global__ void __launch_bounds__(kDecWarps * 32)
    decode_kernel(const ET* __restrict__ logits, int64_t stride, int V, int n, double temp, uint64_t seed,
                  uint64_t version, const uint64_t* __restrict__ keys, const uint64_t* __restrict__ positions,
                  int32_t* __restrict__ out_tok, float* __restrict__ out_lp) {
  __shared__ double s_m[kDecWarps], s_t[kDecWarps], s_u[kDecWarps];
  __shared__ double s_base, s_thresh, s_m_row;
  __shared__ int s_warp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int W = ((V + kDecWarps - 1) / kDecWarps + 31) / 32 * 32;
  for (int row = blockIdx.x; row < n; row += gridDim.x) {
    const ET* z = logits + (int64_t)row * stride;
    const int v0 = warp * W, v1 = min(V, v0 + W);
    // pass 1: online max + fp64 sums over the warp's range
    double m = -INFINITY, st = 0.0, su = 0.0;
    for (int v = v0 + lane; v < v1; v += 32) {
      const double x = logit(z, v);
      if (x > m) {
        if (m != -INFINITY) {
          st *= exp((m - x) / temp);
          su *= exp(m - x);
        }
        m = x;
      }
      st += exp((x - m) / temp);
      su += exp(x - m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // warp combine (max, rescaled sums)
      const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const double t2 = __shfl_xor_sync(0xffffffffu, st, o);
      const double u2 = __shfl_xor_sync(0xffffffffu, su, o);
      const double M = fmax(m, m2);
      if (M != -INFINITY) {
        st = (m == -INFINITY ? 0.0 : st * exp((m - M) / temp)) + (m2 == -INFINITY ? 0.0 : t2 * exp((m2 - M) / temp));
        su = (m == -INFINITY ? 0.0 : su * exp(m - M)) + (m2 == -INFINITY ? 0.0 : u2 * exp(m2 - M));
      }
      m = M;
    }
    if (lane == 0) {
      s_m[warp] = m;
      s_t[warp] = st;
      s_u[warp] = su;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double M = -INFINITY;
      for (int j = 0; j < kDecWarps; ++j) M = fmax(M, s_m[j]);
      double T = 0.0, U = 0.0;
      for (int j = 0; j < kDecWarps; ++j) {
        if (s_m[j] == -INFINITY) {
          s_t[j] = 0.0;
          continue;
        }
        s_t[j] *= exp((s_m[j] - M) / temp);
        T += s_t[j];
        U += s_u[j] * exp(s_m[j] - M);
      }
      const double u = keyed_double4(seed, version, keys[row], positions[row]);  // policy.cpp:158
      const double X = u * T;
      double base = 0.0;
      int jw = -1;
      for (int j = 0; j < kDecWarps; ++j) {
        if (X < base + s_t[j]) {
          jw = j;
          break;
        }
        base += s_t[j];
      }
      s_warp = jw;
      s_base = base;
      s_thresh = X;
      s_m_row = M;
      s_u[0] = M + log(U);  // untempered lse (policy.cpp:117-121)
    }
    __syncthreads();
    const int jw = s_warp;
    int chosen = V - 1;  // policy.cpp:160: no crossing -> last token
    if (warp == jw) {
      const double M = s_m_row, X = s_thresh;
      double acc = s_base;
      const int a0 = jw * W, a1 = min(V, a0 + W);
      for (int c = a0; c < a1; c += 32) {
        const int v = c + lane;
        double p = v < a1 ? exp((logit(z, v) - M) / temp) : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // inclusive prefix
          const double q = __shfl_up_sync(0xffffffffu, p, o);
          if (lane >= o) p += q;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, v < a1 && X < acc + p);
        if (hit) {
          chosen = c + __ffs(hit) - 1;
          break;
        }
        acc += __shfl_sync(0xffffffffu, p, 31);
      }
      // a crossing placed in this warp by the rescaled totals but missed by the
      // in-order prefix (rounding at a CDF boundary): the range's last token
      if (lane == 0) s_warp = chosen == V - 1 ? a1 - 1 : chosen;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      chosen = jw < 0 ? V - 1 : s_warp;
      out_tok[row] = chosen;
      out_lp[row] = (float)(logit(z, chosen) - s_u[0]);  // untempered logp (policy.cpp:168)
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_decode(const void* logits, int32_t dtype, int64_t stride, int32_t V, int32_t n, double temperature,
                          uint64_t seed, uint64_t version, const uint64_t* keys, const uint64_t* positions,
                          int32_t* out_tok, float* out_lp, int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = n < num_sms * 8 ? n : num_sms * 8;
  if (dtype == RLO_DTYPE_BF16)
    decode_kernel<__nv_bfloat16><<<grid, kDecWarps * 32, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(logits), stride,
                                                                  V, n, temperature, seed, version, keys,
                                                                  positions, out_tok, out_lp);
  else
    decode_kernel<float><<<grid, kDecWarps * 32, 0, s>>>(reinterpret_cast<const float*>(logits), stride, V, n,
                                                         temperature, seed, version, keys, positions, out_tok,
                                                         out_lp);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace rlo
