// backward.cu — the callers after the loss: the
// aggregation weights d(L)/d(loss_t) and the actor backward epilogue
// dlogits = w*dlogp*(onehot - softmax) (policy.cpp:375-379).
//
// logits_backward_kernel streams each row once (128-bit loads, the same
// persistent 256-thread layout as the LDG vocab pass), recomputes
// p_v = 2^(z_v*log2e - lse*log2e) from the forward pass's lse, and writes the
// gradient row with streaming 128-bit stores (fp32 or bf16).  HBM-bound:
// V*(s_in + s_out) bytes per row.
#include <cuda_bf16.h>

#include "common.cuh"
#include "grad_io.cuh"
#include "internal.h"

namespace rlo {
namespace {

#ifndef RLO_BW_THREADS
#define RLO_BW_THREADS 256
#endif
constexpr int kBwThreads = RLO_BW_THREADS;
// RLO_BW256 = 1 (default): bf16 -> bf16 rows as 32-byte vector pairs (LDG.256 +
// STG.256): +3.4% on the Qwen-vocabulary backward (profiles/r2_update_step.txt).
#ifndef RLO_BW256
#define RLO_BW256 1
#endif

__global__ void seq_count_kernel(int B, int T, const int32_t* __restrict__ lengths, const uint8_t* __restrict__ mask,
                                 float* __restrict__ counts) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (b >= B) return;
  const int n = seq_len(lengths, b, T);
  int c = 0;
  for (int t = lane; t < n; t += 32) c += (!mask || mask[(int64_t)b * T + t]) ? 1 : 0;
  c = warp_sum(c);
  if (lane == 0) counts[b] = (float)c;
}

__global__ void loss_weight_kernel(int B, int T, int G, int agg, double tokens, double seqs, double groups,
                                   const int32_t* __restrict__ lengths, const uint8_t* __restrict__ mask,
                                   const float* __restrict__ counts, float* __restrict__ w) {
  const int64_t N = (int64_t)B * T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(i / T), t = (int)(i - (int64_t)b * T);
    double x = 0.0;
    if (t < seq_len(lengths, b, T) && (!mask || mask[i])) {
      if (agg == RLO_AGG_SEQ_MEAN_TOKEN_MEAN) {
        x = 1.0 / (seqs * (double)counts[b]);
      } else if (agg == RLO_AGG_SEQ_MEAN_TOKEN_SUM) {
        x = 1.0 / seqs;
      } else if (agg == RLO_AGG_GROUP_MEAN) {
        const int g0 = (b / G) * G, g1 = min(B, g0 + G);
        double M = 0.0;
        for (int k = g0; k < g1; ++k) M += (double)counts[k];
        x = 1.0 / (groups * M);
      } else {
        x = 1.0 / tokens;
      }
    }
    w[i] = (float)x;
  }
}

__global__ void __launch_bounds__(1024) count_reduce_kernel(int B, int G, const float* __restrict__ counts,
                                                            double* __restrict__ out4) {
  __shared__ double sm[3][32];
  double v[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    v[0] += (double)counts[b];
    v[1] += counts[b] > 0.f ? 1.0 : 0.0;
  }
  for (int g0 = threadIdx.x * G; g0 < B; g0 += blockDim.x * G) {
    float c = 0.f;
    for (int b = g0; b < min(B, g0 + G); ++b) c += counts[b];
    v[2] += c > 0.f ? 1.0 : 0.0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v[k] = warp_sum(v[k]);
    if (lane == 0) sm[k][warp] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double x = lane < (int)(blockDim.x >> 5) ? sm[k][lane] : 0.0;
      x = warp_sum(x);
      if (lane == 0) out4[k] = x;
    }
    if (lane == 0) out4[3] = 0.0;
  }
}

struct BwArgs {
  const void* logits;
  int64_t stride;
  const int64_t* seq_start;  // packed logits / gradient rows (NULL = padded)
  int32_t V, B, T;
  const int32_t* lengths;
  const int32_t* tokens;
  const float* lse;
  const double* lse64;  // when set, used instead of lse (hi/lo split in log2 units)
  const float* dlogp;
  const float* weight;
  void* grad;
  int64_t gstride;
};

template <typename ET>
struct In;
template <>
struct In<float> {
  static constexpr int kN = 4;
  __device__ static void load(const float* p, float (&z)[8]) {
    const float4 v = ld_stream(reinterpret_cast<const float4*>(p));
    z[0] = v.x, z[1] = v.y, z[2] = v.z, z[3] = v.w;
  }
  __device__ static float one(const float* p) { return __ldg(p); }
};
template <>
struct In<__nv_bfloat16> {
  static constexpr int kN = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&z)[8]) {
    const uint4 v = ld_stream(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) z[2 * k] = bf16lo(w[k]), z[2 * k + 1] = bf16hi(w[k]);
  }
  __device__ static float one(const __nv_bfloat16* p) { return __bfloat162float(*p); }
};

template <typename ET, typename GT>
__global__ void __launch_bounds__(kBwThreads) logits_backward_kernel(const BwArgs a) {
  constexpr int N = In<ET>::kN;
  constexpr int kOutAlign = N * (int)sizeof(GT) < 16 ? N * (int)sizeof(GT) : 16;  // widest store used
  const int64_t nrows = (int64_t)a.B * a.T;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int b = (int)(row / a.T), t = (int)(row - (int64_t)b * a.T);
    const bool valid = t < seq_len(a.lengths, b, a.T);
    if (a.seq_start && !valid) continue;  // packed: no such row
    const float scale = valid ? __ldg(a.weight + row) * __ldg(a.dlogp + row) : 0.f;
    const int64_t lrow = a.seq_start ? __ldg(a.seq_start + b) + t : row;
    GT* g = reinterpret_cast<GT*>(a.grad) + lrow * a.gstride;
    const ET* z = reinterpret_cast<const ET*>(a.logits) + lrow * a.stride;
    // A row not starting on a 16-byte boundary (e.g. V = 50257 contiguous)
    // takes its first elements scalar; the body is vectorised when the
    // gradient row is then aligned for the widest store too.
    const int mis = (int)(reinterpret_cast<uintptr_t>(z) & 15u);
    int head = min(a.V, mis ? (16 - mis) / (int)sizeof(ET) : 0);
    if (reinterpret_cast<uintptr_t>(g + head) % kOutAlign) head = a.V;  // misaligned against each other: scalar row
    const int nvec = (a.V - head) / N, tail0 = head + nvec * N;
    const ET* zb = z + head;
    GT* gb = g + head;
    if (scale == 0.f) {  // non-participating (or zero-gradient) row: zeros
      float zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int v = threadIdx.x; v < head; v += kBwThreads) Out<GT>::one(g + v, 0.f);
      for (int i = threadIdx.x; i < nvec; i += kBwThreads) Out<GT>::template store<N>(gb + (int64_t)i * N, zero);
      for (int v = tail0 + threadIdx.x; v < a.V; v += kBwThreads) Out<GT>::one(g + v, 0.f);
      continue;
    }
    const int tok = __ldg(a.tokens + row);
    // -(lse * log2e) as hi + lo floats: exact for the fp64 lse, the fp32 lse's own rounding otherwise
    float nl, nlo = 0.f;
    if (a.lse64) {
      const double L = __ldg(a.lse64 + row) * (double)kL2E;
      nl = (float)-L;
      nlo = (float)(-L - (double)nl);
    } else {
      nl = -__ldg(a.lse + row) * kL2E;
    }
    const float ms = -scale;
    auto one = [&](int v) {
      float o = ms * ex2(fmaf(In<ET>::one(z + v), kL2E, nl) + nlo);
      if (v == tok) o += scale;
      Out<GT>::one(g + v, o);
    };
    for (int v = threadIdx.x; v < head; v += kBwThreads) one(v);
    int i0 = 0;
    if constexpr (RLO_BW256 && sizeof(ET) == 2 && sizeof(GT) == 2) {
      // 32-byte pairs of vectors: one LDG.256 and one STG.256 per 16 elements
      if (((reinterpret_cast<uintptr_t>(zb) | reinterpret_cast<uintptr_t>(gb)) & 31u) == 0) {
        const int npair = nvec / 2;
        for (int q = threadIdx.x; q < npair; q += kBwThreads) {
          uint4 r0, r1;
          ld_stream256(reinterpret_cast<const uint4*>(zb) + 2 * q, r0, r1);
          const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
          uint32_t o[8];
          const int d = tok - head - q * 16;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float lo = ms * ex2(fmaf(bf16lo(w[k]), kL2E, nl) + nlo), hi = ms * ex2(fmaf(bf16hi(w[k]), kL2E, nl) + nlo);
            if (d == 2 * k) lo += scale;
            if (d == 2 * k + 1) hi += scale;
            o[k] = Out<GT>::pack(lo, hi);
          }
          st_stream256(reinterpret_cast<uint4*>(gb) + 2 * q, make_uint4(o[0], o[1], o[2], o[3]),
                       make_uint4(o[4], o[5], o[6], o[7]));
        }
        i0 = 2 * npair;
      }
    }
    for (int i = i0 + threadIdx.x; i < nvec; i += kBwThreads) {
      float x[8], o[8];
      In<ET>::load(zb + (int64_t)i * N, x);
#pragma unroll
      for (int k = 0; k < N; ++k) o[k] = ms * ex2(fmaf(x[k], kL2E, nl) + nlo);  // -w*dlp*p_v
      const int d = tok - head - i * N;
      if (d >= 0 && d < N) {
#pragma unroll
        for (int k = 0; k < N; ++k)
          if (k == d) o[k] += scale;  // + w*dlp at the realised token
      }
      Out<GT>::template store<N>(gb + (int64_t)i * N, o);
    }
    for (int v = tail0 + threadIdx.x; v < a.V; v += kBwThreads) one(v);
  }
}

template <typename ET, typename GT>
cudaError_t launch_bw(const BwArgs& a, int num_sms, cudaStream_t s) {
  const int64_t nrows = (int64_t)a.B * a.T;
  if (nrows == 0) return cudaSuccess;
  auto kern = logits_backward_kernel<ET, GT>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBwThreads, 0);
  int64_t grid = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > nrows) grid = nrows;
  kern<<<(int)grid, kBwThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_loss_weights(int32_t B, int32_t T, int32_t G, int32_t agg, double tokens, double seqs,
                                double groups, const int32_t* lengths, const uint8_t* mask, float* counts, float* w,
                                cudaStream_t s) {
  if ((int64_t)B * T == 0) return cudaSuccess;
  seq_count_kernel<<<(B + 7) / 8, 256, 0, s>>>(B, T, lengths, mask, counts);
  int64_t blocks = ((int64_t)B * T + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  loss_weight_kernel<<<(int)blocks, 256, 0, s>>>(B, T, G < 1 ? 1 : G, agg, tokens, seqs, groups, lengths, mask,
                                                 counts, w);
  g_launches.fetch_add(2, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_batch_counts(int32_t B, int32_t T, int32_t G, const int32_t* lengths, const uint8_t* mask,
                                float* counts, double* out4, cudaStream_t s) {
  if (B > 0) seq_count_kernel<<<(B + 7) / 8, 256, 0, s>>>(B, T, lengths, mask, counts);
  count_reduce_kernel<<<1, 1024, 0, s>>>(B, G < 1 ? 1 : G, counts, out4);
  g_launches.fetch_add(B > 0 ? 2 : 1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_logits_backward(const void* logits, int32_t dtype, int64_t stride, const int64_t* seq_start,
                                   int32_t V, int32_t B, int32_t T,
                                   const int32_t* lengths, const int32_t* tokens, const float* lse,
                                   const double* lse64, const float* dlogp, const float* weight, void* grad,
                                   int32_t gdtype, int64_t gstride, int num_sms, cudaStream_t s) {
  const BwArgs a{logits, stride, seq_start, V, B, T, lengths, tokens, lse, lse64, dlogp, weight, grad, gstride};
  if (dtype == RLO_DTYPE_BF16)
    return gdtype == RLO_DTYPE_BF16 ? launch_bw<__nv_bfloat16, __nv_bfloat16>(a, num_sms, s)
                                    : launch_bw<__nv_bfloat16, float>(a, num_sms, s);
  return gdtype == RLO_DTYPE_BF16 ? launch_bw<float, __nv_bfloat16>(a, num_sms, s)
                                  : launch_bw<float, float>(a, num_sms, s);
}

}  // namespace rlo
