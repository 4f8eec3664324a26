// vocab.cu — the HBM-bound vocab pass (K1 logprob/entropy, K3 fused loss).
//
// Replaces the reference's per-position log-softmax + gather
// (policy.cpp:116-122, :227; forward_logprobs :210-233) and the loss part of
// ppo_gradient (:355-374).  One pass over each logits row:
//   * 128-bit streaming loads (ld.global.nc.L1::no_allocate), U vectors in
//     flight per thread, 256 threads per CTA, persistent grid of
//     (#SM x resident CTAs) CTAs striding over rows;
//   * online log-sum-exp in log2 units: per chunk of U*VPT elements the chunk
//     max is found first, the running sum is rescaled only when the max
//     grows, then each element costs one FFMA + one MUFU.EX2 + one FADD
//     (+ one FFMA for the entropy accumulator on the actor row);
//   * warp-shuffle then shared-memory combine; the gathered token logit is
//     a direct 1-element load; the loss epilogue runs in fp64 on one thread
//     per row.  The softmax is never written.
#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct Acc {
  float mL;  // running max of z*log2e (fp32-rounded)
  float s;   // sum 2^(z*log2e - mL)
  float w;   // sum 2^(z*log2e - mL) * (z*log2e - mL)   (entropy, log2 units)
};

__device__ __forceinline__ void acc_init(Acc& a) {
  a.mL = kNegInit * kL2E;
  a.s = 0.f;
  a.w = 0.f;
}

template <bool ENT>
__device__ __forceinline__ void acc_rescale(Acc& a, float newmL) {
  if (newmL > a.mL) {
    const float d = a.mL - newmL;
    const float sc = ex2(d);
    if (ENT) a.w = (a.w + a.s * d) * sc;
    a.s *= sc;
    a.mL = newmL;
  }
}

template <bool ENT>
__device__ __forceinline__ void acc_elem(float z, float mL, float& s, float& w) {
  const float t = fmaf(z, kL2E, -mL);
  const float e = ex2(t);
  s += e;
  if (ENT) w = fmaf(e, fmaxf(t, kNegInit), w);
}

// Combine (mL2, s2, w2) into a.
template <bool ENT>
__device__ __forceinline__ void acc_combine(Acc& a, float mL2, float s2, float w2) {
  const float M = fmaxf(a.mL, mL2);
  const float d1 = a.mL - M, d2 = mL2 - M;
  const float e1 = ex2(d1), e2 = ex2(d2);
  if (ENT) a.w = (a.w + a.s * d1) * e1 + (w2 + s2 * d2) * e2;
  a.s = a.s * e1 + s2 * e2;
  a.mL = M;
}

template <bool ENT>
__device__ __forceinline__ void acc_warp_reduce(Acc& a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, a.mL, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, a.s, o);
    const float w2 = ENT ? __shfl_xor_sync(0xffffffffu, a.w, o) : 0.f;
    acc_combine<ENT>(a, m2, s2, w2);
  }
}

// ---- per-dtype vector chunk processing -------------------------------------

template <typename ET>
struct Vec;

template <>
struct Vec<float> {
  using V = float4;
  static constexpr int kElems = 4;
  // -inf padding: contributes exp2(-inf) = 0 and never raises the running max
  // (a finite sentinel would leave a rounding residual ~ulp(1e30) in t).
  __device__ static V fill() { return make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY); }
  template <int U>
  __device__ static float chunk_max(const V (&v)[U]) {
    float m = fmaxf(fmaxf(v[0].x, v[0].y), fmaxf(v[0].z, v[0].w));
#pragma unroll
    for (int u = 1; u < U; ++u) m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
    return m;
  }
  template <int U, bool ENT>
  __device__ static void accumulate(const V (&v)[U], Acc& a) {
    acc_rescale<ENT>(a, chunk_max<U>(v) * kL2E);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc_elem<ENT>(v[u].x, a.mL, s0, w0);
      acc_elem<ENT>(v[u].y, a.mL, s1, w1);
      acc_elem<ENT>(v[u].z, a.mL, s2, w2);
      acc_elem<ENT>(v[u].w, a.mL, s3, w3);
    }
    a.s += (s0 + s1) + (s2 + s3);
    if (ENT) a.w += (w0 + w1) + (w2 + w3);
  }
  __device__ static float scalar(const float* p) { return __ldg(p); }
};

template <>
struct Vec<__nv_bfloat16> {
  using V = uint4;
  static constexpr int kElems = 8;
  __device__ static V fill() { return make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u); }  // bf16 -inf
  __device__ static __nv_bfloat162 as_b2(uint32_t x) { return *reinterpret_cast<__nv_bfloat162*>(&x); }
  template <int U>
  __device__ static float chunk_max(const V (&v)[U]) {
    __nv_bfloat162 m = __hmax2(__hmax2(as_b2(v[0].x), as_b2(v[0].y)), __hmax2(as_b2(v[0].z), as_b2(v[0].w)));
#pragma unroll
    for (int u = 1; u < U; ++u)
      m = __hmax2(m, __hmax2(__hmax2(as_b2(v[u].x), as_b2(v[u].y)), __hmax2(as_b2(v[u].z), as_b2(v[u].w))));
    return fmaxf(__low2float(m), __high2float(m));
  }
  template <bool ENT>
  __device__ static void word(uint32_t x, float mL, float& s0, float& s1, float& w0, float& w1) {
    acc_elem<ENT>(bf16lo(x), mL, s0, w0);
    acc_elem<ENT>(bf16hi(x), mL, s1, w1);
  }
  template <int U, bool ENT>
  __device__ static void accumulate(const V (&v)[U], Acc& a) {
    acc_rescale<ENT>(a, chunk_max<U>(v) * kL2E);
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      word<ENT>(v[u].x, a.mL, s0, s1, w0, w1);
      word<ENT>(v[u].y, a.mL, s2, s3, w2, w3);
      word<ENT>(v[u].z, a.mL, s0, s1, w0, w1);
      word<ENT>(v[u].w, a.mL, s2, s3, w2, w3);
    }
    a.s += (s0 + s1) + (s2 + s3);
    if (ENT) a.w += (w0 + w1) + (w2 + w3);
  }
  __device__ static float scalar(const __nv_bfloat16* p) {
    return __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(p)));
  }
};

template <typename ET, int U, bool ENT>
__device__ __forceinline__ void row_accumulate(const ET* __restrict__ row, int V, bool vec_ok, Acc& a) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  const int tid = threadIdx.x;
  const int nvec = vec_ok ? V / VT::kElems : 0;
  const VV* __restrict__ vrow = reinterpret_cast<const VV*>(row);
  for (int base = 0; base < nvec; base += kThreads * U) {
    VV v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = base + u * kThreads + tid;
      v[u] = idx < nvec ? ld_stream(vrow + idx) : VT::fill();
    }
    VT::template accumulate<U, ENT>(v, a);
  }
  // scalar tail (or the whole row when rows are not 16-byte aligned)
  for (int i = nvec * VT::kElems + tid; i < V; i += kThreads) {
    const float z = VT::scalar(row + i);
    acc_rescale<ENT>(a, z * kL2E);
    float w = 0.f, s = 0.f;
    acc_elem<ENT>(z, a.mL, s, w);
    a.s += s;
    if (ENT) a.w += w;
  }
}

struct RowResult {
  double lse;
  double entropy;
};

// Finalise a block-reduced accumulator in fp64 (the state is
// kept in log2 units relative to the fp32 constant kL2E; dividing by the same
// constant returns natural units exactly up to the per-element rounding).
__device__ __forceinline__ RowResult finish(const Acc& a) {
  const double l2 = log2((double)a.s);
  RowResult r;
  r.lse = ((double)a.mL + l2) / (double)kL2E;
  r.entropy = (l2 - (double)a.w / (double)a.s) / (double)kL2E;
  return r;
}

template <typename ET>
__device__ __forceinline__ float load_logit(const void* base, int64_t off) {
  return Vec<ET>::scalar(reinterpret_cast<const ET*>(base) + off);
}

__device__ void loss_epilogue(const VocabArgs& a, int64_t row, double lp, double old, bool has_ref, double ref,
                              double ent, double ztok_unused) {
  (void)ztok_unused;
  const double A = (double)a.adv[row];
  const double eps = a.clip_eps;
  const double ratio = exp(lp - old);                       // policy.cpp:358
  const double rcl = clampd(ratio, 1.0 - eps, 1.0 + eps);  // :359
  const double u = ratio * A, c = rcl * A;                  // :360-361
  const double surr = (c < u) ? c : u;                      // :362 std::min
  double pg = -surr;
  bool dual = false;
  if (a.dual_c > 1.0 && A < 0.0) {  // dual-clip extension
    const double cap = -a.dual_c * A;
    if (pg > cap) {
      pg = cap;
      dual = true;
    }
  }
  double k = 0.0, dk = 0.0;
  if (has_ref) {
    const double r = lp - ref;
    if (a.kl_est == RLO_KL_K2) {
      k = 0.5 * r * r;
      dk = r;
    } else if (a.kl_est == RLO_KL_K3) {
      const double er = exp(-r);
      k = er - 1.0 + r;
      dk = 1.0 - er;
    } else {
      k = r;
      dk = 1.0;
    }
  }
  const double kc = a.kl_coef;
  const double loss = pg + kc * (kc > 0.0 ? k : 0.0);  // :364-366
  const bool flows = A >= 0.0 ? ratio <= 1.0 + eps : ratio >= 1.0 - eps;  // :373
  double dlp = (flows && !dual) ? -ratio * A : 0.0;                      // :374
  dlp += kc > 0.0 ? kc * dk : 0.0;
  uint8_t flags = 0;
  if (u > c) flags |= TF_CLIPPED;  // :369
  if (dual) flags |= TF_DUAL;
  if (!isfinite(dlp)) flags |= TF_NONFINITE_GRAD;
  if (!isfinite(loss)) flags |= TF_NONFINITE_LOSS;
  a.s_loss[row] = (float)loss;
  a.s_ratio[row] = (float)ratio;
  a.s_kl[row] = has_ref ? (float)k : 0.f;
  a.s_ent[row] = (float)ent;
  a.s_flags[row] = flags;
  if (a.o_logp) a.o_logp[row] = (float)lp;
  if (a.o_old) a.o_old[row] = (float)old;
  if (a.o_ref) a.o_ref[row] = has_ref ? (float)ref : 0.f;
  if (a.o_ent) a.o_ent[row] = (float)ent;
  if (a.o_dlogp) a.o_dlogp[row] = (float)dlp;
  if (a.o_loss) a.o_loss[row] = (float)loss;
}

__device__ __forceinline__ void flag_error(const VocabArgs& a, int code, int value) {
  if (atomicCAS(&a.err->code, 0, code) == 0) a.err->value = value;
}

// LOSS=false: forward_logprobs (NT==1; every valid position, mask ignored).
// LOSS=true : fused loss over loss-participating positions; slot 0 is the actor.
template <typename ET, int NT, int U, bool LOSS, bool ENT0>
__global__ void __launch_bounds__(kThreads) vocab_kernel(const VocabArgs a) {
  __shared__ float red[2][kWarps][NT][3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nrows = (int64_t)a.B * a.T;
  bool vec_ok = true;
#pragma unroll
  for (int k = 0; k < NT; ++k)
    vec_ok &= ((reinterpret_cast<uintptr_t>(a.logits[k]) & 15u) == 0) &&
              (((a.stride[k] * (int64_t)sizeof(ET)) & 15) == 0);
  int buf = 0;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int b = (int)(row / a.T);
    const int t = (int)(row - (int64_t)b * a.T);
    if (t == 0 && tid == 0) {
      const int raw = __ldg(a.lengths + b);
      if (raw < 0 || raw > a.T) flag_error(a, DE_BAD_LENGTH, b);
    }
    bool active = t < seq_len(a.lengths, b, a.T);
    if (LOSS && active && a.mask) active = __ldg(a.mask + row) != 0;
    if (!active) {
      if (tid == 0) {
        if (!LOSS) {
          a.out_lp[row] = 0.f;
          if (a.out_ent) a.out_ent[row] = 0.f;
          if (a.out_tok) a.out_tok[row] = 0.f;
        } else {
          if (a.o_logp) a.o_logp[row] = 0.f;
          if (a.o_old) a.o_old[row] = 0.f;
          if (a.o_ref) a.o_ref[row] = 0.f;
          if (a.o_ent) a.o_ent[row] = 0.f;
          if (a.o_dlogp) a.o_dlogp[row] = 0.f;
          if (a.o_loss) a.o_loss[row] = 0.f;
        }
      }
      continue;
    }
    // token logit gather (thread 0): bit-exact element load, latency hidden by the row pass
    int tok = 0;
    bool oov = false;
    float ztok[NT];
    if (tid == 0) {
      tok = __ldg(a.tokens + row);
      oov = tok < 0 || tok >= a.V;
#pragma unroll
      for (int k = 0; k < NT; ++k) ztok[k] = oov ? 0.f : load_logit<ET>(a.logits[k], row * a.stride[k] + tok);
    }
    Acc acc[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      acc_init(acc[k]);
      const ET* rp = reinterpret_cast<const ET*>(a.logits[k]) + row * a.stride[k];
      if (k == 0 && ENT0)
        row_accumulate<ET, U, true>(rp, a.V, vec_ok, acc[k]);
      else
        row_accumulate<ET, U, false>(rp, a.V, vec_ok, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if (k == 0 && ENT0)
        acc_warp_reduce<true>(acc[k]);
      else
        acc_warp_reduce<false>(acc[k]);
      if (lane == 0) {
        red[buf][warp][k][0] = acc[k].mL;
        red[buf][warp][k][1] = acc[k].s;
        red[buf][warp][k][2] = acc[k].w;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double lse[NT], ent = 0.0;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        Acc c;
        if (lane < kWarps) {
          c.mL = red[buf][lane][k][0];
          c.s = red[buf][lane][k][1];
          c.w = red[buf][lane][k][2];
        } else {
          acc_init(c);
        }
        if (k == 0 && ENT0)
          acc_warp_reduce<true>(c);
        else
          acc_warp_reduce<false>(c);
        const RowResult r = finish(c);
        lse[k] = r.lse;
        if (k == 0) ent = r.entropy;
      }
      if (lane == 0) {
        if (oov) flag_error(a, LOSS ? DE_OOV_LOSS : DE_OOV_LOGPROB, tok);
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        double lp[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) lp[k] = oov ? nan : (double)ztok[k] - lse[k];  // policy.cpp:122, :227
        if (!LOSS) {
          a.out_lp[row] = (float)lp[0];
          if (a.out_ent) a.out_ent[row] = (float)ent;
          if (a.out_tok) a.out_tok[row] = ztok[0];
        } else {
          double old = 0.0, ref = 0.0;
          bool have_old = false, have_ref = false;
#pragma unroll
          for (int k = 1; k < NT; ++k) {
            if (a.role[k] == ROLE_OLD) { old = lp[k]; have_old = true; }
            if (a.role[k] == ROLE_REF) { ref = lp[k]; have_ref = true; }
          }
          if (!have_old) old = (double)a.old_lp_in[row];
          if (!have_ref && a.ref_lp_in) { ref = (double)a.ref_lp_in[row]; have_ref = true; }
          loss_epilogue(a, row, lp[0], old, have_ref, ref, ent, 0.0);
        }
      }
    }
    buf ^= 1;
  }
}

template <typename K>
int grid_for(K kernel, int num_sms, int64_t nrows) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t g = (int64_t)num_sms * per_sm;
  if (g > nrows) g = nrows;
  return (int)(g < 1 ? 1 : g);
}

template <typename ET, int NT, bool LOSS, bool ENT0>
cudaError_t launch_t(const VocabArgs& a, int num_sms, cudaStream_t s) {
  constexpr int U = sizeof(ET) == 4 ? 8 : 4;
  auto kern = vocab_kernel<ET, NT, U, LOSS, ENT0>;
  const int64_t nrows = (int64_t)a.B * a.T;
  if (nrows == 0) return cudaSuccess;
  const int grid = grid_for(kern, num_sms, nrows);
  kern<<<grid, kThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <typename ET>
cudaError_t launch_loss_dtype(const VocabArgs& a, int num_sms, cudaStream_t s) {
  switch (a.ntens) {
    case 1: return launch_t<ET, 1, true, true>(a, num_sms, s);
    case 2: return launch_t<ET, 2, true, true>(a, num_sms, s);
    default: return launch_t<ET, 3, true, true>(a, num_sms, s);
  }
}

}  // namespace

cudaError_t launch_vocab_logprob(const VocabArgs& a, int num_sms, cudaStream_t s) {
  const bool ent = a.out_ent != nullptr;
  if (a.dtype == RLO_DTYPE_BF16)
    return ent ? launch_t<__nv_bfloat16, 1, false, true>(a, num_sms, s)
               : launch_t<__nv_bfloat16, 1, false, false>(a, num_sms, s);
  return ent ? launch_t<float, 1, false, true>(a, num_sms, s) : launch_t<float, 1, false, false>(a, num_sms, s);
}

cudaError_t launch_vocab_loss(const VocabArgs& a, int num_sms, cudaStream_t s) {
  return a.dtype == RLO_DTYPE_BF16 ? launch_loss_dtype<__nv_bfloat16>(a, num_sms, s)
                                   : launch_loss_dtype<float>(a, num_sms, s);
}

}  // namespace rlo
