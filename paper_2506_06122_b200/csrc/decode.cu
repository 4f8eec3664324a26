// decode.cu — sampling-time log-probs: decode_next
// (policy.cpp:143-169) for a batch of rows.  The reference draws a token by a
// CDF walk in token-id order over the tempered softmax with the keyed uniform
// u = keyed_double({seed, version, sample_key, position}) (rng.hpp:22-31,
// 82-85) and returns the token with its UNtempered log-prob (:168) — the
// "old" log-prob of the PPO ratio, so emitting it here removes the separate
// old-policy logits pass (P = 3 -> 2).
//
// The tempered weights exp((z - m)/T) are fp64 (the reference's precision:
// the CDF walk picks the same token unless u * total falls within fp64
// rounding of a CDF boundary), through a table-driven exp (exp_neg); the
// UNtempered log-sum-exp only feeds the returned log-prob and runs in fp32 in
// log2 units like the vocab pass (relative error ~1e-7).
// Traffic per row ~ (1 + 1/8) x V x s.
//
// Two paths per row.  The screened fp32 path (default) computes the tempered
// weights 2^(z*cT - mT) with MUFU.EX2 in fp32 (vector sums of 4-8 accumulated
// in fp64), walks the CDF the same way, and accepts its pick c only with a
// certificate: X = u * total lies more than margin * total inside
// (CDF(c-1), CDF(c)].  Every element enters the total, the CDF and X through
// ONE computed weight w^_v, so the error of X - CDF(c-1) is
// (u - 1) sum_{v<c} (w^_v - w_v) + u sum_{v>=c} (w^_v - w_v), at most
// max(u, 1-u) * eps_e * total (likewise CDF(c) - X), where
//   eps_e * total >= sum_v |w^_v - w_v|: argument rounding |dt| <= |t| 2^-24
//   and the fp32 constant cT = log2(e)/T, |dt| <= |t| 2^-24, give
//   2^-24 ln2 sum_v w_v |t_v| each, and sum_v w_v |t_v| <= total * log2(V)
//   (sum p (-log2 p) <= log2 V, the max weight being 1); ex2.approx.ftz.f32
//   <= 1.44e-7 relative (exhaustive over t in [-126, 1] on B200,
//   tools/probes/ex2_probe.cu; 1.5e-7 used);
// plus the two summation orders (kScreenSum = 2 x a 3-deep fp32 tree; fp64
// accumulation and the fp64 rescales negligible):
//   margin = 1.1 * (max(u, 1-u) * eps_e(V) + kScreenSum), 0.9-1.6e-6 at V = 152064.
// Under the certificate the exact CDF walk picks the same token, so the draw
// is the fp64 path's.  A row without one (a CDF boundary within the margin,
// most likely on flat rows, profiles/r1_next_rows.txt; or non-finite sums) is
// redone by the fp64 path — the weights exp((z - m)/T) in fp64 through a
// table-driven exp (exp_neg), bound by fp64 throughput (~13 fp64 operations
// per element) — in a second launch that skips the certified rows.
// RLO_DECODE_MARGIN fixes the margin instead (<= 0: fp64 path only; >= 1:
// every row redone, for tests).
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

#ifndef RLO_DEC_WARPS  // warps per row (one CTA per row)
#define RLO_DEC_WARPS 8
#endif
constexpr int kDecWarps = RLO_DEC_WARPS;

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
__device__ __forceinline__ float logit(const ET* p, int v);
template <>
__device__ __forceinline__ float logit<float>(const float* p, int v) {
  return __ldg(p + v);
}
template <>
__device__ __forceinline__ float logit<__nv_bfloat16>(const __nv_bfloat16* p, int v) {
  return __bfloat162float(p[v]);
}

// exp(t) for t <= 0 in fp64 (the reference's std::exp precision, <= 1 ulp):
// t = (256k + j) ln2/256 + r, |r| <= ln2/512; exp(t) = 2^k * 2^(j/256) * e^r
// with 2^(j/256) from a 256-entry shared table and e^r from a degree-4 Taylor
// polynomial (truncation r^5/120 < 4e-17).  9 fp64 operations instead of the
// ~20 of the library exp(); t < -708 is clamped (3e-308, below every sum it
// enters).
constexpr int kExpTab = 256;
// Unclamped core: t must be >= -708 (exp_neg clamps; -inf logits then weigh
// exp(-708) ~ 3e-308 instead of 0 — below any sum they enter).  2^k is added
// to the high word only.
__device__ __forceinline__ double exp_neg_core(double t, const double* __restrict__ tab) {
  constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52: round to integer
  constexpr double k256Ln2 = 369.32993046757462;  // 256 / ln 2
  constexpr double kLn2o256Hi = 0x1.62e42fefa0000p-9, kLn2o256Lo = 0x1.cf79abc9e3b3ap-48;
  const double s = fma(t, k256Ln2, kMagic);
  const int n = __double2loint(s);
  const double nf = s - kMagic;
  double r = fma(nf, -kLn2o256Hi, t);
  r = fma(nf, -kLn2o256Lo, r);
  double p = fma(r, 1.0 / 24, 1.0 / 6);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double v = tab[n & (kExpTab - 1)] * p;
  return __hiloint2double(__double2hiint(v) + ((n >> 8) << 20), __double2loint(v));
}
__device__ __forceinline__ double exp_neg(double t, const double* __restrict__ tab) {
  return exp_neg_core(fmax(t, -708.0), tab);  // branch-free: exp(-708) = 3e-308 stands in for 0
}
// The tempered exponent (x - M) / T of a logit x below the row max M, in fp64
// (x - M is exact for fp32 / bf16 logits).  The clamp to exp_neg's domain is
// applied AFTER the division by T: a bound formed in the logit domain
// (M - 700*T in fp32) rounds to M itself at T <= 1e-9 and lets arguments below
// -708 through at T ~ 1e-7 with |M| >= 128 (the reference decodes greedily at
// T = 1e-6, pipeline.cpp:539).  -inf logits give -708 (3e-308), not NaN.
__device__ __forceinline__ double scaled_gap(float x, double M, double inv_t, bool unit_t) {
  const double d = (double)x - M;
  return unit_t ? d : d * inv_t;
}

template <typename ET>
struct DVec;
template <>
struct DVec<float> {
  static constexpr int E = 4;
  __device__ static void load(const float* p, float (&x)[8]) {
    const float4 v = ld_stream(reinterpret_cast<const float4*>(p));
    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
  }
};
template <>
struct DVec<__nv_bfloat16> {
  static constexpr int E = 8;
  __device__ static void load(const __nv_bfloat16* p, float (&x)[8]) {
    const uint4 v = ld_stream(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) x[2 * k] = bf16lo(w[k]), x[2 * k + 1] = bf16hi(w[k]);
  }
};

// Elements [v, v+E) of the row (fewer at the end of a range / the row):
// vector load when the whole vector is inside and aligned, else per element;
// missing elements -inf.
template <typename ET>
__device__ __forceinline__ void load_e(const ET* z, int v, int lim, bool vec_ok, float (&x)[8]) {
  constexpr int E = DVec<ET>::E;
  if (vec_ok && v + E <= lim) {
    DVec<ET>::load(z + v, x);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = v + e < lim ? logit(z, v + e) : -INFINITY;
  }
}

// The certificate's error terms, relative to the total, for a vocabulary of
// V tokens: eps_e bounds sum_v |w^_v - w_v| (argument rounding and the fp32
// log2(e)/T constant, 2^-24 ln2 sum w|t| each with sum w|t| <= total log2 V;
// ex2.approx 1.5e-7), kScreenSum the summation of two differently grouped
// sums (2 x a 3-deep fp32 tree; fp64 accumulation negligible).
inline double screen_eps(int V) {
  return 2.0 * std::log2((double)(V > 2 ? V : 2)) * 0x1p-24 * 0.6931471805599453 + 1.5e-7;
}
constexpr double kScreenSum = 6.0 * 0x1p-24;
constexpr double kScreenSafety = 1.1;  // second-order terms

#ifndef RLO_SCREEN_U
#define RLO_SCREEN_U 4
#endif
#ifndef RLO_SCREEN_POLY  // untempered exponentials on the FMA pipe: 0 none, 1 half (default), 2 all
#define RLO_SCREEN_POLY 1
#endif
#ifndef RLO_SCREEN_MINB
#define RLO_SCREEN_MINB 4
#endif
constexpr int kScreenU = RLO_SCREEN_U;  // 16-byte loads in flight per lane (screened path)
constexpr int kStepMax = 1024;     // step sums of one warp range kept in shared memory

// Raw 16-byte vectors of E logits (token order) and their fp32 values.
template <typename ET>
struct RawVec;
template <>
struct RawVec<float> {
  static constexpr int E = 4;
  static constexpr uint32_t kNegInf = 0xFF800000u;
  __device__ static float at(const uint4& r, int e) {
    return __uint_as_float(e == 0 ? r.x : e == 1 ? r.y : e == 2 ? r.z : r.w);
  }
  __device__ static uint32_t raw1(const float* z, int v) { return __float_as_uint(__ldg(z + v)); }
  __device__ static uint4 fill(const float* z, int v, int lim) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) w[e] = v + e < lim ? raw1(z, v + e) : kNegInf;
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <>
struct RawVec<__nv_bfloat16> {
  static constexpr int E = 8;
  __device__ static float at(const uint4& r, int e) {
    const uint32_t w = (e >> 1) == 0 ? r.x : (e >> 1) == 1 ? r.y : (e >> 1) == 2 ? r.z : r.w;
    return (e & 1) ? bf16hi(w) : bf16lo(w);
  }
  __device__ static uint32_t raw1(const __nv_bfloat16* z, int v) {
    return (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(z) + v);
  }
  __device__ static uint4 fill(const __nv_bfloat16* z, int v, int lim) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lo = v + 2 * k < lim ? raw1(z, v + 2 * k) : 0xFF80u;
      const uint32_t hi = v + 2 * k + 1 < lim ? raw1(z, v + 2 * k + 1) : 0xFF80u;
      w[k] = lo | (hi << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
// Tokens [v, v+E) of the row, -inf past lim: one 16-byte load when the
// vector is whole and aligned, else per element.
template <typename ET>
__device__ __forceinline__ uint4 load_raw(const ET* z, int v, int lim, bool vec_ok) {
  if (vec_ok && v + RawVec<ET>::E <= lim) return ld_stream(reinterpret_cast<const uint4*>(z + v));
  return v < lim ? RawVec<ET>::fill(z, v, lim) : RawVec<ET>::fill(z, lim, lim);
}

// fp32 sum of the E weights 2^(x*c - mo) of one vector, in fp64: packed
// FFMA2 per element pair, MUFU.EX2 per element, a pairwise FADD2 tree (at
// most 3 roundings deep, the bound kScreenSum uses).
template <typename ET>
__device__ __forceinline__ double vec_wsum(const uint4& r, float c, float mo) {
  constexpr int E = RawVec<ET>::E;
  const f2 c2 = pk2(c, c), m2 = pk2(-mo, -mo);
  f2 acc[2];
#pragma unroll
  for (int p = 0; p < E / 2; ++p) {
    const f2 t = ffma2(pk2(RawVec<ET>::at(r, 2 * p), RawVec<ET>::at(r, 2 * p + 1)), c2, m2);
    float tl, th;
    upk2(t, tl, th);
    const f2 e = pk2(ex2(tl), ex2(th));  // -inf -> 0
    acc[p & 1] = p < 2 ? e : fadd2(acc[p & 1], e);
  }
  float lo, hi;
  upk2(fadd2(acc[0], acc[1]), lo, hi);
  return (double)(lo + hi);
}

// Largest of the U vectors' logits (packed bf16x2 max for bf16; exact).
template <typename ET, int U>
__device__ __forceinline__ float raw_max(const uint4 (&r)[U]) {
  if constexpr (sizeof(ET) == 2) {
    auto b2 = [](uint32_t x) { return *reinterpret_cast<__nv_bfloat162*>(&x); };
    __nv_bfloat162 m = __hmax2(__hmax2(b2(r[0].x), b2(r[0].y)), __hmax2(b2(r[0].z), b2(r[0].w)));
#pragma unroll
    for (int k = 1; k < U; ++k) m = __hmax2(m, __hmax2(__hmax2(b2(r[k].x), b2(r[k].y)), __hmax2(b2(r[k].z), b2(r[k].w))));
    return fmaxf(__low2float(m), __high2float(m));
  } else {
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < U; ++k)
      m = fmaxf(m, fmaxf(fmaxf(__uint_as_float(r[k].x), __uint_as_float(r[k].y)),
                         fmaxf(__uint_as_float(r[k].z), __uint_as_float(r[k].w))));
    return m;
  }
}

// As vec_wsum, half of the element pairs through the FMA-pipe degree-4 exp2
// (relative error 2.9e-6 per term, t clamped to its normal-range domain):
// the untempered sum at T != 1, which only feeds the returned log-prob
// (|lse error| <= 1.5e-6), so the MUFU pipe carries 1.5 instead of 2
// exponentials per element there.  Never used for the certified weights.
// Returns the fp32 vector sum: the caller adds the U vectors of a batch in
// fp32 and converts once (this sum needs ~1e-6, not the certificate's bound).
template <typename ET>
__device__ __forceinline__ float vec_wsum_half_poly(const uint4& r, float c, float mo) {
  constexpr int E = RawVec<ET>::E;
  const f2 c2 = pk2(c, c), m2 = pk2(-mo, -mo);
  f2 acc = pk2(0.f, 0.f);
#pragma unroll
  for (int p = 0; p < E / 2; ++p) {
    const f2 t = ffma2(pk2(RawVec<ET>::at(r, 2 * p), RawVec<ET>::at(r, 2 * p + 1)), c2, m2);  // = two fmaf
    float tl, th;
    upk2(t, tl, th);
    const bool poly = RLO_SCREEN_POLY == 2 ? true : RLO_SCREEN_POLY == 1 ? (p & 1) != 0 : false;
    const f2 e = poly ? exp2_poly2<4>(fmaxf(tl, -126.f), fmaxf(th, -126.f)) : pk2(ex2(tl), ex2(th));
    acc = fadd2(acc, e);
  }
  float lo, hi;
  upk2(acc, lo, hi);
  return lo + hi;
}

// The screened fp32 path for one row (every thread of the CTA calls it; the
// result is uniform).  Weights 2^(z*cT - mT): cT = log2(e)/T as fp32, mT the
// rounded max times cT (a common factor, exact across rescales, which the
// CDF walk does not see).
//   pass 1: warp j owns tokens [j*W, (j+1)*W); per lane kScreenU 16-byte
//           loads in flight; running max, tempered and untempered sums
//           (fp32 vector sums accumulated in fp64);
//   thread 0: totals, lse, X = u * total, the crossing warp range;
//   pass 2a: the 8 warps sum the crossing range's steps of 32*E tokens
//           (kScreenU steps in flight per warp) into shared memory;
//   warp 0: scans the step sums for the crossing step, walks it (warp prefix
//           of the lane sums, then the hit lane's tokens in order) and checks
//           the certificate X - CDF(c-1) > margin * total, CDF(c) - X > margin * total
//           (total and X re-formed with the step sums, see the header).
// Returns true with s_pick / s_lse set when the certificate holds; false
// sends the row to the fp64 path.
template <typename ET>
__device__ __forceinline__ bool screened_row(const ET* __restrict__ z, int V, int W, bool vec_ok, bool unit_t, float cT,
                                             double eps_e, double fixed, double u, double* s_t, double* s_u2,
                                             float* s_mt,
                                             float* s_ml, double* s_step, double& s_thresh, double& s_total,
                                             double& s_lse, int& s_warp, int& s_pick, int& s_ok) {
  constexpr int E = RawVec<ET>::E, S = 32 * E, U = kScreenU;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int v0 = warp * W, v1 = min(V, v0 + W);
  float m = -INFINITY, mL = kNegInit * kL2E, mT = kNegInit * kL2E;
  double st = 0.0, su = 0.0;
  auto load = [&](int b, uint4 (&r)[U]) {
    if (vec_ok && b + (U - 1) * S + E <= v1) {  // whole batch in range: plain vector loads
#pragma unroll
      for (int k = 0; k < U; ++k) r[k] = ld_stream(reinterpret_cast<const uint4*>(z + b + k * S));
    } else {
#pragma unroll
      for (int k = 0; k < U; ++k) r[k] = load_raw<ET>(z, b + k * S, v1, vec_ok);
    }
  };
  auto batch = [&](const uint4 (&r)[U]) {
    const float cm = raw_max<ET, U>(r);
    if (cm > m) {
      const float nL = __fmul_rn(cm, kL2E), nT = unit_t ? nL : __fmul_rn(cm, cT);
      su *= exp2((double)mL - (double)nL);
      st *= exp2((double)mT - (double)nT);
      m = cm, mL = nL, mT = nT;
    }
    if (m == -INFINITY) return;
#pragma unroll
    for (int k = 0; k < U; ++k) {
      if (unit_t) {  // one set of weights, certified precision
        const double qs = vec_wsum<ET>(r[k], kL2E, mL);
        su += qs;
        st += qs;
      } else {
        st += vec_wsum<ET>(r[k], cT, mT);
      }
    }
    if (!unit_t) {
      float sb = 0.f;
#pragma unroll
      for (int k = 0; k < U; ++k) sb += vec_wsum_half_poly<ET>(r[k], kL2E, mL);
      su += (double)sb;
    }
  };
  for (int b = v0 + lane * E; b < v1; b += U * S) {
    uint4 r[U];
    load(b, r);
    batch(r);
  }
#pragma unroll
  {  // warp combine: the warp's max first, then one fp64 rescale per lane and plain sums
    float ML = mL, MT = mT;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ML = fmaxf(ML, __shfl_xor_sync(0xffffffffu, ML, o));
      MT = fmaxf(MT, __shfl_xor_sync(0xffffffffu, MT, o));
    }
    su = warp_sum(su * exp2((double)mL - ML));
    st = warp_sum(st * exp2((double)mT - MT));
    mL = ML, mT = MT;
  }
  if (lane == 0) s_t[warp] = st, s_u2[warp] = su, s_mt[warp] = mT, s_ml[warp] = mL;
  __syncthreads();
  if (warp == 0) {  // combine the 8 warp states: lanes 0-7 in parallel
    const bool in = lane < kDecWarps;
    float MT = in ? s_mt[lane] : -INFINITY, ML = in ? s_ml[lane] : -INFINITY;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      MT = fmaxf(MT, __shfl_xor_sync(0xffffffffu, MT, o));
      ML = fmaxf(ML, __shfl_xor_sync(0xffffffffu, ML, o));
    }
    const double tj = in ? s_t[lane] * exp2((double)s_mt[lane] - MT) : 0.0;
    const double T = warp_sum(tj);
    const double Uu = warp_sum(in ? s_u2[lane] * exp2((double)s_ml[lane] - ML) : 0.0);
    // worst-case margin for the early outs (u-dependent certificate below)
    const double X = u * T, mg = (fixed > 0.0 ? fixed : kScreenSafety * (eps_e + kScreenSum)) * T;
    double incl = tj;  // inclusive prefix of the warp sums in token order
#pragma unroll
    for (int o = 1; o < kDecWarps; o <<= 1) {
      const double q = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += q;
    }
    // a threshold within the margin of the total (the reference's no-crossing
    // fallback to the last token is in play) or non-finite sums: fp64 path
    const bool go = isfinite(T) && T > 0.0 && isfinite(Uu) && Uu > 0.0 && X < T - mg && W / S <= kStepMax;
    const unsigned hit = __ballot_sync(0xffffffffu, go && in && X < incl);
    const int jw = hit ? __ffs(hit) - 1 : -1;
    const double base = jw >= 0 ? __shfl_sync(0xffffffffu, incl - tj, jw) : 0.0;
    const double tw = jw >= 0 ? __shfl_sync(0xffffffffu, tj, jw) : 0.0;
    if (lane == 0) {
      s_warp = jw;
      s_u2[0] = base;                       // CDF before the crossing warp range (pass-1 sums)
      s_u2[1] = jw >= 0 ? T - tw : 0.0;     // pass-1 mass outside it
      s_thresh = X;
      s_total = T;
      s_mt[0] = MT;
      s_lse = ((double)ML + log2(Uu)) / (double)kL2E;
      s_ok = 0;
    }
  }
  __syncthreads();
  const int jw = s_warp;
  if (jw < 0) return false;
  const float MT = s_mt[0];
  const int a0 = jw * W, a1 = min(V, a0 + W);
  const int nsteps = (a1 - a0 + S - 1) / S;
  // pass 2a: step sums of the crossing range, U steps in flight per warp
  for (int s0 = warp; s0 < nsteps; s0 += U * kDecWarps) {
    uint4 r[U];
#pragma unroll
    for (int k = 0; k < U; ++k) r[k] = load_raw<ET>(z, a0 + (s0 + k * kDecWarps) * S + lane * E, a1, vec_ok);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const double ls = warp_sum(vec_wsum<ET>(r[k], cT, MT));
      const int sk = s0 + k * kDecWarps;
      if (lane == 0 && sk < nsteps) s_step[sk] = ls;
    }
  }
  __syncthreads();
  if (warp == 0) {
    // One computed weight per element from here on: the total is re-formed
    // from the pass-1 sums outside the crossing range and the step sums
    // inside it (the walk's weights are bitwise those of the step sums), so
    // with X = u * total the errors of X - CDF(c-1) and CDF(c) - X are
    // (u - 1) e_before + u e_after: at most max(u, 1 - u) * eps_e * total,
    // plus the two summation orders.
    double td = 0.0;
    for (int c = lane; c < nsteps; c += 32) td += s_step[c];
    td = warp_sum(td);
    const double T2 = s_u2[1] + td;
    const double X = u * T2;
    const double mg = (fixed > 0.0 ? fixed : kScreenSafety * (fmax(u, 1.0 - u) * eps_e + kScreenSum)) * T2;
    double base = s_u2[0];
    int ks = -1;
    for (int c = 0; c < nsteps && ks < 0; c += 32) {  // first step whose inclusive CDF passes X
      const double v = c + lane < nsteps ? s_step[c + lane] : 0.0;
      double incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double q = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += q;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, c + lane < nsteps && X < base + incl);
      if (hit) {
        const int hl = __ffs(hit) - 1;
        ks = c + hl;
        base += __shfl_sync(0xffffffffu, incl - v, hl);
      } else {
        base += __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (ks >= 0) {  // walk step ks (else the sums disagree at a range boundary: fp64 path)
      const int b = a0 + ks * S + lane * E;
      const uint4 r = load_raw<ET>(z, b, a1, vec_ok);
      float w[8];
      double ls = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        w[e] = ex2(fmaf(RawVec<ET>::at(r, e), cT, -MT));
        ls += (double)w[e];
      }
      double incl = ls;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double q = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += q;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, b < a1 && X < base + incl);
      if (hit && lane == __ffs(hit) - 1) {
        double a = base + incl - ls;  // CDF before this lane's first token
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double prev = a;
          a += (double)w[e];
          if (b + e < a1 && X < a) {
            // the certificate: X more than margin * total inside (CDF(c-1), CDF(c)]
            s_pick = b + e;
            s_ok = (X - prev > mg && a - X > mg) ? 1 : 0;
            break;
          }
        }
      }
    }
  }
  __syncthreads();
  return s_ok != 0;
}

// One CTA per row, 8 warps; warp j owns the contiguous token range
// [j*W, (j+1)*W), W a multiple of 32*E; lane l takes the E consecutive tokens
// at base + l*E of each 32*E step (16-byte loads, token order preserved).
//   pass 1: per thread, running max m (exact: the logits are fp32/bf16), the
//           fp64 tempered sum of exp((z - m)/T) (rescaled when m grows) and
//           the fp32 untempered online sum (log2 units, as the vocab pass);
//   combine: warp then block (warp order), thread 0 forms the totals, the
//           keyed uniform u, X = u * total, and the warp whose range holds X;
//   pass 2: the 8 warps sum 8 sub-ranges of the crossing range (weights
//           relative to the row max); thread 0 picks the crossing sub-range;
//           warp 0 walks it: per step each lane sums its E weights, a warp
//           inclusive scan, the first lane whose prefix passes X walks its E
//           tokens in order (the reference's first `u < acc`).
template <typename ET>
__global__ void __launch_bounds__(kDecWarps * 32)
    decode_kernel(const ET* __restrict__ logits, int64_t stride, int V, int n, double temp, uint64_t seed,
                  uint64_t version, const uint64_t* __restrict__ keys, const uint64_t* __restrict__ positions,
                  int32_t* __restrict__ out_tok, float* __restrict__ out_lp, bool redo_only) {
  constexpr int E = DVec<ET>::E;
  __shared__ double tab[kExpTab];
  __shared__ double s_t[kDecWarps];
  __shared__ float s_m[kDecWarps], s_ml[kDecWarps], s_su[kDecWarps];
  __shared__ double s_base, s_thresh, s_lse;
  __shared__ float s_M;
  __shared__ int s_warp, s_pick;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j < kExpTab; j += blockDim.x) tab[j] = exp2((double)j / kExpTab);
  __syncthreads();
  const double inv_t = 1.0 / temp;
  const bool unit_t = temp == 1.0;
  const int W = ((V + kDecWarps - 1) / kDecWarps + 32 * E - 1) / (32 * E) * (32 * E);
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(logits) & 15u) == 0) && (((stride * (int64_t)sizeof(ET)) & 15) == 0);
  for (int row = blockIdx.x; row < n; row += gridDim.x) {
    const ET* z = logits + (int64_t)row * stride;
    const int v0 = warp * W, v1 = min(V, v0 + W);
    if (redo_only && out_tok[row] >= 0) continue;  // the screened kernel certified this row
    // pass 1
    float m = -INFINITY, mL = kNegInit * kL2E, su = 0.f;
    double st = 0.0;
    for (int b = v0 + lane * E; b < v1; b += 32 * E) {
      float x[8];
      load_e<ET>(z, b, v1, vec_ok, x);
      float cm = x[0];
#pragma unroll
      for (int e = 1; e < E; ++e) cm = fmaxf(cm, x[e]);
      if (cm > m) {
        if (m != -INFINITY) st *= exp_neg(unit_t ? (double)m - cm : ((double)m - cm) * inv_t, tab);
        m = cm;
        const float nmL = __fmul_rn(cm, kL2E);
        su *= ex2(mL - nmL);
        mL = nmL;
      }
      if (m == -INFINITY) continue;
      double w[8];
      float q[8];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        w[e] = exp_neg(scaled_gap(x[e], (double)m, inv_t, unit_t), tab);
        q[e] = ex2(fmaf(x[e], kL2E, -mL));  // -inf -> ex2(-inf) = 0
      }
#pragma unroll
      for (int h = E / 2; h > 0; h >>= 1) {  // pairwise: no serial chain of fp64 adds
#pragma unroll
        for (int e = 0; e < h; ++e) w[e] += w[e + h], q[e] += q[e + h];
      }
      st += w[0];
      su += q[0];
    }
#pragma unroll
    {  // warp combine: the warp's max first, then one rescale per lane and plain sums
      float M = m, ML = mL;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        ML = fmaxf(ML, __shfl_xor_sync(0xffffffffu, ML, o));
      }
      st = warp_sum(m == -INFINITY ? 0.0 : st * exp_neg(unit_t ? (double)m - M : ((double)m - M) * inv_t, tab));
      su = warp_sum(su * ex2(mL - ML));
      m = M;
      mL = ML;
    }
    if (lane == 0) {
      s_m[warp] = m;
      s_t[warp] = st;
      s_ml[warp] = mL;
      s_su[warp] = su;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float M = -INFINITY, ML = kNegInit * kL2E;
      for (int j = 0; j < kDecWarps; ++j) M = fmaxf(M, s_m[j]), ML = fmaxf(ML, s_ml[j]);
      double T = 0.0, U = 0.0;
      for (int j = 0; j < kDecWarps; ++j) {
        s_t[j] = s_m[j] == -INFINITY ? 0.0
                                      : s_t[j] * exp_neg(unit_t ? (double)s_m[j] - M : ((double)s_m[j] - M) * inv_t, tab);
        T += s_t[j];
        U += (double)s_su[j] * exp2((double)s_ml[j] - (double)ML);
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
      s_M = M;
      s_lse = ((double)ML + log2(U)) / (double)kL2E;  // untempered lse (policy.cpp:117-121)
      s_pick = V - 1;                                 // policy.cpp:160: no crossing -> last token
    }
    __syncthreads();
    const int jw = s_warp;
    if (jw >= 0) {
      // pass 2a: the 8 warps split the crossing warp's range into 8 sub-ranges
      // and sum their weights (relative to the row max) in parallel
      const double M = s_M;
      const int a0 = jw * W, a1 = min(V, a0 + W);
      const int W2 = ((W + kDecWarps - 1) / kDecWarps + 32 * E - 1) / (32 * E) * (32 * E);
      {
        const int c0 = a0 + warp * W2, c1 = min(a1, c0 + W2);
        double ls = 0.0;
        for (int b = c0 + lane * E; b < c1; b += 32 * E) {
          float x[8];
          double w[8];
          load_e<ET>(z, b, c1, vec_ok, x);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            w[e] = b + e < c1 ? exp_neg(scaled_gap(x[e], M, inv_t, unit_t), tab) : 0.0;
          }
#pragma unroll
          for (int h = E / 2; h > 0; h >>= 1) {
#pragma unroll
            for (int e = 0; e < h; ++e) w[e] += w[e + h];
          }
          ls += w[0];
        }
        ls = warp_sum(ls);
        if (lane == 0) s_t[warp] = ls;  // pass 1's warp sums are no longer needed
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const double X = s_thresh;
        double base = s_base;
        int k = kDecWarps - 1;  // rounding between the rescaled totals and the sub-range sums: last sub-range
        for (int j = 0; j < kDecWarps; ++j) {
          if (X < base + s_t[j]) {
            k = j;
            break;
          }
          if (j < kDecWarps - 1) base += s_t[j];
        }
        s_warp = k;
        s_base = base;
      }
      __syncthreads();
      // pass 2b: one warp walks the crossing sub-range in token order
      const int ks = s_warp;
      if (warp == 0) {
        const double X = s_thresh;
        double acc = s_base;
        const int c0 = min(a1, a0 + ks * W2), c1 = min(a1, c0 + W2);
        int pick = -1;
        for (int b0 = c0; b0 < c1 && pick < 0; b0 += 32 * E) {
          const int b = b0 + lane * E;
          float x[8];
          double w[8], ls = 0.0;
          load_e<ET>(z, b, c1, vec_ok, x);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            w[e] = b + e < c1 ? exp_neg(scaled_gap(x[e], M, inv_t, unit_t), tab) : 0.0;
            ls += w[e];
          }
          double incl = ls;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {  // inclusive prefix of the lane sums
            const double q = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += q;
          }
          const unsigned hit = __ballot_sync(0xffffffffu, b < c1 && X < acc + incl);
          if (hit) {
            const int hl = __ffs(hit) - 1;
            int c = min(b + E, c1) - 1;  // rounding between the lane sum and the in-order walk: lane's last token
            double a = acc + incl - ls;  // exclusive prefix: the walk resumes at this lane's first token
            for (int e = 0; e < E; ++e) {
              a += w[e];
              if (b + e < c1 && X < a) {
                c = b + e;
                break;
              }
            }
            pick = __shfl_sync(0xffffffffu, c, hl);
          }
          acc += __shfl_sync(0xffffffffu, incl, 31);
        }
        // a crossing placed here by the sums but missed by the in-order prefix
        // (rounding at a CDF boundary): the sub-range's last token
        if (lane == 0) s_pick = pick >= 0 ? pick : max(c0, c1 - 1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int c = s_pick;
      out_tok[row] = c;
      out_lp[row] = (float)((double)logit(z, c) - s_lse);  // untempered logp (policy.cpp:168)
    }
    __syncthreads();
  }
}

// The screened pass over every row: the certified rows get their token and
// log-prob; the others are marked out_tok = -1 for the fp64 kernel's redo.
template <typename ET>
__global__ void __launch_bounds__(kDecWarps * 32, RLO_SCREEN_MINB)
    decode_screen_kernel(const ET* __restrict__ logits, int64_t stride, int V, int n, double temp, uint64_t seed,
                         uint64_t version, const uint64_t* __restrict__ keys, const uint64_t* __restrict__ positions,
                         int32_t* __restrict__ out_tok, float* __restrict__ out_lp, double eps_e, double fixed) {
  constexpr int E = RawVec<ET>::E;
  __shared__ double s_t[kDecWarps], s_u2[kDecWarps];
  __shared__ double s_step[kStepMax];
  __shared__ float s_mt[kDecWarps], s_ml[kDecWarps];
  __shared__ double s_thresh, s_total, s_lse;
  __shared__ int s_warp, s_pick, s_ok;
  const bool unit_t = temp == 1.0;
  const float cT = unit_t ? kL2E : (float)((double)kL2E / temp);  // tempered log2 scale
  const int W = ((V + kDecWarps - 1) / kDecWarps + 32 * E - 1) / (32 * E) * (32 * E);
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(logits) & 15u) == 0) && (((stride * (int64_t)sizeof(ET)) & 15) == 0);
  for (int row = blockIdx.x; row < n; row += gridDim.x) {
    const ET* z = logits + (int64_t)row * stride;
    const bool ok = screened_row<ET>(z, V, W, vec_ok, unit_t, cT, eps_e, fixed,
                                     keyed_double4(seed, version, keys[row], positions[row]), s_t, s_u2, s_mt, s_ml,
                                     s_step, s_thresh, s_total, s_lse, s_warp, s_pick, s_ok);
    if (threadIdx.x == 0) {
      out_tok[row] = ok ? s_pick : -1;
      if (ok) out_lp[row] = (float)((double)logit(z, s_pick) - s_lse);  // untempered logp (policy.cpp:168)
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_decode(const void* logits, int32_t dtype, int64_t stride, int32_t V, int32_t n, double temperature,
                          uint64_t seed, uint64_t version, const uint64_t* keys, const uint64_t* positions,
                          int32_t* out_tok, float* out_lp, int num_sms, const Tuning& tu, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int grid = n < num_sms * 8 ? n : num_sms * 8;
  // Tuning (read at rlo_create): a fixed margin instead of the derived one (<= 0: no screen)
  const double fixed = tu.decode_fixed_margin ? tu.decode_margin : -1.0;
  const double eps_e = screen_eps(V);
  const bool screen = !tu.decode_fixed_margin || fixed > 0.0;
  const bool bf = dtype == RLO_DTYPE_BF16;
  if (screen) {
    if (bf)
      decode_screen_kernel<__nv_bfloat16><<<grid, kDecWarps * 32, 0, s>>>(
          reinterpret_cast<const __nv_bfloat16*>(logits), stride, V, n, temperature, seed, version, keys, positions,
          out_tok, out_lp, eps_e, fixed);
    else
      decode_screen_kernel<float><<<grid, kDecWarps * 32, 0, s>>>(reinterpret_cast<const float*>(logits), stride, V,
                                                                  n, temperature, seed, version, keys, positions,
                                                                  out_tok, out_lp, eps_e, fixed);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  const bool redo = screen;  // the fp64 kernel redoes only the rows the screen left (out_tok = -1)
  if (redo && tu.decode_noredo) return cudaGetLastError();  // diagnostics: leave the screen's -1 marks
  if (bf)
    decode_kernel<__nv_bfloat16><<<grid, kDecWarps * 32, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(logits), stride,
                                                                  V, n, temperature, seed, version, keys,
                                                                  positions, out_tok, out_lp, redo);
  else
    decode_kernel<float><<<grid, kDecWarps * 32, 0, s>>>(reinterpret_cast<const float*>(logits), stride, V, n,
                                                         temperature, seed, version, keys, positions, out_tok,
                                                         out_lp, redo);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace rlo
