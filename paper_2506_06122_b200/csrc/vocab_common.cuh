// vocab_common.cuh — the online log-sum-exp state, per-dtype chunk math and
// the per-row epilogue of the vocab pass (vocab.cu) and the fused update pass
// (fused.cu).
//
// State per (thread, tensor), in log2 units relative to the fp32 constant kL2E:
//   mL = running max of z*kL2E (fp32-rounded), s = sum 2^(z*kL2E - mL),
//   w  = sum 2^(z*kL2E - mL) * (z*kL2E - mL)   (entropy; actor row only).
// Per element: one FFMA (t = z*kL2E - mL), one MUFU.EX2, one FADD (+ one FFMA
// for w).  The chunk max is taken first so the rescale (one more EX2) happens
// only when a chunk raises the max.  finish() returns to natural units in
// fp64: lse = (mL + log2 s) / kL2E, H = (log2 s - w/s) / kL2E.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace vocab {

struct Acc {
  float mL;
  float s;
  float w;
};

__device__ __forceinline__ void acc_init(Acc& a) {
  a.mL = kNegInit * kL2E;
  a.s = 0.f;
  a.w = 0.f;
}

// zmax = the chunk's largest logit.  newmL is rounded explicitly (__fmul_rn):
// a contracted d = fma(-zmax, kL2E, mL) would rescale s by the unrounded max
// while the elements use the rounded one, an lse error of up to ulp(mL)/2 --
// 2e-4 nats at |z| ~ 1e4.
template <bool ENT>
__device__ __forceinline__ void acc_rescale(Acc& a, float zmax) {
  const float newmL = __fmul_rn(zmax, kL2E);
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
  if (ENT) w = fmaf(e, fmaxf(t, kNegInit), w);  // guard: -inf logits give e = 0, not 0 * -inf
}

template <bool ENT>
__device__ __forceinline__ void acc_combine(Acc& a, float mL2, float s2, float w2) {
  const float M = fmaxf(a.mL, mL2);
  const float d1 = a.mL - M, d2 = mL2 - M;
  const float e1 = ex2(d1), e2 = ex2(d2);
  if (ENT) a.w = (a.w + a.s * d1) * e1 + (w2 + s2 * d2) * e2;
  a.s = a.s * e1 + s2 * e2;
  a.mL = M;
}

#ifndef RLO_WARP_REDUCE_PAIRWISE
#define RLO_WARP_REDUCE_PAIRWISE 0
#endif
// Warp reduction of the online state: the warp's max first (5 FMNMX
// shuffles), then one rescale per lane and plain shuffle sums — one EX2 per
// lane instead of two per level (RLO_WARP_REDUCE_PAIRWISE=1: the pairwise
// combine at every level, kept for A/B).
template <bool ENT>
__device__ __forceinline__ void acc_warp_reduce(Acc& a) {
  if (RLO_WARP_REDUCE_PAIRWISE) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, a.mL, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, a.s, o);
      const float w2 = ENT ? __shfl_xor_sync(0xffffffffu, a.w, o) : 0.f;
      acc_combine<ENT>(a, m2, s2, w2);
    }
    return;
  }
  float M = a.mL;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  const float d = a.mL - M, sc = ex2(d);
  float s = a.s * sc, w = 0.f;
  if (ENT) w = (a.w + a.s * d) * sc;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ENT) w += __shfl_xor_sync(0xffffffffu, w, o);
  }
  a.mL = M;
  a.s = s;
  if (ENT) a.w = w;
}

// ---- per-dtype 16-byte vector math -------------------------------------------
//
// MATH selects the per-element instruction mix (compile-time; the shipped
// defaults per dtype are in vocab.cu: fp32 1, bf16 6 | kMathLazy, bf16 short
// 3-tensor rows 6; the others are A/B options):
//   0  scalar FFMA / MUFU.EX2 / FADD per element;
//   1  packed: FFMA2 / FADD2 on element pairs, MUFU.EX2 per element;
//   2  as 1, plus 1 of 4 element pairs of each non-entropy row through the
//      FMA-pipe degree-5 polynomial exp2 (exp2_poly2) instead of MUFU (25%);
//   3  as 2 with 2 of 4 pairs (50% offload);
//   4  degree-4 polynomial on 1 of 4 pairs of every row, the entropy
//      (actor) row included (25% of all exponentials);
//   5  degree-4 polynomial on 2 of 4 pairs of the old/ref rows (50%);
//   6  as 4 on the old/ref rows, the entropy (actor) row all MUFU.
// Degree 4 has relative error 2.9e-6 per term, so with at most half of a
// row's mass offloaded the lse error stays below 1.5e-6.

// MATH -> polynomial degree of the offloaded pairs (0: none) and whether half
// (rather than a quarter) of the old/ref element pairs are offloaded.
__host__ __device__ constexpr int poly_deg(int math) {
  return math == 2 || math == 3 ? 5 : math == 4 || math == 5 || math == 6 || math == 9 ? 4 : 0;
}
// mix 9: as 6 with the polynomial on the .y word of every other vector only (12.5%).
__host__ __device__ constexpr bool poly_odd_only(int math) { return math == 9; }
__host__ __device__ constexpr bool poly_half(int math) { return math == 3 || math == 5; }
__host__ __device__ constexpr int poly_deg_ent(int math) { return math == 4 ? 4 : 0; }
// Template MATH values may carry kMathGuard (the guarded entropy-row variant).
constexpr int kMathMask = 0xff;
constexpr int kMathGuard = 0x100;
// kMathNoMax: the caller already rescaled the state to a shared running max
// (lockstep streams of several tensors, vocab.cu); skip the per-chunk max.
constexpr int kMathNoMax = 0x200;
// kMathLazy: once a thread's state holds a real running max, a chunk is first
// summed against that max without taking the chunk max; only if the chunk sum
// reaches kLazyCap (an element more than ~27 log2 units above the running
// max, or a non-finite value) is the chunk redone the exact way (chunk max,
// rescale, sum).  The offset of an online log-sum-exp need not be the maximum
// -- any offset that keeps the terms finite gives the same lse and entropy
// (H = log2 s - w/s holds for every offset) -- so this drops the per-element
// max (one HMNMX2 / FMNMX per pair) from almost every chunk.
constexpr int kMathLazy = 0x400;
// kMathDeferred: the offset is the max of the thread's FIRST batch of the
// row (exact path) and every later batch is summed against it with no check
// at all -- no per-batch max, test or branch; the batch sums go into packed
// accumulators.  Valid for the same reason as the lazy max (any offset that
// keeps the terms finite gives the same lse and entropy); a thread whose
// share ends with s >= kDeferCap or a non-finite s / w (an element ~110 log2
// units above that offset: MUFU lanes overflow to inf, polynomial lanes clamp
// at 2^127; or -inf logits in the entropy row) is redone the exact way by the
// caller (stream_checked).
constexpr int kMathDeferred = 0x800;
constexpr float kDeferCap = 0x1p110f;
constexpr float kLazyCap = 4294967296.0f;  // 2^32
constexpr float kLazyMin = -1.0e29f;      // mL above this holds a real max (init is kNegInit * kL2E)

// GUARD (entropy row): clamp t so that -inf logits (masked vocabulary
// entries) give e*t = 2^-126 * -126 (negligible) instead of 0 * -inf = NaN.
// Two FMNMX per element pair, so the entropy row runs unguarded and a thread
// whose entropy sum comes out non-finite redoes its share guarded (vocab.cu,
// fused.cu); the batch padding is finite (fill()) and never triggers it.
template <bool ENT, bool GUARD>
__device__ __forceinline__ void pair2(float zl, float zh, f2 L2, f2 nmL, f2& s, f2& w, int poly) {
  const f2 t = ffma2(pk2(zl, zh), L2, nmL);
  float tl, th;
  upk2(t, tl, th);
  if (poly) {
    // the polynomial's domain: 2^j is inserted into the exponent field, so j
    // must stay in [-126, 127].  The upper clamp matters under the lazy max
    // and lockstep streams, where t can be positive: an element far above the
    // running max then yields 2^127 (the chunk sum fails the lazy cap / the
    // lockstep range check and is redone the exact way) instead of a wrapped
    // exponent that would silently drop the dominant term.
    // (NaN-propagating clamps: a NaN logit keeps the share NaN, as in the reference)
    tl = fmin_nan(fmax_nan(tl, -126.0f), 127.0f);
    th = fmin_nan(fmax_nan(th, -126.0f), 127.0f);
  } else if (ENT && GUARD) {
    tl = fmax_nan(tl, -126.0f);
    th = fmax_nan(th, -126.0f);
  }
  const f2 e = poly == 5 ? exp2_poly2<5>(tl, th) : poly == 4 ? exp2_poly2<4>(tl, th) : pk2(ex2(tl), ex2(th));
  s = fadd2(s, e);
  if (ENT) w = ffma2(e, pk2(tl, th), w);
}

__device__ __forceinline__ float hsum2(f2 a, f2 b) {
  float l, h;
  upk2(fadd2(a, b), l, h);
  return l + h;
}

template <typename ET>
struct Vec;

// One chunk (U 16-byte vectors) into the online state: chunk max + rescale,
// then the sums (or, under kMathLazy, the sums against the current max first).
template <typename VT, int U, bool ENT, int MATHG>
__device__ __forceinline__ void accumulate_chunk(const typename VT::V (&v)[U], Acc& a) {
  float cs, cw = 0.f;
  if (MATHG & kMathLazy) {
    if (a.mL > kLazyMin) {
      VT::template sums<U, ENT, MATHG>(v, a.mL, cs, cw);
      if (cs < kLazyCap) {  // false for inf / NaN: those chunks take the exact path below
        a.s += cs;
        if (ENT) a.w += cw;
        return;
      }
    }
  }
  if (!(MATHG & kMathNoMax)) acc_rescale<ENT>(a, VT::template chunk_max<U>(v));
  VT::template sums<U, ENT, MATHG>(v, a.mL, cs, cw);
  constexpr int kM = MATHG & kMathMask;
  if constexpr ((MATHG & kMathNoMax) == 0 && (ENT ? poly_deg_ent(kM) : poly_deg(kM)) > 0) {
    // Against the chunk's own max every term is <= 1, so a sum >= 2^100 can
    // only come from a NaN logit in a polynomial lane: the exponent insertion
    // of exp2_poly2 turns the NaN into FLT_MAX.  Keep it NaN, as MUFU lanes
    // and the reference do (the lazy / lockstep checks above route such
    // chunks and shares here).
    if (!(cs < 0x1p100f)) cs = __int_as_float(0x7fffffff);
  }
  a.s += cs;
  if (ENT) a.w += cw;
}

template <>
struct Vec<float> {
  using V = float4;
  static constexpr int kElems = 4;
  // Padding of a partial batch: -1e38 contributes 2^(-1.44e38) = 0, never
  // raises the running max (init -1.44e30), and being finite keeps the
  // unguarded entropy product e*t = 0*(-1.44e38) = 0 (a -inf pad would give
  // NaN).  t stays finite: -1e38*log2e - m > -3.4e38.
  __device__ static V fill() { return make_float4(-1e38f, -1e38f, -1e38f, -1e38f); }
  template <int U>
  __device__ static float chunk_max(const V (&v)[U]) {
    float m = fmaxf(fmaxf(v[0].x, v[0].y), fmaxf(v[0].z, v[0].w));
#pragma unroll
    for (int u = 1; u < U; ++u) m = fmaxf(m, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
    return m;
  }
  // The chunk's sums relative to the offset mL (no max, no state update).
  template <int U, bool ENT, int MATHG>
  __device__ static void sums(const V (&v)[U], float mL, float& cs, float& cw) {
    constexpr int MATH = MATHG & kMathMask;
    constexpr bool G = (MATHG & kMathGuard) != 0;
    if (MATH == 0) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc_elem<ENT>(v[u].x, mL, s0, w0);
        acc_elem<ENT>(v[u].y, mL, s1, w1);
        acc_elem<ENT>(v[u].z, mL, s2, w2);
        acc_elem<ENT>(v[u].w, mL, s3, w3);
      }
      cs = (s0 + s1) + (s2 + s3);
      if (ENT) cw = (w0 + w1) + (w2 + w3);
    } else {
      const f2 L2 = pk2(kL2E, kL2E), nmL = pk2(-mL, -mL);
      f2 s0 = 0, s1 = 0, w0 = 0, w1 = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) vec_sums<ENT, MATHG>(v[u], u, L2, nmL, s0, s1, w0, w1);
      cs = hsum2(s0, s1);
      if (ENT) cw = hsum2(w0, w1);
    }
  }
  // One vector (position u of its batch) into packed accumulators (MATH != 0).
  template <bool ENT, int MATHG>
  __device__ static void vec_sums(const V& v, int u, f2 L2, f2 nmL, f2& s0, f2& s1, f2& w0, f2& w1) {
    constexpr int MATH = MATHG & kMathMask;
    constexpr bool G = (MATHG & kMathGuard) != 0;
    pair2<ENT, G>(v.x, v.y, L2, nmL, s0, w0, 0);
    pair2<ENT, G>(v.z, v.w, L2, nmL, s1, w1, (!ENT && (u & 1)) ? poly_deg(MATH) : 0);
  }
  template <int U, bool ENT, int MATHG>
  __device__ static void accumulate(const V (&v)[U], Acc& a) {
    accumulate_chunk<Vec<float>, U, ENT, MATHG>(v, a);
  }
  __device__ static float scalar(const float* p) { return __ldg(p); }
};

template <>
struct Vec<__nv_bfloat16> {
  using V = uint4;
  static constexpr int kElems = 8;
  __device__ static V fill() { return make_uint4(0xFE97FE97u, 0xFE97FE97u, 0xFE97FE97u, 0xFE97FE97u); }  // -1.004e38
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
  template <int U, bool ENT, int MATHG>
  __device__ static void sums(const V (&v)[U], float mL, float& cs, float& cw) {
    constexpr int MATH = MATHG & kMathMask;
    constexpr bool G = (MATHG & kMathGuard) != 0;
    if (MATH == 0) {
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        word<ENT>(v[u].x, mL, s0, s1, w0, w1);
        word<ENT>(v[u].y, mL, s2, s3, w2, w3);
        word<ENT>(v[u].z, mL, s0, s1, w0, w1);
        word<ENT>(v[u].w, mL, s2, s3, w2, w3);
      }
      cs = (s0 + s1) + (s2 + s3);
      if (ENT) cw = (w0 + w1) + (w2 + w3);
    } else {
      const f2 L2 = pk2(kL2E, kL2E), nmL = pk2(-mL, -mL);
      f2 s0 = 0, s1 = 0, w0 = 0, w1 = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) vec_sums<ENT, MATHG>(v[u], u, L2, nmL, s0, s1, w0, w1);
      cs = hsum2(s0, s1);
      if (ENT) cw = hsum2(w0, w1);
    }
  }
  // One vector into packed accumulators (MATH != 0): the polynomial lanes are
  // the .y word (and, for half offload, the .w word) of every vector.
  template <bool ENT, int MATHG>
  __device__ static void vec_sums(const V& v, int u, f2 L2, f2 nmL, f2& s0, f2& s1, f2& w0, f2& w1) {
    constexpr int MATH = MATHG & kMathMask;
    constexpr bool G = (MATHG & kMathGuard) != 0;
    const int py = ENT ? poly_deg_ent(MATH) : (poly_odd_only(MATH) && !(u & 1)) ? 0 : poly_deg(MATH);
    pair2<ENT, G>(bf16lo(v.x), bf16hi(v.x), L2, nmL, s0, w0, 0);
    pair2<ENT, G>(bf16lo(v.y), bf16hi(v.y), L2, nmL, s1, w1, py);
    pair2<ENT, G>(bf16lo(v.z), bf16hi(v.z), L2, nmL, s0, w0, 0);
    pair2<ENT, G>(bf16lo(v.w), bf16hi(v.w), L2, nmL, s1, w1, (ENT || !poly_half(MATH)) ? 0 : poly_deg(MATH));
  }
  template <int U, bool ENT, int MATHG>
  __device__ static void accumulate(const V (&v)[U], Acc& a) {
    accumulate_chunk<Vec<__nv_bfloat16>, U, ENT, MATHG>(v, a);
  }
  __device__ static float scalar(const __nv_bfloat16* p) {
    return __bfloat162float(__ldg(reinterpret_cast<const __nv_bfloat16*>(p)));
  }
};

template <typename ET>
__device__ __forceinline__ float load_logit(const void* base, int64_t off) {
  return Vec<ET>::scalar(reinterpret_cast<const ET*>(base) + off);
}

// One element, scalar (row heads / tails).
template <typename ET, bool ENT>
__device__ __forceinline__ void acc_scalar(const ET* p, Acc& a) {
  const float z = Vec<ET>::scalar(p);
  acc_rescale<ENT>(a, z);
  float w = 0.f, s = 0.f;
  acc_elem<ENT>(z, a.mL, s, w);
  a.s += s;
  if (ENT) a.w += w;
}

// 256-bit loads (sm_100 LDG.256) in the prefetching layout (the bf16 default):
// +0.5-0.8% on cfg3 (profiles/r2_vocab_ab.txt); in the non-prefetching
// layout (the fp32 default, U = 8) they lost 3.5% on cfg2 and stay off.
#ifndef RLO_LDG256
#define RLO_LDG256 1
#endif
#ifndef RLO_LDG256_NOPF
#define RLO_LDG256_NOPF 0
#endif

// One row (or row slice) of V elements streamed by NTH threads with U 128-bit
// loads in flight per thread.  A row that does not start on a 16-byte
// boundary (e.g. V = 50257 in a contiguous tensor) takes its first few
// elements scalar and the aligned body vectorised.  PF: software prefetch —
// the next batch's U loads are issued before the current batch's math,
// doubling the bytes in flight per thread.
template <int NTH, typename ET, int U, bool PF, bool ENT, int MATH>
__device__ __forceinline__ void stream_accumulate(const ET* __restrict__ row, int V, Acc& a) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  constexpr int kStep = NTH * U;
  const int tid = threadIdx.x;
  const int mis = (int)(reinterpret_cast<uintptr_t>(row) & 15u);
  const int head = min(V, mis ? (16 - mis) / (int)sizeof(ET) : 0);  // elements before the first 16-byte boundary
  if (tid < head) acc_scalar<ET, ENT>(row + tid, a);
  row += head;
  V -= head;
  const int nvec = V / VT::kElems;
  const int nfull = nvec / kStep * kStep;
  const VV* __restrict__ vrow = reinterpret_cast<const VV*>(row) + tid;
  if constexpr (PF && (MATH & kMathDeferred) != 0) {
    constexpr int kExact = MATH & ~kMathDeferred;
    const f2 L2 = pk2(kL2E, kL2E);
    f2 nmL = pk2(-a.mL, -a.mL);
    f2 S0 = 0, S1 = 0, W0 = 0, W1 = 0;
    auto batch = [&](const VV (&v)[U]) {
      if (!(a.mL > kLazyMin)) {  // the thread's first batch of the row: exact, sets the offset
        VT::template accumulate<U, ENT, kExact>(v, a);
        nmL = pk2(-a.mL, -a.mL);
        return;
      }
      f2 c0 = 0, c1 = 0, d0 = 0, d1 = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) VT::template vec_sums<ENT, kExact>(v[u], u, L2, nmL, c0, c1, d0, d1);
      S0 = fadd2(S0, c0);
      S1 = fadd2(S1, c1);
      if (ENT) {
        W0 = fadd2(W0, d0);
        W1 = fadd2(W1, d1);
      }
    };
    if (nfull > 0) {
      VV cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = ld_stream(vrow + u * NTH);
      for (int base = kStep; base < nfull; base += kStep) {
        VV nxt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = ld_stream(vrow + base + u * NTH);
        batch(cur);
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = nxt[u];
      }
      batch(cur);
    }
    a.s += hsum2(S0, S1);  // before the exact tail, which may rescale the state
    if (ENT) a.w += hsum2(W0, W1);
  } else if (PF && RLO_LDG256 && (U % 2) == 0) {
    // 256-bit loads: thread tid takes the vector pairs (2 tid, 2 tid + 1) of
    // each 2*NTH-vector group of the batch -- one LDG.256 per pair, half the
    // load instructions, a warp reads 1 KB contiguous per load.  Rows whose
    // aligned body does not start on 32 bytes take the 16-byte layout below.
    if (nfull > 0 && (reinterpret_cast<uintptr_t>(row) & 31u) == 0) {
      const VV* __restrict__ prow = reinterpret_cast<const VV*>(row) + 2 * tid;
      VV cur[U];
#pragma unroll
      for (int u = 0; u < U; u += 2) ld_stream256(prow + u * NTH, cur[u], cur[u + 1]);
      for (int base = kStep; base < nfull; base += kStep) {
        VV nxt[U];
#pragma unroll
        for (int u = 0; u < U; u += 2) ld_stream256(prow + base + u * NTH, nxt[u], nxt[u + 1]);
        VT::template accumulate<U, ENT, MATH>(cur, a);
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = nxt[u];
      }
      VT::template accumulate<U, ENT, MATH>(cur, a);
    } else if (nfull > 0) {
      VV cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = ld_stream(vrow + u * NTH);
      for (int base = kStep; base < nfull; base += kStep) {
        VV nxt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = ld_stream(vrow + base + u * NTH);
        VT::template accumulate<U, ENT, MATH>(cur, a);
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = nxt[u];
      }
      VT::template accumulate<U, ENT, MATH>(cur, a);
    }
  } else if (PF) {
    if (nfull > 0) {
      VV cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = ld_stream(vrow + u * NTH);
      for (int base = kStep; base < nfull; base += kStep) {
        VV nxt[U];
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = ld_stream(vrow + base + u * NTH);
        VT::template accumulate<U, ENT, MATH>(cur, a);
#pragma unroll
        for (int u = 0; u < U; ++u) cur[u] = nxt[u];
      }
      VT::template accumulate<U, ENT, MATH>(cur, a);
    }
  } else if (RLO_LDG256_NOPF && (U % 2) == 0 && (reinterpret_cast<uintptr_t>(row) & 31u) == 0) {
    const VV* __restrict__ prow = reinterpret_cast<const VV*>(row) + 2 * tid;  // 256-bit pairs, as above
    for (int base = 0; base < nfull; base += kStep) {
      VV v[U];
#pragma unroll
      for (int u = 0; u < U; u += 2) ld_stream256(prow + base + u * NTH, v[u], v[u + 1]);
      VT::template accumulate<U, ENT, MATH>(v, a);
    }
  } else {
    for (int base = 0; base < nfull; base += kStep) {  // full batches: unpredicated loads
      VV v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream(vrow + base + u * NTH);
      VT::template accumulate<U, ENT, MATH>(v, a);
    }
  }
  if (nfull < nvec) {  // last partial batch (exact path under kMathDeferred)
    VV v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = nfull + u * NTH + tid;
      v[u] = idx < nvec ? ld_stream(vrow - tid + idx) : VT::fill();
    }
    VT::template accumulate<U, ENT, MATH & ~kMathDeferred>(v, a);
  }
  for (int i = nvec * VT::kElems + tid; i < V; i += NTH) acc_scalar<ET, ENT>(row + i, a);  // scalar tail
}

// stream_accumulate plus the deferred check: a share whose state left the
// safe range (see kMathDeferred) is redone the exact way (entropy rows
// guarded); the redo re-reads the thread's share, which the stream has just
// brought through L2.
template <int NTH, typename ET, int U, bool PF, bool ENT, int MATH>
__device__ __forceinline__ void stream_checked(const ET* __restrict__ row, int V, Acc& a) {
  stream_accumulate<NTH, ET, U, PF, ENT, MATH>(row, V, a);
  constexpr bool kDeferred = (MATH & kMathDeferred) != 0;
  if constexpr (kDeferred || ENT) {
    // deferred: overflowed or not finite; lazy / exact entropy rows: -inf
    // logits make the unguarded e * t = 0 * -inf NaN (w - w != 0 for inf / NaN)
    // (entropy rows: s < 2^32 as the lazy cap -- a share max far above the
    // offset would cancel the bits of log2 s - w/s)
    const bool bad = kDeferred ? (!(a.s < (ENT ? kLazyCap : kDeferCap)) || (ENT && !(a.w - a.w == 0.f)))
                               : !(isfinite(a.s) && isfinite(a.w));
    if (bad) {
      acc_init(a);
      stream_accumulate<NTH, ET, U, PF, ENT, (MATH & ~kMathDeferred) | (ENT ? kMathGuard : 0)>(row, V, a);
    }
  }
}

struct RowResult {
  double lse;
  double entropy;
};

__device__ __forceinline__ RowResult finish(const Acc& a) {
  const double l2 = log2((double)a.s);
  RowResult r;
  r.lse = ((double)a.mL + l2) / (double)kL2E;
  r.entropy = (l2 - (double)a.w / (double)a.s) / (double)kL2E;
  return r;
}

// Row of token (b, t) in the rank-local batch across micro-batches: (seq_offset + b) * T + t.
__device__ __forceinline__ int64_t global_row(const VocabArgs& a, int64_t row) { return row + (int64_t)a.seq_offset * a.T; }

// Report a failing row; the slot keeps the earliest in sample order (internal.h).
__device__ __forceinline__ void flag_error(const VocabArgs& a, int code, int64_t pos, int value) {
  atomicMin(&a.err->key, dev_err_key(code, pos, value));
}

// Loss epilogue for one loss-participating token (policy.cpp:355-374 + extensions), fp64.
// Returns dlogp; `write` = false computes it without touching the outputs (the
// non-leader CTAs of a fused-pass cluster).
__device__ inline double loss_epilogue(const VocabArgs& a, int64_t row, double lp, double old, bool has_ref, double ref,
                                       double ent, double lse, bool write = true) {
  const double A = (double)a.adv[row];
  const double eps = a.clip_eps;
  const double ratio = exp(lp - old);                       // policy.cpp:358
  const double rcl = clampd(ratio, 1.0 - eps, 1.0 + eps);  // :359
  const double u = ratio * A, c = rcl * A;                  // :360-361
  const double surr = (c < u) ? c : u;                      // :362 std::min
  double pg = -surr;
  bool dual = false;
  if (a.dual_c > 1.0 && A < 0.0) {  // dual-clip: cap the A<0 loss at -c*A
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
  const double loss = pg + kc * (kc > 0.0 ? k : 0.0);                   // :364-366
  const bool flows = A >= 0.0 ? ratio <= 1.0 + eps : ratio >= 1.0 - eps;  // :373
  double dlp = (flows && !dual) ? -ratio * A : 0.0;                      // :374
  dlp += kc > 0.0 ? kc * dk : 0.0;
  uint8_t flags = 0;
  if (u > c) flags |= TF_CLIPPED;  // :369
  if (dual) flags |= TF_DUAL;
  if (!isfinite(dlp)) flags |= TF_NONFINITE_GRAD;
  if (!isfinite(loss)) flags |= TF_NONFINITE_LOSS;
  if (!write) return dlp;
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
  if (a.o_lse) a.o_lse[row] = (float)lse;
  if (a.o_lse64) a.o_lse64[row] = lse;
  return dlp;
}

// Old/ref log-probs from the pass's own tensors (by role) or the caller's
// precomputed arrays, then the loss epilogue.  Returns dlogp.
template <int NT>
__device__ __forceinline__ double row_loss(const VocabArgs& a, int64_t row, const double (&lp)[NT], double ent,
                                           double lse0, bool write) {
  double old = 0.0, ref = 0.0;
  bool have_old = false, have_ref = false;
#pragma unroll
  for (int k = 1; k < NT; ++k) {
    if (a.role[k] == ROLE_OLD) {
      old = lp[k];
      have_old = true;
    }
    if (a.role[k] == ROLE_REF) {
      ref = lp[k];
      have_ref = true;
    }
  }
  if (!have_old) old = (double)a.old_lp_in[row];
  if (!have_ref && a.ref_lp_in) {
    ref = (double)a.ref_lp_in[row];
    have_ref = true;
  }
  return loss_epilogue(a, row, lp[0], old, have_ref, ref, ent, lse0, write);
}

// Is `row` processed by this pass?  (forward_logprobs: every valid position;
// loss: valid and mask != 0, policy.cpp:348-351.)  Also reports bad lengths.
template <bool LOSS>
__device__ __forceinline__ bool row_active(const VocabArgs& a, int64_t row, bool report) {
  const int b = (int)(row / a.T);
  const int t = (int)(row - (int64_t)b * a.T);
  if (report && t == 0) {
    const int raw = __ldg(a.lengths + b);
    if (raw < 0 || raw > a.T) flag_error(a, DE_BAD_LENGTH, (int64_t)a.seq_offset + b, a.seq_offset + b);
  }
  bool active = t < seq_len(a.lengths, b, a.T);
  if (LOSS && active && a.mask) active = __ldg(a.mask + row) != 0;
  return active;
}

template <bool LOSS>
__device__ __forceinline__ void write_inactive(const VocabArgs& a, int64_t row) {
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
    if (a.o_lse) a.o_lse[row] = 0.f;
    if (a.o_lse64) a.o_lse64[row] = 0.0;
  }
}

// Row number of token `row` = (b, t) in logits tensor k: packed
// (seq_start[b] + t) or padded (row itself).
__device__ __forceinline__ int64_t logits_row(const VocabArgs& a, int k, int64_t row) {
  const int64_t* ss = a.seq_start[k];
  if (!ss) return row;
  const int b = (int)(row / a.T);
  return __ldg(ss + b) + (row - (int64_t)b * a.T);
}
__device__ __forceinline__ int64_t logits_off(const VocabArgs& a, int k, int64_t row) {
  return logits_row(a, k, row) * a.stride[k];
}
// Does token `row` have a row in the actor logits (and the gradient)?  Packed
// tensors hold only t < lengths[b]; padded ones hold every (b, t).
__device__ __forceinline__ bool row_exists(const VocabArgs& a, int64_t row) {
  if (!a.seq_start[0]) return true;
  const int b = (int)(row / a.T);
  return row - (int64_t)b * a.T < seq_len(a.lengths, b, a.T);
}

// Token gather for the row (one thread): bit-exact element loads.
template <typename ET, int NT>
__device__ __forceinline__ void gather_token(const VocabArgs& a, int64_t row, int& tok, bool& oov, float (&ztok)[NT]) {
  tok = __ldg(a.tokens + row);
  oov = tok < 0 || tok >= a.V;
#pragma unroll
  for (int k = 0; k < NT; ++k) ztok[k] = oov ? 0.f : load_logit<ET>(a.logits[k], logits_off(a, k, row) + tok);
}

// Final cross-warp combine + outputs, executed by one full warp (all lanes):
// lane w holds warp w's (mL, s, w) for each tensor in c[] (acc_init beyond the
// warp count).
template <int NT, bool LOSS, bool ENT0>
__device__ __forceinline__ void row_finish_acc(const VocabArgs& a, Acc (&c)[NT], int64_t row, int tok, bool oov,
                                               const float (&ztok)[NT], int lane) {
  double lse[NT], ent = 0.0;
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    if (k == 0 && ENT0)
      acc_warp_reduce<true>(c[k]);
    else
      acc_warp_reduce<false>(c[k]);
    const RowResult r = finish(c[k]);
    lse[k] = r.lse;
    if (k == 0) ent = r.entropy;
  }
  if (lane != 0) return;
  if (oov) flag_error(a, LOSS ? DE_OOV_LOSS : DE_OOV_LOGPROB, global_row(a, row), tok);
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  double lp[NT];
#pragma unroll
  for (int k = 0; k < NT; ++k) lp[k] = oov ? nan : (double)ztok[k] - lse[k];  // policy.cpp:122, :227
  if (!LOSS) {
    a.out_lp[row] = (float)lp[0];
    if (a.out_ent) a.out_ent[row] = (float)ent;
    if (a.out_tok) a.out_tok[row] = ztok[0];
    return;
  }
  row_loss<NT>(a, row, lp, ent, lse[0], true);
}

// red[w][k][0..2] holds warp w's (mL, s, w) for tensor k.
template <int NWARPS, int NT>
__device__ __forceinline__ void load_red(const float (*red)[NT][3], Acc (&c)[NT], int lane) {
#pragma unroll
  for (int k = 0; k < NT; ++k) {
    if (lane < NWARPS) {
      c[k].mL = red[lane][k][0];
      c[k].s = red[lane][k][1];
      c[k].w = red[lane][k][2];
    } else {
      acc_init(c[k]);
    }
  }
}

template <int NT, int NWARPS, bool LOSS, bool ENT0>
__device__ __forceinline__ void row_finish(const VocabArgs& a, const float (*red)[NT][3], int64_t row, int tok,
                                           bool oov, const float (&ztok)[NT], int lane) {
  Acc c[NT];
  load_red<NWARPS, NT>(red, c, lane);
  row_finish_acc<NT, LOSS, ENT0>(a, c, row, tok, oov, ztok, lane);
}

}  // namespace vocab
}  // namespace rlo
