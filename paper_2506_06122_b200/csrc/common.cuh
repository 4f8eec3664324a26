// common.cuh — device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rlo {

constexpr float kL2E = 1.4426950408889634f;  // log2(e) as fp32 (the exact value used in DESIGN.md error analysis)
constexpr float kNegInit = -1.0e30f;         // finite "minus infinity" for running maxima (x*log2e stays finite)

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Streaming 128-bit loads: read-only path, no L1 allocation (each logit is read once).
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

// sm_100 256-bit streaming load (LDG.E.NA.256): 32 contiguous bytes into two
// 16-byte vectors; p must be 32-byte aligned.
// RLO_LDG256_HINT (A/B): 1 = .L2::evict_first, 2 = .L2::256B prefetch, 3 = both.
#ifndef RLO_LDG256_HINT
#define RLO_LDG256_HINT 0
#endif
#if RLO_LDG256_HINT == 1
#define RLO_LD256_OP "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32"
#elif RLO_LDG256_HINT == 2
#define RLO_LD256_OP "ld.global.nc.L1::no_allocate.L2::256B.v8.b32"
#elif RLO_LDG256_HINT == 3
#define RLO_LD256_OP "ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B.v8.b32"
#else
#define RLO_LD256_OP "ld.global.nc.L1::no_allocate.v8.b32"
#endif
__device__ __forceinline__ void ld_stream256(const uint4* p, uint4& a, uint4& b) {
  asm(RLO_LD256_OP " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
}
__device__ __forceinline__ void ld_stream256(const float4* p, float4& a, float4& b) {
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
      : "l"(p));
}

// sm_100 256-bit streaming store (STG.E.256, evict-first): two 16-byte vectors
// to 32 contiguous bytes; p must be 32-byte aligned.
__device__ __forceinline__ void st_stream256(uint4* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}

// ---- packed fp32x2 (sm_100 FFMA2 / FADD2: two fp32 lanes per instruction) ----
using f2 = unsigned long long;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(f2 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^t for a pair on the FMA pipe (FA4-style MUFU offload): Cody-Waite split
// t = j + f, j = rint(t) via the 1.5*2^23 magic add, f in [-0.5, 0.5];
// degree-5 (relative error 1.9e-7 in fp32 Horner, on par with MUFU.EX2's
// ~2 ulp) or degree-4 polynomial; 2^j inserted into the exponent with one IMAD.
// Precondition (the caller clamps): t >= -126, so the exponent add stays in
// the normal range; t = -126 yields 2^-126 (1.2e-38) where MUFU would give a
// denormal or 0, below the fp32 resolution of any sum it enters (s >= 1).
template <int DEG>  // 5: rel. err 1.9e-7; 4: 2.9e-6 (enough for 1e-5 on a sum whose offloaded share is <= 1/2)
__device__ __forceinline__ f2 exp2_poly2(float tl, float th) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
  const f2 t = pk2(tl, th);
  const f2 r = fadd2(t, pk2(kMagic, kMagic));
  const f2 j = fadd2(r, pk2(-kMagic, -kMagic));
  const f2 f = ffma2(j, pk2(-1.0f, -1.0f), t);
  f2 p;
  if (DEG == 5) {
    p = ffma2(f, pk2(0x1.5bba14p-10f, 0x1.5bba14p-10f), pk2(0x1.3cea88p-7f, 0x1.3cea88p-7f));
    p = ffma2(p, f, pk2(0x1.c6b752p-5f, 0x1.c6b752p-5f));
    p = ffma2(p, f, pk2(0x1.ebf9bcp-3f, 0x1.ebf9bcp-3f));
    p = ffma2(p, f, pk2(0x1.62e42ap-1f, 0x1.62e42ap-1f));
  } else {
    p = ffma2(f, pk2(0x1.3a02ccp-7f, 0x1.3a02ccp-7f), pk2(0x1.c9fc46p-5f, 0x1.c9fc46p-5f));
    p = ffma2(p, f, pk2(0x1.ec0378p-3f, 0x1.ec0378p-3f));
    p = ffma2(p, f, pk2(0x1.62e12cp-1f, 0x1.62e12cp-1f));
  }
  p = ffma2(p, f, pk2(1.0f, 1.0f));
  float pl, ph, rl, rh;
  upk2(p, pl, ph);
  upk2(r, rl, rh);
  const uint32_t bl = __float_as_uint(rl) * 8388608u + __float_as_uint(pl);  // + (j << 23)
  const uint32_t bh = __float_as_uint(rh) * 8388608u + __float_as_uint(ph);
  return pk2(__uint_as_float(bl), __uint_as_float(bh));
}

// max / min that return NaN when either input is NaN (FMNMX.NAN, same cost as
// fmaxf / fminf, which return the other operand): a clamp of an exponent
// argument must not turn a NaN logit into a finite term -- the reference's
// log-sum-exp of a row holding a NaN is NaN (policy.cpp:117-121).
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmin_nan(float a, float b) {
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// std::clamp semantics (NaN passes through), matching policy.cpp:277/309/359.
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

// Response length of sequence b clamped to [0, T] (out-of-range lengths are
// reported by the vocab pass as an input error).
__device__ __forceinline__ int seq_len(const int32_t* lengths, int b, int T) {
  const int n = __ldg(lengths + b);
  return n < 0 ? 0 : (n > T ? T : n);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rlo
