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
