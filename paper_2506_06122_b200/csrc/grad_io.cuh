// grad_io.cuh — streaming stores of gradient rows (fp32 or bf16) shared by
// the separate backward epilogue (backward.cu) and the fused update pass
// (fused.cu).  st.global.cs: each gradient element is written once and not
// re-read by this pass.
#pragma once

#include <cuda_bf16.h>

#include "common.cuh"

namespace rlo {

template <typename GT>
struct Out;
template <>
struct Out<float> {
  template <int N>
  __device__ static void store(float* p, const float (&g)[8]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(g[0], g[1], g[2], g[3]));
    if (N == 8) __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(g[4], g[5], g[6], g[7]));
  }
  __device__ static void one(float* p, float g) { p[0] = g; }
};
template <>
struct Out<__nv_bfloat16> {
  __device__ static uint32_t pack(float lo, float hi) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(lo)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(hi)) << 16);
  }
  template <int N>
  __device__ static void store(__nv_bfloat16* p, const float (&g)[8]) {
    if (N == 8)
      __stcs(reinterpret_cast<uint4*>(p), make_uint4(pack(g[0], g[1]), pack(g[2], g[3]), pack(g[4], g[5]), pack(g[6], g[7])));
    else
      __stcs(reinterpret_cast<uint2*>(p), make_uint2(pack(g[0], g[1]), pack(g[2], g[3])));
  }
  __device__ static void one(__nv_bfloat16* p, float g) { p[0] = __float2bfloat16_rn(g); }
};

}  // namespace rlo
