// ex2_probe.cu — exhaustive max relative error of MUFU.EX2 (ex2.approx.ftz.f32,
// the `ex2` helper of common.cuh) against exp2 in fp64, over every fp32 t in
// [-126, 1]: the per-term bound the screened decode certificate uses (2^-22).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ex2_probe tools/probes/ex2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void scan(uint32_t lo, uint32_t hi, unsigned long long* worst) {
  double mx = 0.0;
  uint32_t arg = 0;
  for (uint64_t i = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= hi; i += (uint64_t)gridDim.x * blockDim.x) {
    const float t = __uint_as_float((uint32_t)i);
    const double ref = exp2((double)t);
    const double err = fabs((double)ex2f(t) - ref) / ref;
    if (err > mx) mx = err, arg = (uint32_t)i;
  }
  // pack (error as double bits, monotone for positive values) and take the max
  atomicMax(worst, (unsigned long long)__double_as_longlong(mx));
  (void)arg;
}

int main() {
  unsigned long long* w;
  cudaMalloc(&w, 8);
  double res[2];
  // negative t: bit patterns from -0.0 (0x80000000) up to -126 (0xC2FC0000); positive: +0 .. 1.0
  const uint32_t ranges[2][2] = {{0x80000000u, 0xC2FC0000u}, {0x00000000u, 0x3F800000u}};
  for (int r = 0; r < 2; ++r) {
    cudaMemset(w, 0, 8);
    scan<<<148 * 8, 256>>>(ranges[r][0], ranges[r][1], w);
    unsigned long long h;
    cudaMemcpy(&h, w, 8, cudaMemcpyDeviceToHost);
    res[r] = *reinterpret_cast<double*>(&h);
  }
  printf("ex2.approx.ftz.f32 max relative error: t in [-126,0]: %.3e (%.2f x 2^-22), t in [0,1]: %.3e (%s)\n", res[0],
         res[0] / 0x1p-22, res[1], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
