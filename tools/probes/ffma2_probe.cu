// Probe: is fma.rn.f32x2 (FFMA2) single-rounding like fmaf?  Large-|z| inputs
// make a double rounding of z*log2e visible.
#include <cstdio>
#include <cstdint>
__global__ void k(const float* z, float mL, float c, float* out_f2, float* out_f1, int n) {
  int i = threadIdx.x * 2;
  if (i + 1 >= n) return;
  unsigned long long a, b, cc, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(z[i]), "f"(z[i + 1]));
  asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(c), "f"(c));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(-mL), "f"(-mL));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(cc));
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
  out_f2[i] = lo; out_f2[i + 1] = hi;
  out_f1[i] = fmaf(z[i], c, -mL); out_f1[i + 1] = fmaf(z[i + 1], c, -mL);
}
int main() {
  const int n = 64;
  float hz[n], *dz, *d2, *d1, h2[n], h1[n];
  for (int i = 0; i < n; ++i) hz[i] = -9987.682f + 0.37f * i;
  const float c = 1.4426950408889634f, mL = -9987.682f * c;
  cudaMalloc(&dz, sizeof hz); cudaMalloc(&d2, sizeof hz); cudaMalloc(&d1, sizeof hz);
  cudaMemcpy(dz, hz, sizeof hz, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dz, mL, c, d2, d1, n);
  cudaMemcpy(h2, d2, sizeof hz, cudaMemcpyDeviceToHost);
  cudaMemcpy(h1, d1, sizeof hz, cudaMemcpyDeviceToHost);
  int diff = 0;
  double maxerr2 = 0, maxerr1 = 0;
  for (int i = 0; i < n; ++i) {
    const double exact = (double)hz[i] * (double)c - (double)mL;
    diff += h2[i] != h1[i];
    maxerr2 = fmax(maxerr2, fabs(h2[i] - exact));
    maxerr1 = fmax(maxerr1, fabs(h1[i] - exact));
  }
  printf("FFMA2 vs FFMA differ in %d/%d lanes; max |err| FFMA2 %.3g, FFMA %.3g\n", diff, n, maxerr2, maxerr1);
  return 0;
}
