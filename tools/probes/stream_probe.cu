// stream_probe.cu — the memory ceiling of the vocab pass's access pattern.
// Streams NT tensors of R rows x RB bytes with the LDG kernel's layout
// (persistent grid #SM x 4 CTAs x 256 threads, rows strided over CTAs,
// U 16-byte ld.global.nc.L1::no_allocate per thread per batch, one
// __syncthreads per row) but with trivial work per word (XOR), so the
// difference to the real pass is what the math costs.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_probe tools/probes/stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int U, int NT>
__global__ void __launch_bounds__(256, 4) stream_kernel(const uint4* t0, const uint4* t1, const uint4* t2, int64_t rows,
                                                        int nvec, unsigned* out) {
  __shared__ unsigned red[8];
  const uint4* ts[3] = {t0, t1, t2};
  unsigned acc = 0;
  const int tid = threadIdx.x;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      const uint4* row = ts[k] + r * nvec + tid;
      for (int base = 0; base + 256 * U <= nvec; base += 256 * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(row + base + u * 256);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
      }
    }
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) acc ^= red[1] ^ red[7];
  }
  if (acc == 0x12345678u) out[0] = acc;  // keep the loads
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? atoll(argv[1]) : 32768;
  const int64_t rb = argc > 2 ? atoll(argv[2]) : 304128;  // bytes per row (V=152064 bf16)
  const int U = argc > 3 ? atoi(argv[3]) : 4;
  const int nvec = (int)(rb / 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4* t[3];
  for (int k = 0; k < 3; ++k) {
    cudaMalloc(&t[k], rows * rb);
    cudaMemset(t[k], k + 1, rows * rb);
  }
  unsigned* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&]() {
    if (U == 8) stream_kernel<8, 3><<<sms * 4, 256>>>(t[0], t[1], t[2], rows, nvec, out);
    else if (U == 2) stream_kernel<2, 3><<<sms * 4, 256>>>(t[0], t[1], t[2], rows, nvec, out);
    else stream_kernel<4, 3><<<sms * 4, 256>>>(t[0], t[1], t[2], rows, nvec, out);
  };
  for (int i = 0; i < 3; ++i) run();
  cudaEventRecord(e0);
  const int it = 20;
  for (int i = 0; i < it; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 3.0 * rows * (double)(nvec / (256 * U) * 256 * U) * 16;
  printf("stream_probe rows=%lld row_bytes=%lld U=%d: %.3f ms/launch, %.0f GB/s (%s)\n", (long long)rows,
         (long long)rb, U, ms / it, bytes / (ms / it) / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
