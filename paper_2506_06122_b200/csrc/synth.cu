// synth.cu — deterministic synthetic logits/tokens (include/rlo_synth.h) for
// the bench and the full-size parity checks.  Not on the objective path.
#include "../../include/rlo_synth.h"
#include "common.cuh"
#include "internal.h"

namespace rlo {
namespace {

__global__ void synth_logits_kernel(void* dst, int dtype, int64_t rows, int V, int64_t row_stride, uint64_t seed,
                                    int model, int64_t key_off) {
  const uint64_t k0 = rlo_synth_model_key(seed, 0), km = rlo_synth_model_key(seed, model);
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint64_t key = (uint64_t)(key_off + r);
    int32_t spikes[RLO_SYNTH_SPIKES];
#pragma unroll
    for (int k = 0; k < RLO_SYNTH_SPIKES; ++k) spikes[k] = rlo_synth_spike(seed, key, k, V);
    for (int v = threadIdx.x; v < V; v += blockDim.x) {
      const float z = rlo_synth_logit(k0, km, model, key, v, spikes);
      if (dtype == RLO_DTYPE_F32)
        reinterpret_cast<float*>(dst)[r * row_stride + v] = z;
      else
        reinterpret_cast<uint16_t*>(dst)[r * row_stride + v] = rlo_f32_to_bf16_rne(z);
    }
  }
}

__global__ void synth_tokens_kernel(int32_t* dst, int64_t rows, int V, uint64_t seed, int64_t key_off,
                                    int64_t key_rows) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = rlo_synth_token(seed, (uint64_t)((key_off + r) % key_rows), V);
}

}  // namespace

cudaError_t launch_synth_logits(void* dst, int32_t dtype, int64_t rows, int32_t V, int64_t row_stride,
                                uint64_t seed, int32_t model_id, int64_t row_key_offset, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const int64_t grid = rows < 148 * 16 ? rows : 148 * 16;
  synth_logits_kernel<<<(int)grid, 512, 0, s>>>(dst, dtype, rows, V, row_stride, seed, model_id, row_key_offset);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

cudaError_t launch_synth_tokens(int32_t* dst, int64_t rows, int32_t V, uint64_t seed, int64_t row_key_offset,
                                int64_t key_rows, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  int64_t grid = (rows + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  synth_tokens_kernel<<<(int)grid, 256, 0, s>>>(dst, rows, V, seed, row_key_offset, key_rows);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

}  // namespace rlo
