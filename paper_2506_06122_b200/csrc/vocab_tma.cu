// vocab_tma.cu — the vocab pass fed by TMA bulk copies (cp.async.bulk) into a
// shared-memory ring.
//
// One CTA per SM (persistent, rows strided by gridDim):
//   * warp kConsWarps (the producer) walks the CTA's active rows and, for each
//     of the NT logits tensors, streams the row in kChunk-byte chunks:
//     wait empty[stage] -> arrive.expect_tx(full[stage]) ->
//     cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes
//     (L2 evict_first).  It runs up to kStages chunks (192 KB) ahead, across
//     row boundaries, so the row epilogues never drain the memory pipe.
//   * warps 0..kConsWarps-1 (the consumers) wait full[stage], copy their
//     slice of the chunk (4 x 16 B per thread, conflict-free LDS.128) into
//     registers, release the stage (one arrive per warp on empty[stage]) and
//     run the online log-sum-exp math (vocab_common.cuh).  Per row: warp
//     shuffles, one named barrier over the consumers, warp 0 finishes.
// Bytes in flight per SM are held in shared memory, not registers, which is
// what the latency-bound bf16 path (V=152064) needs.
#include "vocab_common.cuh"

namespace rlo {
namespace vocab {

namespace {

constexpr int kConsWarps = 16;
constexpr int kCons = kConsWarps * 32;
constexpr int kThreadsTma = kCons + 32;
constexpr int kChunk = 32768;  // bytes per stage
constexpr int kStages = 6;
constexpr int kPer = kChunk / 16 / kCons;  // 16-byte vectors per consumer thread per chunk
static_assert(kPer * 16 * kCons == kChunk, "chunk must split evenly over consumers");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH>
__global__ void __launch_bounds__(kThreadsTma, 1) vocab_tma_kernel(const VocabArgs a) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kChunk);
  uint64_t* empty = full + kStages;
  auto red = reinterpret_cast<float(*)[kConsWarps][NT][3]>(empty + kStages);  // [2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t nrows = (int64_t)a.B * a.T;
  const int64_t rowbytes = (int64_t)a.V * (int64_t)sizeof(ET);
  const int nchunks = (int)((rowbytes + kChunk - 1) / kChunk);

  if (warp == kConsWarps) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
        if (!row_active<LOSS>(a, row, false)) continue;
#pragma unroll 1
        for (int k = 0; k < NT; ++k) {
          const char* src =
              reinterpret_cast<const char*>(a.logits[k]) + logits_off(a, k, row) * (int64_t)sizeof(ET);
          for (int c = 0; c < nchunks; ++c) {
            const int64_t rem = rowbytes - (int64_t)c * kChunk;
            const uint32_t bytes = (uint32_t)(rem < kChunk ? rem : kChunk);
            mbar_wait(&empty[stage], phase ^ 1u);
            mbar_arrive_expect_tx(&full[stage], bytes);
            bulk_g2s(ring + stage * kChunk, src + (int64_t)c * kChunk, bytes, &full[stage], pol);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int ctid = threadIdx.x;
  int stage = 0, buf = 0;
  uint32_t phase = 0;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    if (!row_active<LOSS>(a, row, ctid == 0)) {
      if (ctid == 0) write_inactive<LOSS>(a, row);
      continue;
    }
    int tok = 0;
    bool oov = false;
    float ztok[NT];
    if (ctid == 0) gather_token<ET, NT>(a, row, tok, oov, ztok);
    Acc acc[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      acc_init(acc[k]);
      for (int c = 0; c < nchunks; ++c) {
        const int64_t rem = rowbytes - (int64_t)c * kChunk;
        const int nvec = (int)((rem < kChunk ? rem : kChunk) / 16);
        mbar_wait(&full[stage], phase);
        const VV* sv = reinterpret_cast<const VV*>(ring + stage * kChunk);
        VV v[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
          const int idx = ctid + j * kCons;
          v[j] = idx < nvec ? sv[idx] : VT::fill();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);  // slice is in registers: release the stage early
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1u;
        }
        if (k == 0 && ENT0)
          VT::template accumulate<kPer, true, MATH | kMathGuard>(v, acc[k]);  // streamed: no redo, always guarded
        else
          VT::template accumulate<kPer, false, MATH>(v, acc[k]);
      }
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
    consumer_bar();
    if (warp == 0) row_finish<NT, kConsWarps, LOSS, ENT0>(a, red[buf], row, tok, oov, ztok, lane);
    buf ^= 1;
  }
}

template <int NT>
constexpr size_t smem_bytes() {
  return (size_t)kStages * kChunk + 2 * kStages * sizeof(uint64_t) + 2 * kConsWarps * NT * 3 * sizeof(float);
}

}  // namespace

bool tma_eligible(const VocabArgs& a, int esz) {
  if (((int64_t)a.V * esz) % 16 != 0) return false;
  for (int k = 0; k < a.ntens; ++k) {
    if ((reinterpret_cast<uintptr_t>(a.logits[k]) & 15u) != 0) return false;
    if ((a.stride[k] * esz) % 16 != 0) return false;
  }
  return true;
}

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH>
cudaError_t launch_tma(const VocabArgs& a, int num_sms, cudaStream_t s) {
  auto kern = vocab_tma_kernel<ET, NT, LOSS, ENT0, MATH>;
  constexpr size_t smem = smem_bytes<NT>();
  static bool configured = false;  // per instantiation; the attribute is per function
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int64_t nrows = (int64_t)a.B * a.T;
  const int grid = (int)(nrows < num_sms ? nrows : num_sms);
  kern<<<grid, kThreadsTma, smem, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

#define RLO_INST1(ET, NT, LOSS, ENT0, M) \
  template cudaError_t launch_tma<ET, NT, LOSS, ENT0, M>(const VocabArgs&, int, cudaStream_t);
#define RLO_INST_F(NT, LOSS, ENT0)         \
  RLO_INST1(float, NT, LOSS, ENT0, 0)     \
  RLO_INST1(float, NT, LOSS, ENT0, 1)     \
  RLO_INST1(float, NT, LOSS, ENT0, 1 | kMathLazy)
#define RLO_INST_B(NT, LOSS, ENT0)                 \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 1)     \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 2)     \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 3)     \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 4)     \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 5)     \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 6)     \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 6 | kMathLazy) \
  RLO_INST1(__nv_bfloat16, NT, LOSS, ENT0, 1 | kMathLazy)
RLO_INST_F(1, false, false)
RLO_INST_F(1, false, true)
RLO_INST_F(1, true, true)
RLO_INST_F(2, true, true)
RLO_INST_F(3, true, true)
RLO_INST_B(1, false, false)
RLO_INST_B(1, false, true)
RLO_INST_B(1, true, true)
RLO_INST_B(2, true, true)
RLO_INST_B(3, true, true)
#undef RLO_INST_F
#undef RLO_INST_B
#undef RLO_INST1

}  // namespace vocab
}  // namespace rlo
