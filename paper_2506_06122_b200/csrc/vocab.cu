// vocab.cu — the HBM-bound vocab pass (K1 forward_logprobs, K3 fused loss):
// launch dispatch + the 128-bit LDG streaming kernel.
//
// Replaces the reference's per-position log-softmax + gather
// (policy.cpp:116-122, :227; forward_logprobs :210-233) and the loss part of
// ppo_gradient (:355-374).  Two sm_100a implementations of one pass:
//   * vocab_ldg_kernel (here, default): persistent CTAs of 256 threads, U
//     128-bit ld.global.nc.L1::no_allocate loads in flight per thread;
//   * vocab_tma_kernel (vocab_tma.cu, RLO_VOCAB_IMPL=tma): one CTA per SM, a
//     producer warp streams 32 KB row chunks with cp.async.bulk into a
//     6-stage shared-memory ring (mbarrier full/empty), 16 consumer warps
//     reduce.  Measured 3-7% slower than LDG on B200 for both dtypes
//     (profiles/r1_vocab_sweep.txt), kept as the alternative producer.
// Both share the math and the epilogue (vocab_common.cuh); the softmax is
// never written.
#include <cstdlib>
#include <cstring>

#include "vocab_common.cuh"

namespace rlo {
namespace vocab {

// vocab_tma.cu
bool tma_eligible(const VocabArgs& a, int esz);
template <typename ET, int NT, bool LOSS, bool ENT0, int MATH>
cudaError_t launch_tma(const VocabArgs& a, int num_sms, cudaStream_t s);

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Build-time knob for A/B library builds (make EXTRA="-D..."):
// RLO_LDG_MIN_BLOCKS = __launch_bounds__ minimum CTAs per SM (register cap).
#ifndef RLO_LDG_MIN_BLOCKS
#define RLO_LDG_MIN_BLOCKS 4
#endif
// RLO_ENT_GUARD_ALWAYS = 1: the entropy row always runs the guarded math
// (no redo path).
#ifndef RLO_ENT_GUARD_ALWAYS
#define RLO_ENT_GUARD_ALWAYS 0
#endif

// Lockstep streams (LS): the NT tensors of a row are streamed together, U
// vectors of each per batch, and the old/ref states share the actor's running
// max instead of taking their own chunk maxima (saves the per-chunk max and
// rescale on NT-1 tensors — the bf16 pass is bound by SM power, so fewer
// instructions per byte buy clock).  An old/ref element more than ~2^126 above
// the actor's max would overflow its sum: such a thread's share (s non-finite
// or 0) is redone with the tensor's own max.  Rows must all be 16-byte
// aligned (else the sequential streams).
template <typename ET, int NT, int U, int MATH>
__device__ __forceinline__ void lockstep_accumulate(const ET* const (&rows)[NT], int V, Acc (&acc)[NT]) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  constexpr int kStep = kThreads * U;
  const int tid = threadIdx.x;
  const int nvec = V / VT::kElems;
  const int nfull = nvec / kStep * kStep;
  auto step = [&](const VV (&v)[NT][U]) {
    const float newmL = __fmul_rn(VT::template chunk_max<U>(v[0]), kL2E);
    if (newmL > acc[0].mL) {  // rescale every state to the new shared max
      const float d = acc[0].mL - newmL, sc = ex2(d);
      acc[0].w = (acc[0].w + acc[0].s * d) * sc;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        acc[k].s *= sc;
        acc[k].mL = newmL;
      }
    }
    VT::template accumulate<U, true, MATH | kMathNoMax>(v[0], acc[0]);
#pragma unroll
    for (int k = 1; k < NT; ++k) VT::template accumulate<U, false, MATH | kMathNoMax>(v[k], acc[k]);
  };
  for (int base = 0; base < nfull; base += kStep) {
    VV v[NT][U];
#pragma unroll
    for (int k = 0; k < NT; ++k)
#pragma unroll
      for (int u = 0; u < U; ++u) v[k][u] = ld_stream(reinterpret_cast<const VV*>(rows[k]) + base + u * kThreads + tid);
    step(v);
  }
  if (nfull < nvec) {
    VV v[NT][U];
#pragma unroll
    for (int k = 0; k < NT; ++k)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = nfull + u * kThreads + tid;
        v[k][u] = idx < nvec ? ld_stream(reinterpret_cast<const VV*>(rows[k]) + idx) : VT::fill();
      }
    step(v);
  }
#pragma unroll
  for (int k = 0; k < NT; ++k)
    for (int i = nvec * VT::kElems + tid; i < V; i += kThreads) {
      if (k == 0)
        acc_scalar<ET, true>(rows[k] + i, acc[k]);
      else
        acc_scalar<ET, false>(rows[k] + i, acc[k]);
    }
}

template <typename ET, int NT, int U, bool PF, bool LOSS, bool ENT0, int MATH, bool LS = false>
__global__ void __launch_bounds__(kThreads, RLO_LDG_MIN_BLOCKS) vocab_ldg_kernel(const VocabArgs a) {
  __shared__ float red[2][kWarps][NT][3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nrows = (int64_t)a.B * a.T;
  int buf = 0;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    if (!row_active<LOSS>(a, row, tid == 0)) {  // uniform across the CTA
      if (tid == 0) write_inactive<LOSS>(a, row);
      continue;
    }
    int tok = 0;
    bool oov = false;
    float ztok[NT];
    if (tid == 0) gather_token<ET, NT>(a, row, tok, oov, ztok);
    Acc acc[NT];
    if constexpr (LS && NT >= 2 && ENT0) {
      const ET* rows[NT];
      bool aligned = true;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        rows[k] = reinterpret_cast<const ET*>(a.logits[k]) + logits_off(a, k, row);
        aligned &= (reinterpret_cast<uintptr_t>(rows[k]) & 15u) == 0;
        acc_init(acc[k]);
      }
      if (__all_sync(0xffffffffu, aligned)) {  // aligned is uniform per row anyway
        lockstep_accumulate<ET, NT, U, MATH>(rows, a.V, acc);
        if (!(isfinite(acc[0].s) && isfinite(acc[0].w))) {  // -inf logits in the actor share: guarded redo
          acc_init(acc[0]);
          stream_accumulate<kThreads, ET, U, PF, true, MATH | kMathGuard>(rows[0], a.V, acc[0]);
        }
#pragma unroll
        for (int k = 1; k < NT; ++k)
          if (!(isfinite(acc[k].s) && acc[k].s > 0.f)) {  // above the shared max (or empty): own max
            acc_init(acc[k]);
            stream_accumulate<kThreads, ET, U, PF, false, MATH>(rows[k], a.V, acc[k]);
          }
        goto reduce;
      }
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      acc_init(acc[k]);
      const ET* rp = reinterpret_cast<const ET*>(a.logits[k]) + logits_off(a, k, row);
      if (k == 0 && ENT0) {
        if (RLO_ENT_GUARD_ALWAYS || sizeof(ET) == 4) {  // fp32 rows are memory-bound: one guarded body
          stream_accumulate<kThreads, ET, U, PF, true, MATH | kMathGuard>(rp, a.V, acc[k]);
        } else {
          stream_accumulate<kThreads, ET, U, PF, true, MATH>(rp, a.V, acc[k]);
          if (!(isfinite(acc[k].s) && isfinite(acc[k].w))) {
            // -inf logits in this thread's share: redo it guarded (the share
            // was just streamed, so the re-read mostly hits L2)
            acc_init(acc[k]);
            stream_accumulate<kThreads, ET, U, PF, true, MATH | kMathGuard>(rp, a.V, acc[k]);
          }
        }
      } else
        stream_accumulate<kThreads, ET, U, PF, false, MATH>(rp, a.V, acc[k]);
    }
  reduce:
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
    __syncthreads();  // double-buffered red[]: one barrier per row
    if (warp == 0) row_finish<NT, kWarps, LOSS, ENT0>(a, red[buf], row, tok, oov, ztok, lane);
    buf ^= 1;
  }
}

// Epilogue-warp variant (RLO_VOCAB_EPI=1): 7 streaming warps + 1 epilogue
// warp per 256-thread CTA.  The streaming warps hand each row's per-warp
// partials to the epilogue warp through named barriers (RED: partials ready;
// FREE: the double-buffered slot may be rewritten) and go straight on to the
// next row; the epilogue warp gathers the token logits, combines, and runs the
// fp64 loss epilogue.  In the default kernel the warp that runs row_finish
// reaches the next row's __syncthreads late and the other warps wait for it
// (ncu: ~11% of cfg2's warp samples at that barrier).
constexpr int kEpiStreamWarps = 7;
constexpr int kEpiStreamThreads = kEpiStreamWarps * 32;
template <int ID>
__device__ __forceinline__ void nb_arrive() { asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(kThreads) : "memory"); }
template <int ID>
__device__ __forceinline__ void nb_sync() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(kThreads) : "memory"); }

template <typename ET, int NT, int U, bool LOSS, bool ENT0, int MATH>
__global__ void __launch_bounds__(kThreads, RLO_LDG_MIN_BLOCKS) vocab_epi_kernel(const VocabArgs a) {
  __shared__ float red[2][kEpiStreamWarps][NT][3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool epi = warp == kEpiStreamWarps;
  const int64_t nrows = (int64_t)a.B * a.T;
  if (epi) {  // both slots start free
    nb_arrive<1>();
    nb_arrive<2>();
  }
  int buf = 0;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    if (!row_active<LOSS>(a, row, epi && lane == 0)) {  // uniform across the CTA
      if (epi && lane == 0) write_inactive<LOSS>(a, row);
      continue;
    }
    if (!epi) {
      Acc acc[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        acc_init(acc[k]);
        const ET* rp = reinterpret_cast<const ET*>(a.logits[k]) + logits_off(a, k, row);
        if (k == 0 && ENT0) {
          stream_accumulate<kEpiStreamThreads, ET, U, false, true, MATH>(rp, a.V, acc[k]);
          if (!(isfinite(acc[k].s) && isfinite(acc[k].w))) {  // -inf logits: guarded redo of this share
            acc_init(acc[k]);
            stream_accumulate<kEpiStreamThreads, ET, U, false, true, MATH | kMathGuard>(rp, a.V, acc[k]);
          }
        } else {
          stream_accumulate<kEpiStreamThreads, ET, U, false, false, MATH>(rp, a.V, acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (k == 0 && ENT0)
          acc_warp_reduce<true>(acc[k]);
        else
          acc_warp_reduce<false>(acc[k]);
      }
      if (buf) nb_sync<2>(); else nb_sync<1>();  // slot free (read by the epilogue two rows ago)
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          red[buf][warp][k][0] = acc[k].mL;
          red[buf][warp][k][1] = acc[k].s;
          red[buf][warp][k][2] = acc[k].w;
        }
      }
      if (buf) nb_arrive<4>(); else nb_arrive<3>();  // partials ready
    } else {
      int tok = 0;
      bool oov = false;
      float ztok[NT];
      if (lane == 0) gather_token<ET, NT>(a, row, tok, oov, ztok);
      if (buf) nb_sync<4>(); else nb_sync<3>();
      Acc c[NT];
      load_red<kEpiStreamWarps, NT>(red[buf], c, lane);
      __syncwarp();
      if (buf) nb_arrive<2>(); else nb_arrive<1>();  // slot read: free for row + 2
      row_finish_acc<NT, LOSS, ENT0>(a, c, row, tok, oov, ztok, lane);
    }
    buf ^= 1;
  }
  if (!epi) {  // consume the epilogue warp's last two FREE arrivals (barrier phases stay balanced)
    if (buf) nb_sync<2>(); else nb_sync<1>();
    if (buf) nb_sync<1>(); else nb_sync<2>();
  }
}

// Barrier-free variant (RLO_VOCAB_LF=1): the per-warp partials of a row go
// to one of kLfSlots shared-memory slots, each warp announces itself with an
// atomicAdd on the slot's arrival counter, and the LAST warp to arrive
// combines the row and runs the fp64 epilogue — nobody waits for it, and no
// warp waits at a per-row __syncthreads for the one that finished the
// previous row.  A slot is reused kLfSlots rows later; a writer spins (shared
// memory, same CTA) until the slot's previous finisher has read it, which it
// almost never has to.
constexpr int kLfSlots = 4;

template <typename ET, int NT, int U, bool LOSS, bool ENT0, int MATH>
__global__ void __launch_bounds__(kThreads, RLO_LDG_MIN_BLOCKS) vocab_lf_kernel(const VocabArgs a) {
  __shared__ float red[kLfSlots][kWarps][NT][3];
  __shared__ int arrivals[kLfSlots];
  __shared__ int done[kLfSlots];  // completed uses of the slot (rows finished from it)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t nrows = (int64_t)a.B * a.T;
  if (tid < kLfSlots) {
    arrivals[tid] = 0;
    done[tid] = 0;
  }
  __syncthreads();
  int j = 0;  // this CTA's active-row counter
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    if (!row_active<LOSS>(a, row, tid == 0)) {  // uniform across the CTA
      if (tid == 0) write_inactive<LOSS>(a, row);
      continue;
    }
    Acc acc[NT];
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      acc_init(acc[k]);
      const ET* rp = reinterpret_cast<const ET*>(a.logits[k]) + logits_off(a, k, row);
      if (k == 0 && ENT0) {
        stream_accumulate<kThreads, ET, U, false, true, MATH>(rp, a.V, acc[k]);
        if (!(isfinite(acc[k].s) && isfinite(acc[k].w))) {  // -inf logits: guarded redo of this share
          acc_init(acc[k]);
          stream_accumulate<kThreads, ET, U, false, true, MATH | kMathGuard>(rp, a.V, acc[k]);
        }
      } else {
        stream_accumulate<kThreads, ET, U, false, false, MATH>(rp, a.V, acc[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) {
      if (k == 0 && ENT0)
        acc_warp_reduce<true>(acc[k]);
      else
        acc_warp_reduce<false>(acc[k]);
    }
    const int slot = j % kLfSlots, use = j / kLfSlots;
    int last = 0;
    if (lane == 0) {
      while (*reinterpret_cast<volatile int*>(&done[slot]) < use) {
      }  // the slot's previous row has been read by its finisher
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        red[slot][warp][k][0] = acc[k].mL;
        red[slot][warp][k][1] = acc[k].s;
        red[slot][warp][k][2] = acc[k].w;
      }
      __threadfence_block();  // release the partials
      last = atomicAdd(&arrivals[slot], 1) == kWarps - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {  // the final arrival finishes the row
      __threadfence_block();  // acquire the other warps' partials
      int tok = 0;
      bool oov = false;
      float ztok[NT];
      if (lane == 0) gather_token<ET, NT>(a, row, tok, oov, ztok);
      Acc c[NT];
      load_red<kWarps, NT>(red[slot], c, lane);
      __syncwarp();
      if (lane == 0) {
        arrivals[slot] = 0;
        __threadfence_block();
        atomicAdd(&done[slot], 1);  // slot free for row j + kLfSlots
      }
      row_finish_acc<NT, LOSS, ENT0>(a, c, row, tok, oov, ztok, lane);
    }
    ++j;
  }
}

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH, int U>
cudaError_t launch_lf(const VocabArgs& a, int num_sms, cudaStream_t s) {
  auto kern = vocab_lf_kernel<ET, NT, U, LOSS, ENT0, MATH>;
  const int64_t nrows = (int64_t)a.B * a.T;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
  int64_t grid = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > nrows) grid = nrows;
  kern<<<(int)grid, kThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH, int U>
cudaError_t launch_epi(const VocabArgs& a, int num_sms, cudaStream_t s) {
  auto kern = vocab_epi_kernel<ET, NT, U, LOSS, ENT0, MATH>;
  const int64_t nrows = (int64_t)a.B * a.T;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
  int64_t grid = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > nrows) grid = nrows;
  kern<<<(int)grid, kThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH, int U, bool PF, bool LS = false>
cudaError_t launch_ldg(const VocabArgs& a, int num_sms, cudaStream_t s) {
  auto kern = vocab_ldg_kernel<ET, NT, U, PF, LOSS, ENT0, MATH, LS>;
  const int64_t nrows = (int64_t)a.B * a.T;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
  int64_t grid = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > nrows) grid = nrows;
  kern<<<(int)grid, kThreads, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Implementation / instruction-mix selection.  Defaults are the measured
// best per dtype (profiles/r1_vocab_sweep.txt); for
// experiments RLO_VOCAB_IMPL=ldg|tma, RLO_VOCAB_MATH (fp32 0-1, bf16 1-6),
// RLO_VOCAB_LDG (bf16 loss-pass layouts 1-4) and RLO_VOCAB_EPI=1 override them.
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

bool use_tma(int esz) {
  const char* e = std::getenv("RLO_VOCAB_IMPL");
  if (e && std::strcmp(e, "ldg") == 0) return false;
  if (e && std::strcmp(e, "tma") == 0) return true;
  (void)esz;
  return false;  // default: LDG streaming (measured faster than the TMA ring for fp32 and bf16, profiles/)
}

constexpr int kLongRowV = 65536;  // bf16 rows of >= 128 KB count as long

// LDG layout per dtype: fp32 U=8 (128 B in flight per thread); bf16 U=4
// (64 B).  RLO_VOCAB_LDG selects the alternatives compiled for the hot bf16
// fused-loss pass: 1 = U4 + prefetch, 2 = U8, 3 = U2 + prefetch.
template <typename ET, int NT, bool LOSS, bool ENT0, int MATH>
cudaError_t launch_ldg_layout(const VocabArgs& a, int num_sms, cudaStream_t s) {
  if constexpr (sizeof(ET) == 2 && (MATH & kMathLazy)) {
    // lazy max: software prefetch (U4 + the next batch in flight) measured +2% on cfg3
    const int l = env_int("RLO_VOCAB_LDG", 1);
    if (l == 1) return launch_ldg<ET, NT, LOSS, ENT0, MATH, 4, true>(a, num_sms, s);
    if (NT == 3 && LOSS && l == 2) return launch_ldg<ET, NT, LOSS, ENT0, MATH, 8, false>(a, num_sms, s);
  } else if constexpr (sizeof(ET) == 2 && NT == 3 && LOSS) {
    switch (env_int("RLO_VOCAB_LDG", a.V < kLongRowV ? 4 : 0)) {  // short rows: lockstep streams
      case 1: return launch_ldg<ET, NT, LOSS, ENT0, MATH, 4, true>(a, num_sms, s);
      case 2: return launch_ldg<ET, NT, LOSS, ENT0, MATH, 8, false>(a, num_sms, s);
      case 3: return launch_ldg<ET, NT, LOSS, ENT0, MATH, 2, true>(a, num_sms, s);
      case 4: return launch_ldg<ET, NT, LOSS, ENT0, MATH, 2, false, true>(a, num_sms, s);  // lockstep, U2 per tensor
      default: break;
    }
  }
  return launch_ldg<ET, NT, LOSS, ENT0, MATH, sizeof(ET) == 4 ? 8 : 4, false>(a, num_sms, s);
}

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH>
cudaError_t launch_impl(const VocabArgs& a, int num_sms, cudaStream_t s) {
  if (use_tma((int)sizeof(ET)) && tma_eligible(a, (int)sizeof(ET)))
    return launch_tma<ET, NT, LOSS, ENT0, MATH>(a, num_sms, s);
  if (env_int("RLO_VOCAB_EPI", 0)) return launch_epi<ET, NT, LOSS, ENT0, MATH, sizeof(ET) == 4 ? 8 : 4>(a, num_sms, s);
  if (env_int("RLO_VOCAB_LF", 0)) return launch_lf<ET, NT, LOSS, ENT0, MATH, sizeof(ET) == 4 ? 8 : 4>(a, num_sms, s);
  return launch_ldg_layout<ET, NT, LOSS, ENT0, MATH>(a, num_sms, s);
}

// Instruction mix (vocab_common.cuh): fp32 {0, 1, 2 = 1 + lazy max}, default 1; bf16 {1..6, 7 = 6 + lazy
// max, 8 = 1 + lazy max}, default 7 with the U4 + prefetch layout (profiles/r1_vocab_sweep.txt).
template <typename ET, int NT, bool LOSS, bool ENT0>
cudaError_t launch_any(const VocabArgs& a, int num_sms, cudaStream_t s) {
  if ((int64_t)a.B * a.T == 0) return cudaSuccess;
  // bf16: the lazy max + prefetch (mix 7), except the 3-tensor loss pass over
  // short rows (< 128 KB), which takes mix 6 with lockstep streams (per-row
  // cold starts dominate there; profiles/r1_vocab_sweep.txt)
  const bool short3 = NT == 3 && LOSS && a.V < kLongRowV;
  const int math = env_int("RLO_VOCAB_MATH", sizeof(ET) == 2 ? (short3 ? 6 : 7) : 1);
  if constexpr (sizeof(ET) == 4) {
    return math == 0   ? launch_impl<ET, NT, LOSS, ENT0, 0>(a, num_sms, s)
           : math == 2 ? launch_impl<ET, NT, LOSS, ENT0, 1 | kMathLazy>(a, num_sms, s)
                       : launch_impl<ET, NT, LOSS, ENT0, 1>(a, num_sms, s);
  } else {
    switch (math) {
      case 1: return launch_impl<ET, NT, LOSS, ENT0, 1>(a, num_sms, s);
      case 3: return launch_impl<ET, NT, LOSS, ENT0, 3>(a, num_sms, s);
      case 4: return launch_impl<ET, NT, LOSS, ENT0, 4>(a, num_sms, s);
      case 5: return launch_impl<ET, NT, LOSS, ENT0, 5>(a, num_sms, s);
      case 6: return launch_impl<ET, NT, LOSS, ENT0, 6>(a, num_sms, s);
      case 7: return launch_impl<ET, NT, LOSS, ENT0, 6 | kMathLazy>(a, num_sms, s);
      case 8: return launch_impl<ET, NT, LOSS, ENT0, 1 | kMathLazy>(a, num_sms, s);
      default: return launch_impl<ET, NT, LOSS, ENT0, 2>(a, num_sms, s);
    }
  }
}

template <typename ET>
cudaError_t launch_loss_dtype(const VocabArgs& a, int num_sms, cudaStream_t s) {
  switch (a.ntens) {
    case 1: return launch_any<ET, 1, true, true>(a, num_sms, s);
    case 2: return launch_any<ET, 2, true, true>(a, num_sms, s);
    default: return launch_any<ET, 3, true, true>(a, num_sms, s);
  }
}

}  // namespace
}  // namespace vocab

cudaError_t launch_vocab_logprob(const VocabArgs& a, int num_sms, cudaStream_t s) {
  using namespace vocab;
  const bool ent = a.out_ent != nullptr;
  if (a.dtype == RLO_DTYPE_BF16)
    return ent ? launch_any<__nv_bfloat16, 1, false, true>(a, num_sms, s)
               : launch_any<__nv_bfloat16, 1, false, false>(a, num_sms, s);
  return ent ? launch_any<float, 1, false, true>(a, num_sms, s) : launch_any<float, 1, false, false>(a, num_sms, s);
}

cudaError_t launch_vocab_loss(const VocabArgs& a, int num_sms, cudaStream_t s) {
  return a.dtype == RLO_DTYPE_BF16 ? vocab::launch_loss_dtype<__nv_bfloat16>(a, num_sms, s)
                                   : vocab::launch_loss_dtype<float>(a, num_sms, s);
}

}  // namespace rlo
