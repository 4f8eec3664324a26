// vocab.cu — the HBM-bound vocab pass (K1 forward_logprobs, K3 fused loss):
// launch dispatch + the 128-bit LDG streaming kernel.
//
// Replaces the reference's per-position log-softmax + gather
// (policy.cpp:116-122, :227; forward_logprobs :210-233) and the loss part of
// ppo_gradient (:355-374).  One sm_100a kernel template: persistent CTAs
// streaming rows with U 128-bit ld.global.nc.L1::no_allocate loads in flight
// per thread -- one warp per row for bf16 (32-thread CTAs, the row finished
// inside the warp), 256 threads per row for fp32; the math and the epilogue
// live in vocab_common.cuh; the softmax is never written.
//
// The library ships exactly one instantiation per (dtype, tensors, mode,
// entropy) — the measured defaults (profiles/r1_vocab_sweep.txt);
// every one of them is exercised by a -m gpu oracle test.  The losing
// producers of round 1 (TMA bulk-copy ring, epilogue warp, last-finisher
// hand-off) live only in the git history; the instruction mix and layout are
// compile-time (A/B builds: make EXTRA="-DRLO_BF16_MATH=... -DRLO_BF16_U=...").

#include "vocab_common.cuh"

namespace rlo {
namespace vocab {

namespace {

// CTA size per dtype (compile-time): bf16 rows are streamed by
// ONE warp per row (CTAs of 32 threads: no cross-warp reduction, no barrier),
// fp32 rows by 256-thread CTAs (the 2/3-tensor fp32 passes read 3-5% less
// with 32-128-thread CTAs, profiles/r2_vocab_ab.txt calls ag, am).
#ifndef RLO_F32_THREADS
#define RLO_F32_THREADS 256
#endif
#ifndef RLO_F32_THREADS_1T  // fp32 1-tensor passes (P = 1 loss, forward_logprobs): +2.8% at 128 (call an)
#define RLO_F32_THREADS_1T 128
#endif
#ifndef RLO_BF16_THREADS
#define RLO_BF16_THREADS 32
#endif
// Build-time knob for A/B library builds (make EXTRA="-D..."):
// RLO_LDG_THREADS_PER_SM = resident threads per SM the register cap of
// __launch_bounds__ is sized for (1024: 64 registers).
#ifndef RLO_LDG_THREADS_PER_SM
#define RLO_LDG_THREADS_PER_SM 1024
#endif
// The bf16 lockstep kernel (P >= 2): 768 resident threads per SM (24 rows in
// flight per SM, 80 registers, no spills): +2.1% on cfg3 against 1024 (the
// 1-tensor pass and the fp32 passes lose at 768 and keep 1024;
// profiles/r2_vocab_ab.txt calls ap-at).
#ifndef RLO_BF16_LS_THREADS_PER_SM
#define RLO_BF16_LS_THREADS_PER_SM 768
#endif
#ifndef RLO_BF16_PAIR_THREADS_PER_SM
#define RLO_BF16_PAIR_THREADS_PER_SM 768
#endif
// RLO_ENT_GUARD_ALWAYS = 1: the entropy row always runs the guarded math
// (no redo path).
#ifndef RLO_ENT_GUARD_ALWAYS
#define RLO_ENT_GUARD_ALWAYS 0
#endif

// Lockstep streams (LS): the NT tensors of a row are streamed together, U
// vectors of each per batch, and the old/ref states share the actor's running
// max instead of taking their own chunk maxima (saves the per-chunk max and
// rescale on NT-1 tensors; one cold start per row).  A thread's old/ref share whose sum on the
// shared max leaves [2^-80, 2^100) — an element far above the actor's max, or
// a tensor so far below it that flushed terms matter — is redone with the
// tensor's own max (the kernel below).  Rows must all be 16-byte aligned
// (else the sequential streams).
// DEF (deferred offset; the shipped layout): the shared offset is the
// actor max of the thread's first batch only; later batches take no max, test
// or rescale at all -- the kernel's range checks on the finished shares redo
// any share that left the safe range.
// Thread tid's share is the vectors base + u * NTH + tid -- the layout of
// stream_accumulate with the same U, so a redo covers exactly the share it
// replaces (a 256-bit pair layout here would break that; it also read 0.6%
// fewer bytes, profiles/r2_vocab_ab.txt call t).
template <int NTH, typename ET, int NT, int U, int MATH, bool DEF = false>
__device__ __forceinline__ void lockstep_accumulate(const ET* const (&rows)[NT], int V, Acc (&acc)[NT]) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  constexpr int kStep = NTH * U;
  const int tid = threadIdx.x;
  const int nvec = V / VT::kElems;
  const int nfull = nvec / kStep * kStep;
  auto step = [&](const VV (&v)[NT][U]) {
    if (DEF && acc[0].mL > kLazyMin) {
      VT::template accumulate<U, true, MATH | kMathNoMax>(v[0], acc[0]);
#pragma unroll
      for (int k = 1; k < NT; ++k) VT::template accumulate<U, false, MATH | kMathNoMax>(v[k], acc[k]);
      return;
    }
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
      for (int u = 0; u < U; ++u) v[k][u] = ld_stream(reinterpret_cast<const VV*>(rows[k]) + base + u * NTH + tid);
    step(v);
  }
  if (nfull < nvec) {
    VV v[NT][U];
#pragma unroll
    for (int k = 0; k < NT; ++k)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = nfull + u * NTH + tid;
        v[k][u] = idx < nvec ? ld_stream(reinterpret_cast<const VV*>(rows[k]) + idx) : VT::fill();
      }
    step(v);
  }
#pragma unroll
  for (int k = 0; k < NT; ++k)
    for (int i = nvec * VT::kElems + tid; i < V; i += NTH) {
      if (k == 0)
        acc_scalar<ET, true>(rows[k] + i, acc[k]);
      else
        acc_scalar<ET, false>(rows[k] + i, acc[k]);
    }
}

// U / PF: the layout of the entropy (actor) row; UN / PFN: the layout of the
// other rows (old / ref, or the rows of a pass without entropy).
// NTH: threads per CTA (one row per CTA at a time); NTH = 32 finishes each
// row inside the warp (no shared-memory reduction, no barrier).
template <int NTH, typename ET, int NT, int U, bool PF, bool LOSS, bool ENT0, int MATH, bool LS = false, int UN = U,
          bool PFN = PF>
__global__ void __launch_bounds__(NTH, (LS && sizeof(ET) == 2 ? RLO_BF16_LS_THREADS_PER_SM : RLO_LDG_THREADS_PER_SM) / NTH)
    vocab_ldg_kernel(const VocabArgs a) {
  constexpr int kWarps = NTH / 32;
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
        lockstep_accumulate<NTH, ET, NT, U, MATH & kMathMask, (MATH & kMathDeferred) != 0>(rows, a.V, acc);
        // Redo the actor share exactly (and guarded) on -inf logits (w = 0 * -inf)
        // or, under the deferred offset, when the share's max sat so far above
        // the offset (s >= 2^32, as the lazy max's cap) that the entropy's
        // log2 s - w/s would cancel too many bits.
        if (!(isfinite(acc[0].s) && isfinite(acc[0].w)) || ((MATH & kMathDeferred) && !(acc[0].s < kLazyCap))) {
          acc_init(acc[0]);
          stream_accumulate<NTH, ET, U, PF, true, MATH | kMathGuard>(rows[0], a.V, acc[0]);
        }
#pragma unroll
        for (int k = 1; k < NT; ++k)
          // Redo the share with the tensor's own max unless its sum sits safely
          // inside fp32 on the shared max: >= 2^100 means an element far above
          // the actor's max (MUFU lanes overflow to inf, polynomial lanes clamp
          // at 2^127), < 2^-80 means the share sits so far below it that
          // ex2.approx.ftz flushed part of its mass to zero; NaN fails both.
          if (!(acc[k].s >= 0x1p-80f && acc[k].s < 0x1p100f)) {
            acc_init(acc[k]);
            stream_accumulate<NTH, ET, UN, PFN, false, MATH>(rows[k], a.V, acc[k]);
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
          stream_accumulate<NTH, ET, U, PF, true, MATH | kMathGuard>(rp, a.V, acc[k]);
        } else if constexpr ((MATH & kMathDeferred) != 0) {
          stream_checked<NTH, ET, U, PF, true, MATH>(rp, a.V, acc[k]);
        } else {
          stream_accumulate<NTH, ET, U, PF, true, MATH>(rp, a.V, acc[k]);
          if (!(isfinite(acc[k].s) && isfinite(acc[k].w))) {
            // -inf logits in this thread's share: redo it guarded (the share
            // was just streamed, so the re-read mostly hits L2)
            acc_init(acc[k]);
            stream_accumulate<NTH, ET, U, PF, true, MATH | kMathGuard>(rp, a.V, acc[k]);
          }
        }
      } else if constexpr ((MATH & kMathDeferred) != 0) {
        stream_checked<NTH, ET, UN, PFN, false, MATH>(rp, a.V, acc[k]);
      } else {
        stream_accumulate<NTH, ET, UN, PFN, false, MATH>(rp, a.V, acc[k]);
      }
    }
  reduce:
    if constexpr (kWarps == 1) {  // the row's warp combines its lanes and finishes
      row_finish_acc<NT, LOSS, ENT0>(a, acc, row, tok, oov, ztok, lane);
      continue;
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
    __syncthreads();  // double-buffered red[]: one barrier per row
    if (warp == 0) row_finish<NT, kWarps, LOSS, ENT0>(a, red[buf], row, tok, oov, ztok, lane);
    buf ^= 1;
  }
}

// The bf16 1-tensor passes (the P = 1 loss pass: old / ref log-probs
// precomputed; forward_logprobs, +4%, call az): TWO rows per warp in lockstep (consecutive tokens), U = 5 vectors of each per
// batch, each row on its own deferred offset (the max of its first batch),
// 768 resident threads per SM: +2.9% over the lazy-max stream with prefetch
// (profiles/r2_vocab_ab.txt calls ax-ay).  A row whose share leaves the safe
// range (non-finite, or s >= 2^32: the entropy's cancellation) is redone
// exactly and guarded; a pair with an inactive or misaligned row streams its
// rows one by one (the lazy-max stream).
template <typename ET, int U, int MATH, bool ENT>
__device__ __forceinline__ void pair_accumulate(const ET* const (&rows)[2], int V, Acc (&acc)[2]) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  constexpr int kStep = 32 * U;
  const int lane = threadIdx.x & 31;
  const int nvec = V / VT::kElems;
  const int nfull = nvec / kStep * kStep;
  auto step = [&](const VV (&v)[2][U]) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (acc[k].mL > kLazyMin)
        VT::template accumulate<U, ENT, MATH | kMathNoMax>(v[k], acc[k]);
      else
        VT::template accumulate<U, ENT, MATH>(v[k], acc[k]);
    }
  };
  for (int base = 0; base < nfull; base += kStep) {
    VV v[2][U];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int u = 0; u < U; ++u) v[k][u] = ld_stream(reinterpret_cast<const VV*>(rows[k]) + base + u * 32 + lane);
    step(v);
  }
  if (nfull < nvec) {
    VV v[2][U];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int idx = nfull + u * 32 + lane;
        v[k][u] = idx < nvec ? ld_stream(reinterpret_cast<const VV*>(rows[k]) + idx) : VT::fill();
      }
    step(v);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k)
    for (int i = nvec * VT::kElems + lane; i < V; i += 32) acc_scalar<ET, ENT>(rows[k] + i, acc[k]);
}

// MATHS / US / PFS: the single-row stream (lazy max) for a pair with an
// inactive or misaligned row.
// LOSS / ENT0: the loss pass (P = 1) or forward_logprobs, with or without
// the entropy (a row without entropy takes the polynomial lanes of MATH and
// is redone when its share leaves [.., 2^100) on its own offset).
template <typename ET, int U, int MATH, int MATHS, int US, bool PFS, bool LOSS, bool ENT0>
__global__ void __launch_bounds__(32, RLO_BF16_PAIR_THREADS_PER_SM / 32) vocab_pair_kernel(const VocabArgs a) {
  const int lane = threadIdx.x;
  const int64_t nrows = (int64_t)a.B * a.T, npairs = (nrows + 1) / 2;
  for (int64_t pr = blockIdx.x; pr < npairs; pr += gridDim.x) {
    const int64_t r[2] = {2 * pr, 2 * pr + 1};
    bool act[2];
    int tok[2] = {0, 0};
    bool oov[2] = {false, false};
    float ztok[2][1];
    const ET* rp[2];
    Acc acc[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      act[k] = r[k] < nrows && row_active<LOSS>(a, r[k], lane == 0);
      if (r[k] < nrows && !act[k] && lane == 0) write_inactive<LOSS>(a, r[k]);
      if (act[k] && lane == 0) gather_token<ET, 1>(a, r[k], tok[k], oov[k], ztok[k]);
      rp[k] = reinterpret_cast<const ET*>(a.logits[0]) + (r[k] < nrows ? logits_off(a, 0, r[k]) : 0);
      acc_init(acc[k]);
    }
    const bool aligned = ((reinterpret_cast<uintptr_t>(rp[0]) | reinterpret_cast<uintptr_t>(rp[1])) & 15u) == 0;
    if (act[0] && act[1] && aligned) {
      pair_accumulate<ET, U, MATH, ENT0>(rp, a.V, acc);
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (ENT0 ? (!(isfinite(acc[k].s) && isfinite(acc[k].w)) || !(acc[k].s < kLazyCap)) : !(acc[k].s < kDeferCap)) {
          acc_init(acc[k]);
          stream_accumulate<32, ET, U, false, ENT0, MATH | (ENT0 ? kMathGuard : 0)>(rp[k], a.V, acc[k]);
        }
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k)
        if (act[k]) {
          stream_accumulate<32, ET, US, PFS, ENT0, MATHS>(rp[k], a.V, acc[k]);
          if (ENT0 && !(isfinite(acc[k].s) && isfinite(acc[k].w))) {  // -inf logits: guarded redo
            acc_init(acc[k]);
            stream_accumulate<32, ET, US, PFS, ENT0, MATHS | kMathGuard>(rp[k], a.V, acc[k]);
          }
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (act[k]) {
        Acc c[1] = {acc[k]};
        row_finish_acc<1, LOSS, ENT0>(a, c, r[k], tok[k], oov[k], ztok[k], lane);
      }
  }
}

template <typename ET, int U, int MATH, int MATHS, int US, bool PFS, bool LOSS, bool ENT0>
cudaError_t launch_pair(const VocabArgs& a, int num_sms, cudaStream_t s) {
  auto kern = vocab_pair_kernel<ET, U, MATH, MATHS, US, PFS, LOSS, ENT0>;
  const int64_t npairs = ((int64_t)a.B * a.T + 1) / 2;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32, 0);
  int64_t grid = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > npairs) grid = npairs;
  kern<<<(int)grid, 32, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <typename ET, int NT, bool LOSS, bool ENT0, int MATH, int U, bool PF, bool LS = false, int UN = U,
          bool PFN = PF>
cudaError_t launch_ldg(const VocabArgs& a, int num_sms, cudaStream_t s) {
  constexpr int NTH = sizeof(ET) == 4 ? (NT == 1 ? RLO_F32_THREADS_1T : RLO_F32_THREADS) : RLO_BF16_THREADS;
  auto kern = vocab_ldg_kernel<NTH, ET, NT, U, PF, LOSS, ENT0, MATH, LS, UN, PFN>;
  const int64_t nrows = (int64_t)a.B * a.T;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTH, 0);
  int64_t grid = (int64_t)num_sms * (per_sm < 1 ? 1 : per_sm);
  if (grid > nrows) grid = nrows;
  kern<<<(int)grid, NTH, 0, s>>>(a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Compile-time defaults per dtype (A/B builds override them):
//  fp32: mix 1 (packed FFMA2/FADD2, MUFU.EX2), U = 8 (128 B in flight per
//        thread), entropy row always guarded (memory-bound: one body);
//  bf16 loss pass with 2 or 3 logits tensors (cfg 3-5 and every bf16
//        P >= 2 row): the tensors of a token streamed in lockstep, U = 3
//        vectors of each per batch, one warp per row, on a deferred offset
//        (the actor max of the lane's first batch; no per-batch max, test or
//        rescale), mix 6 (degree-4 FMA-pipe exp2 on 1 of 4 old/ref element
//        pairs, the entropy row all MUFU): +3-4% over per-tensor lazy-max
//        streams on Qwen rows, +7% over the round-2 short-row lockstep
//        (shared running max, U = 2) on V = 32000 rows (profiles/r2_vocab_ab.txt);
//  bf16 P = 1 loss pass and forward_logprobs: two rows per warp in lockstep
//        (vocab_pair_kernel); a pair with an inactive or misaligned row
//        streams them one by one: mix 7 = mix 6 + the lazy running max, U = 4
//        with the next batch in flight (software prefetch).
#ifndef RLO_F32_MATH
#define RLO_F32_MATH 1
#endif
#ifndef RLO_BF16_MATH
#define RLO_BF16_MATH (6 | kMathLazy)
#endif
#ifndef RLO_BF16_U
#define RLO_BF16_U 4
#endif
#ifndef RLO_BF16_PF
#define RLO_BF16_PF true
#endif
#ifndef RLO_BF16_UN
#define RLO_BF16_UN RLO_BF16_U
#endif
#ifndef RLO_BF16_PFN
#define RLO_BF16_PFN RLO_BF16_PF
#endif
#ifndef RLO_BF16_MATH_P1
#define RLO_BF16_MATH_P1 RLO_BF16_MATH
#endif
#ifndef RLO_BF16_LS_U  // lockstep vectors per tensor per batch (0: per-tensor lazy streams, A/B)
#define RLO_BF16_LS_U 3
#endif
#ifndef RLO_BF16_PAIR_FWD  // forward_logprobs through the pair kernel too: +4% (call az)
#define RLO_BF16_PAIR_FWD 1
#endif
#ifndef RLO_BF16_PAIR_U  // 0: the lazy-max stream (A/B)
#define RLO_BF16_PAIR_U 5
#endif
#ifndef RLO_BF16_LS_MATH
#define RLO_BF16_LS_MATH 6
#endif

template <typename ET, int NT, bool LOSS, bool ENT0>
cudaError_t launch_any(const VocabArgs& a, int num_sms, cudaStream_t s) {
  if ((int64_t)a.B * a.T == 0) return cudaSuccess;
  if constexpr (sizeof(ET) == 4) {
    return launch_ldg<ET, NT, LOSS, ENT0, RLO_F32_MATH, 8, false>(a, num_sms, s);
  } else if constexpr (NT >= 2 && LOSS && RLO_BF16_LS_U != 0) {  // lockstep on a deferred offset
    return launch_ldg<ET, NT, LOSS, ENT0, RLO_BF16_LS_MATH | kMathDeferred, RLO_BF16_LS_U, false, true>(a, num_sms, s);
  } else if constexpr (NT == 1 && RLO_BF16_PAIR_U > 0 && (LOSS || RLO_BF16_PAIR_FWD)) {  // two rows per warp
    return launch_pair<ET, RLO_BF16_PAIR_U, 6, RLO_BF16_MATH, RLO_BF16_U, RLO_BF16_PF, LOSS, ENT0>(a, num_sms, s);
  } else {
    if constexpr (NT == 1 && LOSS && ENT0 && RLO_BF16_MATH_P1 != RLO_BF16_MATH)  // A/B: actor-only loss pass
      return launch_ldg<ET, NT, LOSS, ENT0, RLO_BF16_MATH_P1, RLO_BF16_U, RLO_BF16_PF>(a, num_sms, s);
    return launch_ldg<ET, NT, LOSS, ENT0, RLO_BF16_MATH, RLO_BF16_U, RLO_BF16_PF, false, RLO_BF16_UN, RLO_BF16_PFN>(
        a, num_sms, s);
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
