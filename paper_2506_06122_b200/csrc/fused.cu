// fused.cu — the fused actor update pass: the loss part of ppo_gradient
// (policy.cpp:355-374, a1-a9) and the actor backward epilogue
// dlogits = w * dlogp * (onehot - softmax) (policy.cpp:375-379) in ONE read
// of the actor logits.
//
// A thread-block cluster of K CTAs owns one row at a time.  CTA r streams the
// slice [r*S, r*S + S) of the actor row with 128-bit LDG and keeps it in its
// shared memory in a thread-private layout (vector j lives with thread
// j mod 256, so no intra-CTA hazards), and streams the same slice of the
// old-policy / reference rows without keeping them.  The K partial (mL, s, w)
// states meet over DSMEM: one cluster barrier per row, double-buffered slots.
// Every CTA combines the K partials in the same order (so all of them hold the
// identical lse), runs the fp64 loss epilogue (the leader CTA writes the
// per-token outputs and reduction scratch), and writes its gradient slice
// straight from shared memory:
//     g_v = -(w*dlp / s) * 2^(z_v*log2e - mL)   (+ w*dlp at the realised token)
// where (mL, s) is the row's online state, so the softmax is neither stored
// nor rebuilt from a rounded fp32 lse.
//
// HBM bytes per participating row: P*V*s_in + V*s_out, against
// (P+1)*V*s_in + V*s_out for rlo_ppo_gradient followed by rlo_logits_backward.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "grad_io.cuh"
#include "vocab_common.cuh"

namespace cg = cooperative_groups;

namespace rlo {
namespace vocab {
namespace {

// A/B build knob: software prefetch in the old/ref streams (make EXTRA=-DRLO_FUSED_PF=1).
#ifndef RLO_FUSED_PF
#define RLO_FUSED_PF 0
#endif
// The entropy row always guarded in the fused pass (no redo path): the fused
// pass runs fp32 rows, which are memory-bound, and the smaller kernel measured
// 0.6% faster (profiles/r1_fused.txt).  0 = unguarded + guarded redo.
#ifndef RLO_FUSED_GUARD_ALWAYS
#define RLO_FUSED_GUARD_ALWAYS 1
#endif

constexpr int kFT = 256;
constexpr int kFW = kFT / 32;

struct FusedArgs {
  VocabArgs v;
  const float* weight;
  void* grad;
  int64_t gstride;
  int32_t slice;  // elements per CTA slice (a multiple of the 16-byte vector width)
};

// This CTA's actor slice (n elements at src, 16-byte aligned).  LOAD: stream it
// from HBM with U 128-bit loads in flight per thread and keep each vector in
// shared memory; !LOAD: run the accumulation from shared memory.  The
// sub-vector tail (last slice only) is read from global memory.
template <typename ET, int U, int MATHG, bool LOAD>
__device__ __forceinline__ void slice_pass(const ET* __restrict__ src, int n, typename Vec<ET>::V* sm, Acc& a) {
  using VT = Vec<ET>;
  using VV = typename VT::V;
  constexpr int kStep = kFT * U;
  const int tid = threadIdx.x;
  const int nvec = n / VT::kElems;
  const int nfull = nvec / kStep * kStep;
  const VV* __restrict__ vsrc = reinterpret_cast<const VV*>(src);
  for (int base = 0; base < nfull; base += kStep) {
    VV v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = LOAD ? ld_stream(vsrc + base + u * kFT + tid) : sm[base + u * kFT + tid];
    if (LOAD) {
#pragma unroll
      for (int u = 0; u < U; ++u) sm[base + u * kFT + tid] = v[u];
    }
    VT::template accumulate<U, true, MATHG>(v, a);
  }
  if (nfull < nvec) {
    VV v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int idx = nfull + u * kFT + tid;
      v[u] = idx < nvec ? (LOAD ? ld_stream(vsrc + idx) : sm[idx]) : VT::fill();
      if (LOAD && idx < nvec) sm[idx] = v[u];
    }
    VT::template accumulate<U, true, MATHG>(v, a);
  }
  for (int i = nvec * VT::kElems + tid; i < n; i += kFT) {
    const float z = VT::scalar(src + i);
    acc_rescale<true>(a, z);
    float w = 0.f, s = 0.f;
    acc_elem<true>(z, a.mL, s, w);
    a.s += s;
    a.w += w;
  }
}

template <typename ET>
__device__ __forceinline__ void unpack(const typename Vec<ET>::V& v, float (&x)[8]);
template <>
__device__ __forceinline__ void unpack<float>(const float4& v, float (&x)[8]) {
  x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& v, float (&x)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) x[2 * k] = bf16lo(w[k]), x[2 * k + 1] = bf16hi(w[k]);
}

// Gradient slice from shared memory: g = c * 2^(z*log2e - mL) (+ scale at the
// token, tok_rel relative to the slice start).  scale == 0 writes zeros.
template <typename ET, typename GT>
__device__ __forceinline__ void slice_grad(const ET* __restrict__ src, int n, const typename Vec<ET>::V* sm,
                                           GT* __restrict__ g, float mL, float c, int tok_rel, float scale) {
  constexpr int E = Vec<ET>::kElems;
  const int nvec = n / E;
  if (scale == 0.f) {
    float zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = threadIdx.x; j < nvec; j += kFT) Out<GT>::template store<E>(g + (int64_t)j * E, zero);
    for (int i = nvec * E + threadIdx.x; i < n; i += kFT) Out<GT>::one(g + i, 0.f);
    return;
  }
  for (int j = threadIdx.x; j < nvec; j += kFT) {  // exactly the vectors this thread stored
    float x[8], o[8];
    unpack<ET>(sm[j], x);
#pragma unroll
    for (int k = 0; k < E; ++k) o[k] = c * ex2(fmaf(x[k], kL2E, -mL));
    const int d = tok_rel - j * E;
    if (d >= 0 && d < E) {
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (k == d) o[k] += scale;
    }
    Out<GT>::template store<E>(g + (int64_t)j * E, o);
  }
  for (int i = nvec * E + threadIdx.x; i < n; i += kFT) {
    float o = c * ex2(fmaf(Vec<ET>::scalar(src + i), kL2E, -mL));
    if (i == tok_rel) o += scale;
    Out<GT>::one(g + i, o);
  }
}

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

constexpr int kEpiWarp = kFW;               // warp 8: the epilogue warp
constexpr int kFTotal = kFT + 32;           // 8 streaming warps + the epilogue warp

// Named barriers (ids 1-4; 0 is __syncthreads), by iteration parity: RED =
// "per-warp partials of row i are in red[i&1]" (streaming warps arrive, the
// epilogue warp syncs); BC = "the epilogue of row i is in bc[i&1]" (the
// epilogue warp arrives, the streaming warps sync).
template <int ID>
__device__ __forceinline__ void bar_arrive_id() { asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(kFTotal) : "memory"); }
template <int ID>
__device__ __forceinline__ void bar_sync_id() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(kFTotal) : "memory"); }
// RED slot s uses barrier 1 + s, BC slot s uses 1 + NB + s (NB <= 3 slots)
// immediate barrier ids (a register id makes ptxas reserve all 16)
__device__ __forceinline__ void bar_arrive(int id) {
  switch (id) {
    case 1: bar_arrive_id<1>(); break;
    case 2: bar_arrive_id<2>(); break;
    case 3: bar_arrive_id<3>(); break;
    case 4: bar_arrive_id<4>(); break;
    case 5: bar_arrive_id<5>(); break;
    default: bar_arrive_id<6>(); break;
  }
}
__device__ __forceinline__ void bar_sync(int id) {
  switch (id) {
    case 1: bar_sync_id<1>(); break;
    case 2: bar_sync_id<2>(); break;
    case 3: bar_sync_id<3>(); break;
    case 4: bar_sync_id<4>(); break;
    case 5: bar_sync_id<5>(); break;
    default: bar_sync_id<6>(); break;
  }
}

// Warp-specialised and software-pipelined over the cluster's rows.
// Streaming warps 0-7, iteration i: stream row i (the actor slice into
// shared-memory buffer i&1), deposit per-warp partials (arrive RED), move
// through the cluster barrier (wait for phase i-1, arrive for phase i), then
// take row i-1's epilogue (sync BC) and write its gradient from buffer
// (i-1)&1.  The epilogue warp, iteration i: gather row i's token logits, take
// the partials (sync RED), publish the CTA partial part[i&1] over DSMEM,
// arrive + wait at the cluster barrier, combine the K partials in rank order,
// run the fp64 epilogue into bc[i&1] (arrive BC).  The streaming warps never
// wait on the epilogue of the row they just streamed, and wait for the
// cluster only one phase late, so a slower peer or a long epilogue costs
// nothing unless it falls a whole row behind.  Hazards: red, bc and the actor
// slices are double-buffered by parity and each is rewritten two iterations
// later, after the consumer's next hand-off; part[i&1] is rewritten in
// iteration i+2 only after every peer's epilogue warp has arrived for phase
// i+1, i.e. after it read phase i's slots.  Only the epilogue warp writes
// part, so only it arrives with release semantics.
template <typename ET, typename GT, int NT, int U, int MATH, int NB>
__global__ void __launch_bounds__(kFTotal, 3) fused_kernel(const FusedArgs f) {
  constexpr int kRed = 1, kBc = 1 + NB;
  using VV = typename Vec<ET>::V;
  extern __shared__ __align__(16) unsigned char smraw[];
  __shared__ float part[NB][NT][3];  // this CTA's partial state per tensor, read by the cluster over DSMEM
  __shared__ float red[NB][kFW][NT][3];
  __shared__ float bc[NB][4];  // per row: mL, -scale/s, scale, token offset in this slice
  cg::cluster_group cl = cg::this_cluster();
  const int K = (int)cl.num_blocks(), r = (int)cl.block_rank();
  const VocabArgs& a = f.v;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool epi = warp == kEpiWarp;
  const int64_t nrows = (int64_t)a.B * a.T;
  const int64_t ncl = gridDim.x / K;
  const int c0 = r * f.slice;
  const int n = max(0, min(a.V - c0, f.slice));
  VV* const smb = reinterpret_cast<VV*>(smraw);  // NB actor slices
  const int slice_vecs = f.slice / Vec<ET>::kElems;
  // Next loss-participating row of this cluster at or after `row` (the same
  // for every CTA of the cluster); rows passed over get their zero gradient
  // slice (streaming warps) and inactive outputs here.
  // Gradient rows follow the actor logits' layout (padded or packed).
  auto grad_row = [&](int64_t row) { return reinterpret_cast<GT*>(f.grad) + logits_row(a, 0, row) * f.gstride + c0; };
  auto next_active = [&](int64_t row) {
    for (; row < nrows; row += ncl) {
      if (row_active<true>(a, row, r == 0 && tid == 0)) break;
      if (r == 0 && tid == 0) write_inactive<true>(a, row);
      if (!epi && row_exists(a, row)) slice_grad<ET, GT>(nullptr, n, nullptr, grad_row(row), 0.f, 0.f, -1, 0.f);
    }
    return row;
  };
  auto backward = [&](int64_t row, int b) {
    const float* q = bc[b];
    slice_grad<ET, GT>(reinterpret_cast<const ET*>(a.logits[0]) + logits_off(a, 0, row) + c0, n,
                       smb + b * slice_vecs, grad_row(row), q[0], q[1], __float_as_int(q[3]), q[2]);
  };
  int64_t pend[NB];  // row streamed into slot s, awaiting its gradient (-1: none)
#pragma unroll
  for (int s = 0; s < NB; ++s) pend[s] = -1;
  int64_t prev = -1;
  int b = 0;
  for (int64_t row = next_active(blockIdx.x / K); row < nrows; row = next_active(row + ncl), b = (b + 1) % NB) {
    if (!epi) {
      VV* sm = smb + b * slice_vecs;
      const ET* rp0 = reinterpret_cast<const ET*>(a.logits[0]) + logits_off(a, 0, row) + c0;
      Acc acc[NT];
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        acc_init(acc[k]);
        if (k == 0) {
          if (RLO_FUSED_GUARD_ALWAYS) {  // one guarded pass: less code (i-cache), the fp32 row is memory-bound
            slice_pass<ET, U, MATH | kMathGuard, true>(rp0, n, sm, acc[0]);
          } else {
            slice_pass<ET, U, MATH, true>(rp0, n, sm, acc[0]);
            if (!(isfinite(acc[0].s) && isfinite(acc[0].w))) {
              acc_init(acc[0]);  // -inf logits in this thread's share: redo it guarded, from shared memory
              slice_pass<ET, U, MATH | kMathGuard, false>(rp0, n, sm, acc[0]);
            }
          }
        } else {
          const ET* rp = reinterpret_cast<const ET*>(a.logits[k]) + logits_off(a, k, row) + c0;
          stream_accumulate<kFT, ET, U, RLO_FUSED_PF != 0, false, MATH>(rp, n, acc[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        if (k == 0)
          acc_warp_reduce<true>(acc[k]);
        else
          acc_warp_reduce<false>(acc[k]);
        if (lane == 0) {
          red[b][warp][k][0] = acc[k].mL;
          red[b][warp][k][1] = acc[k].s;
          red[b][warp][k][2] = acc[k].w;
        }
      }
      bar_arrive(kRed + b);
      if (prev >= 0) cluster_wait();  // phase of row prev (one phase of slack)
      cluster_arrive_relaxed();        // phase of row `row`
      const int sb = (b + 1) % NB;     // oldest pending slot: the row of NB-1 iterations ago
      if (pend[sb] >= 0) {
        bar_sync(kBc + sb);  // that row's epilogue
        backward(pend[sb], sb);
        pend[sb] = -1;
      }
      pend[b] = row;
    } else {
      int tok = 0;
      bool oov = false;
      float ztok[NT];
      if (lane == 0) gather_token<ET, NT>(a, row, tok, oov, ztok);
      bar_sync(kRed + b);
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        Acc c;
        if (lane < kFW) {
          c.mL = red[b][lane][k][0];
          c.s = red[b][lane][k][1];
          c.w = red[b][lane][k][2];
        } else {
          acc_init(c);
        }
        if (k == 0)
          acc_warp_reduce<true>(c);
        else
          acc_warp_reduce<false>(c);
        if (lane == 0) {
          part[b][k][0] = c.mL;
          part[b][k][1] = c.s;
          part[b][k][2] = c.w;
        }
      }
      cluster_arrive_release();  // publish part[b]
      cluster_wait();            // peers' part[b] visible
      double lse[NT], ent = 0.0;
      float mL0 = 0.f, s0 = 1.f;
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        Acc c;
        if (lane < K) {
          const float* p = cl.map_shared_rank(&part[b][k][0], lane);
          c.mL = p[0];
          c.s = p[1];
          c.w = p[2];
        } else {
          acc_init(c);
        }
        if (k == 0)
          acc_warp_reduce<true>(c);
        else
          acc_warp_reduce<false>(c);
        const RowResult rr = finish(c);
        lse[k] = rr.lse;
        if (k == 0) {
          ent = rr.entropy;
          mL0 = c.mL;
          s0 = c.s;
        }
      }
      if (lane == 0) {
        if (oov && r == 0) flag_error(a, DE_OOV_LOSS, global_row(a, row), tok);
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        double lp[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) lp[k] = oov ? nan : (double)ztok[k] - lse[k];
        const double dlp = row_loss<NT>(a, row, lp, ent, lse[0], r == 0);
        const float scale = __ldg(f.weight + row) * (float)dlp;
        bc[b][0] = mL0;
        bc[b][1] = (float)(-(double)scale / (double)s0);
        bc[b][2] = scale;
        bc[b][3] = __int_as_float(tok - c0);
      }
      __syncwarp();
      bar_arrive(kBc + b);
    }
    prev = row;
  }
  if (!epi && prev >= 0) {
    cluster_wait();  // the last phase
#pragma unroll
    for (int j = 1; j <= NB; ++j) {  // the remaining rows, oldest first
      const int sb = (b + j) % NB;
      if (pend[sb] >= 0) {
        bar_sync(kBc + sb);
        backward(pend[sb], sb);
      }
    }
  }
  cl.sync();  // DSMEM lifetime: no CTA exits while a peer may still read its slots
}

template <typename ET, typename GT, int NT, int NB>
cudaError_t launch_t(const FusedArgs& f, int K, bool debug, cudaStream_t s) {
  constexpr int U = sizeof(ET) == 4 ? 8 : 4;
  constexpr int MATH = sizeof(ET) == 4 ? 1 : 6;  // the vocab pass's measured defaults
  auto kern = fused_kernel<ET, GT, NT, U, MATH, NB>;
  const size_t smem = (size_t)f.slice * sizeof(ET) * NB;  // NB actor slices in flight
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(K);
  cfg.blockDim = dim3(kFTotal);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  if (e != cudaSuccess) return e;
  if (ncl < 1) return cudaErrorInvalidConfiguration;
  const int64_t nrows = (int64_t)f.v.B * f.v.T;
  if (ncl > nrows) ncl = (int)nrows;
  cfg.gridDim = dim3((unsigned)(ncl * K));
  if (debug)
    fprintf(stderr, "[rlo] fused pass: K=%d slice=%d smem=%zu clusters=%d\n", K, f.slice, smem, ncl);
  e = cudaLaunchKernelEx(&cfg, kern, f);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename ET, typename GT, int NB>
cudaError_t launch_nb(const FusedArgs& f, int K, bool debug, cudaStream_t s) {
  switch (f.v.ntens) {
    case 1: return launch_t<ET, GT, 1, NB>(f, K, debug, s);
    case 2: return launch_t<ET, GT, 2, NB>(f, K, debug, s);
    default: return launch_t<ET, GT, 3, NB>(f, K, debug, s);
  }
}

// RLO_FUSED_NB=3: the gradient of a row is written two rows later (three
// actor slices in flight), giving the epilogue and the cluster another row of
// slack at the cost of shared memory (A/B knob, profiles/r1_fused.txt).
template <typename ET, typename GT>
cudaError_t launch_nt(const FusedArgs& f, int K, const Tuning& tu, cudaStream_t s) {
  return tu.fused_nb == 3 ? launch_nb<ET, GT, 3>(f, K, tu.fused_debug, s) : launch_nb<ET, GT, 2>(f, K, tu.fused_debug, s);
}

}  // namespace
}  // namespace vocab

// Cluster size for a fused pass, or 0 when the two-pass form is used instead:
// rows not 16-byte aligned, or an actor row that needs more than
// kMaxCluster CTAs of the slice budget.  Measured (profiles/r1_fused.txt):
// fp32 V=32000 runs best as 4 CTAs x 32 KB slices (3 CTAs/SM) and beats the
// two-pass form by 12%.  bf16 rows lose to the two-pass form at every size
// measured (V = 32000: 8.08 vs 7.59 ms; the Qwen row, 8 CTAs of 38 KB: 11.7 vs
// 8.3 ms) — the bf16 pass is bound by SM power, not bytes — so bf16 stays
// two-pass.  RLO_FUSED_SLICE_KB overrides the budget (and then allows any
// dtype and clusters up to 8) for experiments.
int fused_cluster_size(const VocabArgs& a, const void* grad, int32_t gdtype, int64_t gstride, const Tuning& tu,
                       int32_t* slice) {
  if (tu.fused_off) return 0;
  const int esz = a.dtype == RLO_DTYPE_BF16 ? 2 : 4, gsz = gdtype == RLO_DTYPE_BF16 ? 2 : 4;
  const int E = 16 / esz;
  for (int k = 0; k < a.ntens; ++k)
    if ((reinterpret_cast<uintptr_t>(a.logits[k]) & 15u) || ((a.stride[k] * esz) & 15)) return 0;
  const int gal = E * gsz < 16 ? E * gsz : 16;  // widest gradient store
  if ((reinterpret_cast<uintptr_t>(grad) % gal) || ((gstride * gsz) % gal)) return 0;
  const int forced = tu.fused_slice_kb;
  if (forced <= 0 && a.dtype == RLO_DTYPE_BF16) return 0;  // measured slower than two passes for bf16 (see above)
  const int64_t budget = (int64_t)(forced > 0 ? forced : 32) * 1024;
  const int kmax = forced > 0 ? 8 : 4;
  for (int K = 1; K <= kmax; K *= 2) {
    const int64_t per = ((int64_t)a.V + K - 1) / K;
    const int64_t sl = (per + E - 1) / E * E;
    if (sl * esz <= budget) {
      *slice = (int32_t)sl;
      return K;
    }
  }
  return 0;
}

cudaError_t launch_vocab_fused(const VocabArgs& a, const float* weight, void* grad, int32_t gdtype, int64_t gstride,
                               int K, int32_t slice, const Tuning& tu, cudaStream_t s) {
  using namespace vocab;
  if ((int64_t)a.B * a.T == 0) return cudaSuccess;
  FusedArgs f;
  f.v = a;
  f.weight = weight;
  f.grad = grad;
  f.gstride = gstride;
  f.slice = slice;
  if (a.dtype == RLO_DTYPE_BF16)
    return gdtype == RLO_DTYPE_BF16 ? launch_nt<__nv_bfloat16, __nv_bfloat16>(f, K, tu, s)
                                    : launch_nt<__nv_bfloat16, float>(f, K, tu, s);
  return gdtype == RLO_DTYPE_BF16 ? launch_nt<float, __nv_bfloat16>(f, K, tu, s) : launch_nt<float, float>(f, K, tu, s);
}

}  // namespace rlo
