/*
 * rlo_synth.h — the deterministic synthetic-input generator shared bit-for-bit
 * by the CUDA bench/test kernels (paper_2506_06122_b200/csrc/synth.cu) and the
 * CPU oracle (oracle/oracle.c).  Not part of the objective path.
 *
 * Counter-based: every logit is a pure function of (seed, model, row_key, v),
 * keyed with the splitmix64 finaliser the reference uses for all derived
 * randomness (include/rollmini/rng.hpp:15-31), so any row can be regenerated
 * on either side without storing it.
 *
 *   z_actor(k, v) = g0(k, v) * SIGMA_SCALE  (+ 8 if v is one of the row's 4 spike tokens)
 *   z_m(k, v)     = z_actor(k, v) + g_m(k, v) * PERT_SCALE      (m = 1 old policy, 2 reference)
 *
 * g(h) = sum of the four 16-bit fields of a 64-bit hash minus 131070: an
 * exact integer with mean 0 and std 37837.23, so z has std 3 (actor) and the
 * old/ref models differ from the actor by std 0.05.  Each float operation is
 * a single explicitly rounded step (no FMA contraction), so CPU and GPU agree
 * exactly; bf16 uses round-to-nearest-even.
 */
#ifndef RLO_SYNTH_H_
#define RLO_SYNTH_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define RLO_HD __host__ __device__ __forceinline__
#else
#define RLO_HD static inline
#endif

#define RLO_SYNTH_MAX_V 262144 /* 2^18: v is packed below the row key */
#define RLO_SYNTH_SPIKES 4
#define RLO_SYNTH_SIGMA_SCALE 0x1.4c8dc2p-14f /* 3.0f / 37837.227 */
#define RLO_SYNTH_PERT_SCALE 0x1.62b958p-20f  /* 0.05f / 37837.227 */
#define RLO_SYNTH_SPIKE 8.0f

RLO_HD uint64_t rlo_sm64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

RLO_HD int32_t rlo_synth_gint(uint64_t h) {
  return (int32_t)((h & 0xFFFFu) + ((h >> 16) & 0xFFFFu) + ((h >> 32) & 0xFFFFu) + (h >> 48)) - 131070;
}

RLO_HD uint64_t rlo_synth_model_key(uint64_t seed, int32_t model) {
  return rlo_sm64(seed ^ (0xA5A5000000000000ULL + (uint64_t)(uint32_t)model));
}

RLO_HD int32_t rlo_synth_spike(uint64_t seed, uint64_t row_key, int32_t k, int32_t V) {
  uint64_t h = rlo_sm64(rlo_sm64(seed ^ 0x5B1CE5ULL) ^ (row_key * RLO_SYNTH_SPIKES + (uint64_t)k));
  return (int32_t)(h % (uint64_t)V);
}

RLO_HD int32_t rlo_synth_token(uint64_t seed, uint64_t row_key, int32_t V) {
  uint64_t u = rlo_sm64(rlo_sm64(seed ^ 0x70CE5ULL) ^ row_key);
  if ((u & 3u) != 0) return rlo_synth_spike(seed, row_key, (int32_t)((u >> 2) & 3u), V);
  return (int32_t)((u >> 8) % (uint64_t)V);
}

#if defined(__CUDA_ARCH__)
#define RLO_FMUL(a, b) __fmul_rn((a), (b))
#define RLO_FADD(a, b) __fadd_rn((a), (b))
#else
#define RLO_FMUL(a, b) ((float)((float)(a) * (float)(b)))
#define RLO_FADD(a, b) ((float)((float)(a) + (float)(b)))
#endif

/* Logit of (row_key, v) for `model`, given the row's spike set and the two
 * model keys (actor key always needed; model key only for model != 0). */
RLO_HD float rlo_synth_logit(uint64_t k0, uint64_t km, int32_t model, uint64_t row_key, int32_t v,
                             const int32_t* spikes) {
  const uint64_t x = (row_key << 18) | (uint64_t)(uint32_t)v;
  float z = RLO_FMUL((float)rlo_synth_gint(rlo_sm64(x ^ k0)), RLO_SYNTH_SIGMA_SCALE);
  int hit = 0;
  for (int k = 0; k < RLO_SYNTH_SPIKES; ++k) hit |= (spikes[k] == v);
  if (hit) z = RLO_FADD(z, RLO_SYNTH_SPIKE);
  if (model != 0) z = RLO_FADD(z, RLO_FMUL((float)rlo_synth_gint(rlo_sm64(x ^ km)), RLO_SYNTH_PERT_SCALE));
  return z;
}

RLO_HD uint16_t rlo_f32_to_bf16_rne(float f) {
  union { float f; uint32_t u; } c;
  c.f = f;
  uint32_t bias = 0x7FFFu + ((c.u >> 16) & 1u);
  return (uint16_t)((c.u + bias) >> 16);
}

RLO_HD float rlo_bf16_to_f32(uint16_t b) {
  union { float f; uint32_t u; } c;
  c.u = ((uint32_t)b) << 16;
  return c.f;
}

#endif /* RLO_SYNTH_H_ */
