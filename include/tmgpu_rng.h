/*
 * tmgpu_rng.h — host-side random streams used by the B200 Tsetlin engine.
 *
 * The synchronous mirror mode must replay the reference's random streams bit
 * for bit, so this header restates the reference generator family:
 *   - splitmix64 finaliser            (reference: proj/include/tsetlin/rng.hpp:26-31)
 *   - xoshiro256++ seeded by (seed, stream) (rng.hpp:39-54)
 *   - 53-bit uniform double           (rng.hpp:63)
 *   - Lemire bounded draw w/ rejection (rng.hpp:68-79)
 *   - top-down Fisher-Yates           (rng.hpp:91-103)
 *   - stream mixing / clause offsets  (proj/src/trainer.cpp:29-44)
 *
 * Header-only C99 so the C ABI, the C++ facade and the synthetic-data
 * generators share one definition. The device side has its own copy in
 * csrc/xoshiro_dev.cuh.
 */
#ifndef TMGPU_RNG_H_
#define TMGPU_RNG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMG_GOLDEN_GAMMA 0x9E3779B97F4A7C15ULL

/* Stream kinds of the asynchronous trainer (trainer.cpp:29-31). */
enum { TMG_STREAM_SEQUENTIAL = 1, TMG_STREAM_PERMUTATION = 2, TMG_STREAM_WORKER = 3 };

typedef struct tmg_rng {
  uint64_t s[4];
} tmg_rng;

static inline uint64_t tmg_splitmix64(uint64_t* state) {
  uint64_t z;
  *state += TMG_GOLDEN_GAMMA;
  z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline void tmg_rng_seed(tmg_rng* r, uint64_t seed, uint64_t stream) {
  uint64_t mix = seed ^ (TMG_GOLDEN_GAMMA * (stream + 1));
  int w;
  for (w = 0; w < 4; ++w) r->s[w] = tmg_splitmix64(&mix);
}

static inline uint64_t tmg_rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static inline uint64_t tmg_rng_next(tmg_rng* r) {
  uint64_t* s = r->s;
  const uint64_t out = tmg_rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t shifted = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= shifted;
  s[3] = tmg_rotl64(s[3], 45);
  return out;
}

/* (next >> 11) * 2^-53: every value is an exact multiple of 2^-53. */
static inline double tmg_rng_uniform(tmg_rng* r) {
  return (double)(tmg_rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
}

static inline int tmg_rng_bernoulli(tmg_rng* r, double p) { return tmg_rng_uniform(r) < p; }

static inline uint32_t tmg_rng_below(tmg_rng* r, uint32_t bound) {
  uint64_t prod = (uint64_t)(uint32_t)tmg_rng_next(r) * (uint64_t)bound;
  uint32_t lo = (uint32_t)prod;
  if (lo < bound) {
    const uint32_t reject_below = (uint32_t)(0u - bound) % bound;
    while (lo < reject_below) {
      prod = (uint64_t)(uint32_t)tmg_rng_next(r) * (uint64_t)bound;
      lo = (uint32_t)prod;
    }
  }
  return (uint32_t)(prod >> 32);
}

/* order[0..count) = identity shuffled from the top down. */
static inline void tmg_shuffled_indices(int32_t count, tmg_rng* r, int32_t* order) {
  int32_t i;
  for (i = 0; i < count; ++i) order[i] = i;
  for (i = count; i > 1; --i) {
    const uint32_t j = tmg_rng_below(r, (uint32_t)i);
    const int32_t tmp = order[i - 1];
    order[i - 1] = order[j];
    order[j] = tmp;
  }
}

static inline uint64_t tmg_mix_stream(uint64_t kind, uint64_t a, uint64_t b) {
  uint64_t x = kind;
  x = tmg_splitmix64(&x) ^ a;
  x = tmg_splitmix64(&x) ^ b;
  return tmg_splitmix64(&x);
}

/* Starting position of clause g (global index c*n+j) in the epoch order. */
static inline uint64_t tmg_clause_offset(uint64_t global_index, int64_t pool_size) {
  uint64_t x = global_index + 1;
  return tmg_splitmix64(&x) % (uint64_t)pool_size;
}

#ifdef __cplusplus
}
#endif

#endif /* TMGPU_RNG_H_ */
