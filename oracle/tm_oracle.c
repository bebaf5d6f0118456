/*
 * tm_oracle.c — plain-C restatement of the reference hot path (checker only;
 * see tm_oracle.h). Each function cites the reference file:line it restates.
 * Paths are relative to /root/reference/proj.
 */
#include "tm_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG --- */

/* include/tsetlin/rng.hpp:26-31 */
uint64_t orc_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.hpp:39-42 */
void orc_rng_init(orc_rng* r, uint64_t seed, uint64_t stream) {
  uint64_t x = seed ^ (0x9E3779B97F4A7C15ULL * (stream + 1));
  for (int k = 0; k < 4; ++k) r->s[k] = orc_splitmix64(&x);
}

static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* rng.hpp:44-54 (xoshiro256++) */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
  uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

/* rng.hpp:63 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:68-79 */
uint32_t orc_rng_below(orc_rng* r, uint32_t bound) {
  uint64_t m = (uint64_t)(uint32_t)orc_rng_next(r) * bound;
  uint32_t low = (uint32_t)m;
  if (low < bound) {
    uint32_t cutoff = (uint32_t)(-bound) % bound;
    while (low < cutoff) {
      m = (uint64_t)(uint32_t)orc_rng_next(r) * bound;
      low = (uint32_t)m;
    }
  }
  return (uint32_t)(m >> 32);
}

/* rng.hpp:91-103 */
void orc_shuffled_indices(int32_t count, orc_rng* r, int32_t* out) {
  for (int32_t i = 0; i < count; ++i) out[i] = i;
  for (int64_t i = count; i > 1; --i) {
    uint32_t j = orc_rng_below(r, (uint32_t)i);
    int32_t t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

/* src/trainer.cpp:33-39 */
uint64_t orc_mix_stream(uint64_t kind, uint64_t a, uint64_t b) {
  uint64_t x = kind;
  x = orc_splitmix64(&x) ^ a;
  x = orc_splitmix64(&x) ^ b;
  return orc_splitmix64(&x);
}

/* src/trainer.cpp:41-44 */
uint64_t orc_clause_offset(uint64_t g, int64_t q) {
  uint64_t x = g + 1;
  return orc_splitmix64(&x) % (uint64_t)q;
}

/* --------------------------------------------------------------- core --- */

/* src/core.cpp:34-46: bit f = x_f, bit o+f = !x_f */
void orc_pack_literals(int32_t o, const uint8_t* x, uint64_t* words) {
  int32_t nw = (2 * o + 63) / 64;
  memset(words, 0, sizeof(uint64_t) * (size_t)nw);
  for (int32_t f = 0; f < o; ++f) {
    int32_t k = x[f] ? f : o + f;
    words[k >> 6] |= 1ULL << (k & 63);
  }
}

/* src/feedback.cpp:24-28 */
double orc_clause_update_probability(int32_t v, int32_t y, int32_t T) {
  int32_t c = v < -T ? -T : (v > T ? T : v);
  int32_t e = y == 1 ? T - c : T + c;
  return (double)e / (2.0 * (double)T);
}

static size_t cidx(const orc_machine* tm, int c, int j) { return (size_t)c * tm->n + (size_t)j; }

/* src/core.cpp:128-139 */
void orc_rebuild_masks(orc_machine* tm) {
  size_t clauses = (size_t)tm->m * tm->n;
  memset(tm->masks, 0, sizeof(uint64_t) * clauses * tm->W64);
  memset(tm->counts, 0, sizeof(int32_t) * clauses);
  for (size_t g = 0; g < clauses; ++g)
    for (int k = 0; k < tm->L; ++k)
      if (tm->counters[g * tm->L + k] > tm->N) {
        tm->masks[g * tm->W64 + (k >> 6)] |= 1ULL << (k & 63);
        tm->counts[g]++;
      }
}

/* include/tsetlin/core.hpp:208-219 */
int orc_evaluate_clause(const orc_machine* tm, int c, int j, const uint64_t* lits, int mode) {
  size_t g = cidx(tm, c, j);
  if (tm->counts[g] == 0) return mode == ORC_TRAIN ? 1 : 0;
  const uint64_t* mk = tm->masks + g * tm->W64;
  for (int w = 0; w < tm->W64; ++w)
    if ((mk[w] & lits[w]) != mk[w]) return 0;
  return 1;
}

/* core.hpp:46-65 (apply_transition) + core.hpp:134-145 (reinforce).
 * dir: +1 = Reward, -1 = Penalty. */
static void reinforce(orc_machine* tm, size_t g, int k, int reward) {
  uint16_t* cell = tm->counters + g * tm->L + k;
  int N = tm->N, before = *cell, after = before;
  int included = before > N;
  if (reward) after = included ? before + 1 : before - 1;
  else after = included ? before - 1 : before + 1;
  if (after < 1) after = 1;
  if (after > 2 * N) after = 2 * N;
  if (after == before) return;
  *cell = (uint16_t)after;
  if ((after > N) == included) return;
  tm->masks[g * tm->W64 + (k >> 6)] ^= 1ULL << (k & 63);
  tm->counts[g] += (after > N) ? 1 : -1;
}

static int bit_of(const uint64_t* w, int k) { return (int)((w[k >> 6] >> (k & 63)) & 1u); }

/* src/feedback.cpp:32-70 — one uniform per literal, always consumed. */
void orc_type_i(orc_machine* tm, int c, int j, const uint64_t* lits, int out, double s, int boost,
                orc_rng* r) {
  size_t g = cidx(tm, c, j);
  double p_high = (s - 1.0) / s, p_low = 1.0 / s;
  for (int k = 0; k < tm->L; ++k) {
    int included = tm->counters[g * tm->L + k] > tm->N;
    double u = orc_rng_uniform(r);
    if (out == 1) {
      if (bit_of(lits, k)) {
        if (included) {
          if (boost || u < p_high) reinforce(tm, g, k, 1);
        } else if (u < p_high) {
          reinforce(tm, g, k, 0);
        }
      } else if (u < p_low) {
        reinforce(tm, g, k, 1);
      }
    } else if (u < p_low) {
      reinforce(tm, g, k, included ? 0 : 1);
    }
  }
}

/* src/feedback.cpp:72-83 */
void orc_type_ii(orc_machine* tm, int c, int j, const uint64_t* lits, int out) {
  if (out != 1) return;
  size_t g = cidx(tm, c, j);
  for (int k = 0; k < tm->L; ++k)
    if (!bit_of(lits, k) && tm->counters[g * tm->L + k] <= tm->N) reinforce(tm, g, k, 0);
}

/* src/core.cpp:117-126 */
int orc_bind(orc_machine* tm, int32_t q) {
  tm->q_bound = q;
  tm->out_words = (q + 63) / 64;
  memset(tm->prev, 0, sizeof(uint64_t) * (size_t)tm->m * tm->n * tm->out_words);
  return 0;
}

static int prev_bit(const orc_machine* tm, size_t g, int64_t i) {
  return (int)((tm->prev[g * tm->out_words + (i >> 6)] >> (i & 63)) & 1u);
}

/* src/pool.cpp:93-106 (index checks elided: callers pass valid indices) */
static void record_output_and_tally(orc_machine* tm, orc_pool* pool, int64_t i, int c, int j,
                                    int out) {
  size_t g = cidx(tm, c, j);
  int prev = prev_bit(tm, g, i), cur = out != 0;
  if (prev == cur) return;
  int32_t delta = cur ? 1 : -1;
  if (j % 2 != 0) delta = -delta; /* negative polarity: odd 0-based j */
  pool->tallies[i * pool->m + c] += delta;
  tm->prev[g * tm->out_words + (i >> 6)] ^= 1ULL << (i & 63);
}

/* src/trainer.cpp:102-136 */
uint64_t orc_update_clause(orc_machine* tm, orc_pool* pool, int c, int j, const int32_t* order,
                           int64_t offset, int64_t batch, int32_t margin, double s, int boost,
                           orc_rng* r) {
  int64_t q = pool->q;
  uint64_t events = 0;
  int positive = (j % 2) == 0;
  if (tm->q_bound != q) orc_bind(tm, (int32_t)q);
  for (int64_t t = 0; t < batch; ++t) {
    int64_t pos = (offset + t) % q;
    int64_t i = order ? order[pos] : pos;
    int32_t v = pool->tallies[i * pool->m + c];
    int32_t target = pool->labels[i] == c ? 1 : 0;
    double p = orc_clause_update_probability(v, target, margin);
    if (orc_rng_uniform(r) >= p) continue;
    ++events;
    const uint64_t* lits = pool->lits + i * pool->W64;
    int before = orc_evaluate_clause(tm, c, j, lits, ORC_TRAIN);
    if ((target == 1) != positive) orc_type_ii(tm, c, j, lits, before);
    else orc_type_i(tm, c, j, lits, before, s, boost, r);
    int after = orc_evaluate_clause(tm, c, j, lits, ORC_TRAIN);
    record_output_and_tally(tm, pool, i, c, j, after);
  }
  return events;
}

/* src/trainer.cpp:181-242. Workers run one after another: a legal schedule
 * of the reference's concurrent threads (exactly the reference for W=1). */
void orc_train_epoch_parallel(orc_machine* tm, orc_pool* pool, int32_t margin, double s, int boost,
                              uint64_t seed, int32_t workers, int32_t epoch, uint64_t* events) {
  int64_t q = pool->q;
  int64_t total = (int64_t)tm->m * tm->n;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)q);
  orc_rng perm;
  if (tm->q_bound != q) orc_bind(tm, (int32_t)q);
  orc_rng_init(&perm, seed, orc_mix_stream(2, (uint64_t)epoch, 0));
  orc_shuffled_indices((int32_t)q, &perm, order);
  for (int c = 0; c < tm->m; ++c) events[c] = 0;
  for (int32_t w = 0; w < workers; ++w) {
    orc_rng r;
    orc_rng_init(&r, seed, orc_mix_stream(3, (uint64_t)epoch, (uint64_t)w));
    for (int64_t g = w; g < total; g += workers) {
      int c = (int)(g / tm->n), j = (int)(g % tm->n);
      int64_t off = (int64_t)orc_clause_offset((uint64_t)g, q);
      events[c] += orc_update_clause(tm, pool, c, j, order, off, q, margin, s, boost, &r);
    }
  }
  free(order);
}

/* src/trainer.cpp:57-85 (feed_bank_sequential) */
static uint64_t feed_bank(orc_machine* tm, int c, const uint64_t* lits, int target, int32_t margin,
                          double s, int boost, uint8_t* outputs, orc_rng* r) {
  int32_t sum = 0;
  for (int j = 0; j < tm->n; ++j) {
    int out = orc_evaluate_clause(tm, c, j, lits, ORC_TRAIN);
    outputs[j] = (uint8_t)out;
    sum += (j % 2 == 0) ? out : -out;
  }
  double p = orc_clause_update_probability(sum, target, margin);
  uint64_t events = 0;
  for (int j = 0; j < tm->n; ++j) {
    if (orc_rng_uniform(r) >= p) continue;
    ++events;
    int positive = (j % 2) == 0;
    if ((target == 1) != positive) orc_type_ii(tm, c, j, lits, outputs[j]);
    else orc_type_i(tm, c, j, lits, outputs[j], s, boost, r);
  }
  return events;
}

/* src/trainer.cpp:138-179 */
void orc_train_epoch_sequential(orc_machine* tm, orc_pool* pool, int32_t margin, double s, int boost,
                                uint64_t seed, int32_t epoch, uint64_t* events) {
  int64_t q = pool->q;
  int m = tm->m;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)q);
  uint8_t* outputs = (uint8_t*)malloc((size_t)tm->n);
  orc_rng r;
  orc_rng_init(&r, seed, orc_mix_stream(1, (uint64_t)epoch, 0));
  orc_shuffled_indices((int32_t)q, &r, order);
  for (int c = 0; c < m; ++c) events[c] = 0;
  for (int64_t t = 0; t < q; ++t) {
    int64_t i = order[t];
    const uint64_t* lits = pool->lits + i * pool->W64;
    int y = pool->labels[i], neg;
    if (m == 2) {
      neg = 1 - y;
    } else {
      neg = (int)orc_rng_below(&r, (uint32_t)(m - 1));
      if (neg >= y) ++neg;
    }
    events[y] += feed_bank(tm, y, lits, 1, margin, s, boost, outputs, &r);
    events[neg] += feed_bank(tm, neg, lits, 0, margin, s, boost, outputs, &r);
  }
  free(order);
  free(outputs);
}

/* src/pool.cpp:82-91 */
int32_t orc_vote_sum(const orc_machine* tm, int c, const uint64_t* lits, int mode) {
  int32_t sum = 0;
  for (int j = 0; j < tm->n; ++j) {
    int out = orc_evaluate_clause(tm, c, j, lits, mode);
    sum += (j % 2 == 0) ? out : -out;
  }
  return sum;
}

/* src/trainer.cpp:262-270 (export_vote_sums, per example) */
void orc_class_sums(const orc_machine* tm, const uint64_t* lits, int64_t q, int32_t* sums) {
  for (int64_t i = 0; i < q; ++i)
    for (int c = 0; c < tm->m; ++c)
      sums[i * tm->m + c] = orc_vote_sum(tm, c, lits + i * tm->W64, ORC_PREDICT);
}

/* src/trainer.cpp:244-260 (classify) + 272-279 (predict_all) */
void orc_predict(const orc_machine* tm, const uint64_t* lits, int64_t q, int32_t* pred) {
  for (int64_t i = 0; i < q; ++i) {
    const uint64_t* row = lits + i * tm->W64;
    if (tm->m == 1) {
      pred[i] = orc_vote_sum(tm, 0, row, ORC_PREDICT) >= 0 ? 1 : 0;
      continue;
    }
    int best = 0;
    int32_t best_sum = orc_vote_sum(tm, 0, row, ORC_PREDICT);
    for (int c = 1; c < tm->m; ++c) {
      int32_t v = orc_vote_sum(tm, c, row, ORC_PREDICT);
      if (v > best_sum) {
        best_sum = v;
        best = c;
      }
    }
    pred[i] = best;
  }
}

/* src/pool.cpp:108-124 */
void orc_refresh_tallies(orc_machine* tm, orc_pool* pool) {
  int64_t q = pool->q;
  if (tm->q_bound != q) orc_bind(tm, (int32_t)q);
  for (int c = 0; c < tm->m; ++c)
    for (int64_t i = 0; i < q; ++i) {
      const uint64_t* lits = pool->lits + i * pool->W64;
      int32_t sum = 0;
      for (int j = 0; j < tm->n; ++j) {
        size_t g = cidx(tm, c, j);
        int out = orc_evaluate_clause(tm, c, j, lits, ORC_TRAIN);
        sum += (j % 2 == 0) ? out : -out;
        uint64_t bit = 1ULL << (i & 63);
        if (out) tm->prev[g * tm->out_words + (i >> 6)] |= bit;
        else tm->prev[g * tm->out_words + (i >> 6)] &= ~bit;
      }
      pool->tallies[i * pool->m + c] = sum;
    }
}
