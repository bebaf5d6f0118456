/*
 * tm_oracle_regress.c — plain-C restatement of the reference regression head
 * (proj/src/regression.cpp). TEST INFRASTRUCTURE ONLY (see tm_oracle.h).
 * The machine has m = 1 bank whose clauses all vote +1
 * (PolarityScheme::AllPositive, core.hpp:102,122-124); pool labels are the
 * scaled integer targets t in [0, T].
 */
#include <stdlib.h>

#include "tm_oracle.h"

/* regression.cpp:46-48 */
double orc_regress_gate(int32_t t, int32_t v, int32_t T) {
  double p = (double)abs(t - v) / (2.0 * (double)T);
  return p < 1.0 ? p : 1.0;
}

static int clamp0T(int32_t v, int32_t T) { return v < 0 ? 0 : (v > T ? T : v); }

static int32_t count_train(const orc_machine* tm, const uint64_t* lits) {
  int32_t sum = 0;
  for (int j = 0; j < tm->n; ++j) sum += orc_evaluate_clause(tm, 0, j, lits, ORC_TRAIN);
  return sum;
}

/* regression.cpp:50-67 (feed_clause_regress) */
static uint64_t feed_clause(orc_machine* tm, int j, const uint64_t* lits, int32_t t, int32_t v, int32_t T,
                            double s, int boost, orc_rng* r) {
  if (orc_rng_uniform(r) >= orc_regress_gate(t, v, T)) return 0;
  int out = orc_evaluate_clause(tm, 0, j, lits, ORC_TRAIN);
  if (v < t) orc_type_i(tm, 0, j, lits, out, s, boost, r);
  else orc_type_ii(tm, 0, j, lits, out);
  return 1;
}

/* regression.cpp:101-123 */
uint64_t orc_update_regress(orc_machine* tm, const uint64_t* lits, int32_t t, int32_t T, double s, int boost,
                            orc_rng* r) {
  int32_t v = clamp0T(count_train(tm, lits), T);
  uint64_t events = 0;
  for (int j = 0; j < tm->n; ++j) events += feed_clause(tm, j, lits, t, v, T, s, boost, r);
  return events;
}

/* regression.cpp:125-161 */
uint64_t orc_train_epoch_regress_sequential(orc_machine* tm, orc_pool* pool, int32_t T, double s, int boost,
                                            uint64_t seed, int32_t epoch) {
  int64_t q = pool->q;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)q);
  orc_rng r;
  uint64_t events = 0;
  orc_rng_init(&r, seed, orc_mix_stream(4, (uint64_t)epoch, 0));
  orc_shuffled_indices((int32_t)q, &r, order);
  for (int64_t k = 0; k < q; ++k) {
    int64_t i = order[k];
    const uint64_t* lits = pool->lits + i * pool->W64;
    int32_t t = pool->labels[i];
    int32_t v = clamp0T(count_train(tm, lits), T);
    for (int j = 0; j < tm->n; ++j) events += feed_clause(tm, j, lits, t, v, T, s, boost, &r);
  }
  free(order);
  return events;
}

/* regression.cpp:163-227 — workers run one after another (a legal schedule
 * of the reference's threads; exactly the reference for one worker). */
uint64_t orc_train_epoch_regress_parallel(orc_machine* tm, orc_pool* pool, int32_t T, double s, int boost,
                                          uint64_t seed, int32_t workers, int32_t epoch) {
  int64_t q = pool->q;
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)q);
  orc_rng perm;
  uint64_t events = 0;
  if (tm->q_bound != q) orc_bind(tm, (int32_t)q);
  orc_rng_init(&perm, seed, orc_mix_stream(5, (uint64_t)epoch, 0));
  orc_shuffled_indices((int32_t)q, &perm, order);
  for (int32_t w = 0; w < workers; ++w) {
    orc_rng r;
    orc_rng_init(&r, seed, orc_mix_stream(6, (uint64_t)epoch, (uint64_t)w));
    for (int j = w; j < tm->n; j += workers) {
      uint64_t off = orc_clause_offset((uint64_t)j, q);
      for (int64_t step = 0; step < q; ++step) {
        int64_t i = order[(off + (uint64_t)step) % (uint64_t)q];
        int32_t t = pool->labels[i];
        int32_t v = clamp0T(pool->tallies[i * pool->m], T);
        const uint64_t* lits = pool->lits + i * pool->W64;
        if (!feed_clause(tm, j, lits, t, v, T, s, boost, &r)) continue;
        ++events;
        /* record_output_and_tally (pool.cpp:93-106), positive polarity */
        int after = orc_evaluate_clause(tm, 0, j, lits, ORC_TRAIN);
        uint64_t* word = tm->prev + (size_t)j * tm->out_words + (i >> 6);
        int prev = (int)((*word >> (i & 63)) & 1u);
        if (prev != after) {
          pool->tallies[i * pool->m] += after ? 1 : -1;
          *word ^= 1ULL << (i & 63);
        }
      }
    }
  }
  free(order);
  return events;
}

/* regression.cpp:86-93 */
void orc_predict_scaled(const orc_machine* tm, const uint64_t* lits, int64_t q, int32_t T, int32_t* out) {
  for (int64_t i = 0; i < q; ++i) {
    int32_t sum = 0;
    for (int j = 0; j < tm->n; ++j) sum += orc_evaluate_clause(tm, 0, j, lits + i * tm->W64, ORC_PREDICT);
    out[i] = clamp0T(sum, T);
  }
}
