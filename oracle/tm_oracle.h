/*
 * tm_oracle.h — CPU restatement of the reference's asynchronous Tsetlin
 * Machine path, in plain C. TEST INFRASTRUCTURE ONLY: imported by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker;
 * the product (paper_2009_04861_b200) never links or calls it.
 *
 * Parity of this restatement is PINNED against the compiled reference
 * (oracle/_ref/ref_driver golden dumps under tests/golden/, checked by
 * tests/test_oracle_golden.py).
 *
 * Storage mirrors the reference exactly:
 *   counters  m x n x 2o uint16 in [1, 2N]     (core.hpp:40, 200)
 *   masks     m x n x ceil(2o/64) uint64        (core.hpp:201)
 *   counts    m x n int32                       (core.hpp:202)
 *   prev      m x n x ceil(q/64) uint64         (core.hpp:203)
 *   literals  q x ceil(2o/64) uint64, features then negations (core.cpp:34-46)
 *   tallies   q x m int32, example-major        (pool.hpp:66-69)
 */
#ifndef TM_ORACLE_H_
#define TM_ORACLE_H_

#include <stdint.h>

typedef struct {
  uint64_t s[4];
} orc_rng;

typedef struct {
  int32_t o, L, m, n, N, W64;
  int32_t q_bound, out_words;
  uint16_t* counters;
  uint64_t* masks;
  int32_t* counts;
  uint64_t* prev;
} orc_machine;

typedef struct {
  int32_t o, m, W64;
  int64_t q;
  const uint64_t* lits;
  const int32_t* labels;
  int32_t* tallies;
} orc_pool;

enum { ORC_TRAIN = 0, ORC_PREDICT = 1 };

uint64_t orc_splitmix64(uint64_t* state);
void orc_rng_init(orc_rng* r, uint64_t seed, uint64_t stream);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
uint32_t orc_rng_below(orc_rng* r, uint32_t bound);
void orc_shuffled_indices(int32_t count, orc_rng* r, int32_t* out);
uint64_t orc_mix_stream(uint64_t kind, uint64_t a, uint64_t b);
uint64_t orc_clause_offset(uint64_t g, int64_t q);

void orc_pack_literals(int32_t o, const uint8_t* x, uint64_t* words);
double orc_clause_update_probability(int32_t vote_sum, int32_t y, int32_t margin);
void orc_rebuild_masks(orc_machine* tm);
int orc_evaluate_clause(const orc_machine* tm, int c, int j, const uint64_t* lits, int mode);
void orc_type_i(orc_machine* tm, int c, int j, const uint64_t* lits, int clause_output, double s,
                int boost, orc_rng* r);
void orc_type_ii(orc_machine* tm, int c, int j, const uint64_t* lits, int clause_output);
int orc_bind(orc_machine* tm, int32_t q);  /* caller must size prev for q first */
uint64_t orc_update_clause(orc_machine* tm, orc_pool* pool, int c, int j, const int32_t* order,
                           int64_t offset, int64_t batch, int32_t margin, double s, int boost,
                           orc_rng* r);
void orc_train_epoch_parallel(orc_machine* tm, orc_pool* pool, int32_t margin, double s, int boost,
                              uint64_t seed, int32_t workers, int32_t epoch, uint64_t* events);
void orc_train_epoch_sequential(orc_machine* tm, orc_pool* pool, int32_t margin, double s, int boost,
                                uint64_t seed, int32_t epoch, uint64_t* events);
int32_t orc_vote_sum(const orc_machine* tm, int c, const uint64_t* lits, int mode);
void orc_class_sums(const orc_machine* tm, const uint64_t* lits, int64_t q, int32_t* sums);
void orc_predict(const orc_machine* tm, const uint64_t* lits, int64_t q, int32_t* pred);
void orc_refresh_tallies(orc_machine* tm, orc_pool* pool);

/* Regression head (tm_oracle_regress.c; m = 1 all-positive bank). */
double orc_regress_gate(int32_t t, int32_t v, int32_t T);
uint64_t orc_update_regress(orc_machine* tm, const uint64_t* lits, int32_t t, int32_t T, double s, int boost,
                            orc_rng* r);
uint64_t orc_train_epoch_regress_sequential(orc_machine* tm, orc_pool* pool, int32_t T, double s, int boost,
                                            uint64_t seed, int32_t epoch);
uint64_t orc_train_epoch_regress_parallel(orc_machine* tm, orc_pool* pool, int32_t T, double s, int boost,
                                          uint64_t seed, int32_t workers, int32_t epoch);
void orc_predict_scaled(const orc_machine* tm, const uint64_t* lits, int64_t q, int32_t T, int32_t* out);

/* tm_oracle_async.c: the async engine's Philox Type I draw, restated. */
void orc_philox4x32(const uint32_t ctr[4], uint32_t k0, uint32_t k1, int rounds, uint32_t out[4]);
void orc_async_key(uint64_t seed, int32_t epoch, uint32_t* key0, uint32_t* key1);
uint32_t orc_prob_threshold(double p);
void orc_async_type_i(uint16_t* counters, const uint64_t* lits, int32_t o, int32_t N, int32_t out, double s,
                      int32_t boost, uint32_t g, uint32_t i, uint32_t key0, uint32_t key1, int32_t nw,
                      int32_t rounds, const uint32_t* alias8);

#endif
