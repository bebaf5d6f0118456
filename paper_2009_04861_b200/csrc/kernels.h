// kernels.h — launch interface between the host engine and the sm_100a kernels.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace tmg {

// One 256 x 256 GF(2) jump matrix as nibble tables (tm_device.cuh gf2_apply).
constexpr int kGf2TabWords = 64 * 16 * 8;

// Number of kernels this library has launched (evidence for bench.py's gpu_launches).
extern unsigned long long g_launches;
inline void count_launch() { __atomic_fetch_add(&g_launches, 1ULL, __ATOMIC_RELAXED); }

// Threshold bits of the async Bernoulli sampler (tm_device.cuh), precomputed
// on the host: bits 31..24 of P as all-ones / all-zeros masks, bits 23..0 as
// an integer, for P_high = round((s-1)/s * 2^32) and P_low = round(1/s * 2^32).
struct BernThresholds {
  uint32_t hi_mask[8], lo_mask[8];
  uint32_t hi_rest, lo_rest;
  uint32_t one;  // 1, opaque to the compiler (IMAD-as-add in the sampler)
};

constexpr int kMaxPhiloxRounds = 10;
constexpr int kMaxPeers = 7;  // tally replicas of the other ranks (8 GPUs per node)

// Device view of one machine shard + pool, shared by all training kernels.
struct TrainParams {
  // Machine shard: every class keeps clauses [j_begin, j_begin + n_loc).
  uint32_t* state;     // [m*n_loc][B][2][Wp] bit-sliced automaton planes
  int32_t* inc_count;  // [m*n_loc] include count (refreshed at kernel end)
  uint32_t* prev;      // [m*n_loc][Wq] previous clause output per example
  int32_t n, n_loc, j_begin, m, o, Wp, Wq;
  uint32_t lo, hi;  // plane value range of counters [1, 2N]
  // Pool.
  // Literal rows: [q][2][Wp] words, x-plane then !x-plane (tm_device.cuh);
  // nplane == xplane + Wp, row stride 2 * Wp.
  const uint32_t* xplane;  // literals k < o
  const uint32_t* nplane;  // literals k >= o
  const int32_t* labels;   // [q]
  int32_t* tallies;        // [q][m]
  int32_t* tally_delta;    // [q][m] or null: deltas also published here (multi-GPU)
  int32_t* peer_tallies[kMaxPeers];  // other ranks' [q][m] replicas (peer memory)
  int32_t npeers;
  int64_t q;
  // Epoch.
  const int32_t* order;  // [q] epoch permutation, or null = natural order
  int32_t margin;
  int32_t boost;
  // Regression head (proj/src/regression.cpp): one all-positive bank, labels
  // are scaled targets t in [0, T], gate |t - v| / 2T with v = clamp(tally, 0,
  // T), Type I when v < t else Type II (regression.cpp:46-67).
  int32_t regress;
  // Clause order over the grid: 0 = class-major (warp w -> class w / n_loc),
  // 1 = interleaved (warp w -> class w % m, clause w / m), so each resident
  // wave holds a slice of every class instead of all clauses of a few.
  int32_t interleave;
  // Launch over clause-order warps [w_begin, w_end) only (a wave of a
  // sharded epoch); the whole machine is [0, m * n_loc).
  int32_t w_begin, w_end;
  int32_t all_positive;
  uint32_t thr_high, thr_low;  // async: P(u < p) thresholds as 32-bit fixed point
  BernThresholds bern;         // the same, split for the sampler
  const uint32_t* alias8;      // [256] alias table of Bernoulli(thr_low/2^32)^8 (threshold<<8 | alias)
  int32_t alias_sel;           // thr_high + thr_low == 2^32: clause-output-1 draws use the table too
  uint32_t key0, key1;         // async: Philox key for (seed, epoch)
  // The same key's round schedule (key0 + r*0x9E3779B9, key1 + r*0xBB67AE85),
  // precomputed so the rounds read it from the constant bank, not registers.
  uint32_t rkey[2][kMaxPhiloxRounds];
  int64_t t_begin, t_end;      // async: window of each clause's pass
  unsigned long long* events;  // [2m]: feedback events per class, then Type I events per class
  unsigned long long* dbg;     // [kDebugCounters] instrumentation (TMG_STATS builds), else null
  int32_t* work;               // [1] clause counter of the persistent shared-memory kernel (zeroed per launch)
};

constexpr int kDebugCounters = 256;

struct MirrorJob {
  int32_t c, j;  // class, global clause index
  int32_t worker;
  int32_t forced;  // 0: gated update_clause steps; 1/2: one forced Type I/II
                   // feedback on literal row 0 (type_i/ii_feedback, feedback.cpp:87-99)
  int32_t out_override;  // forced jobs: -1 evaluate, 0/1 given clause output
  int32_t pad;
  int64_t offset, batch;
};

// One clause on one literal row (evaluate_clause, core.hpp:208-219).
void eval_one_launch(const uint32_t* state, int lc, int B, int Wp, const uint32_t* x, const uint32_t* n,
                     int train_mode, int32_t* out, cudaStream_t s);

struct MirrorParams {
  const MirrorJob* jobs;
  int32_t njobs;
  uint64_t* rng;  // [workers][4] xoshiro states, in/out
  double p_high, p_low;
  // Type I draws by warp-cooperative jump-ahead (as SeqParams; null: lane 0 draws them serially)
  const uint32_t* jump_chunk;
  const uint32_t* jump_lits;
  int32_t chunk;
};

struct SeqParams {  // classic sequential trainer mirror (trainer.cpp:138-179)
  uint64_t* rng;  // xoshiro state after the epoch shuffle (written back at the end)
  double p_high, p_low;
  unsigned long long* events;  // [m]
  // Parallel replay of the Type I draws (null: the serial replay). The
  // xoshiro256 state transition is linear over GF(2); jump_chunk = M^chunk
  // and jump_lits = M^(2o) as 256 x 256 bit matrices, each as kGf2TabWords
  // words of nibble tables (see tm_device.cuh gf2_apply).
  const uint32_t* jump_chunk;
  const uint32_t* jump_lits;
  int32_t chunk;          // draws per lane: ceil(2o / 32)
  int32_t par_warps;      // warps applying gated clauses in parallel (each with its own draw buffers)
  uint64_t* tstate;       // [n][4]: a gated Type I clause's generator state at its first draw
  // grid-wide replay (cooperative launch over all SMs; null: one CTA):
  // clause-output bits of the two alternating feed slots, gated bits, and
  // [vote slot 0, vote slot 1, negative class]
  uint32_t* g_outs;  // [2][ceil(n/32)]
  uint32_t* g_gbits;  // [ceil(n/32)]
  int32_t* g_misc;    // [3]
};
bool train_sequential_launch(const TrainParams& p, const SeqParams& sp, int B, cudaStream_t s);

// Example-sliced class sums (eval.cu): included-literal lists per clause
// against feature-major bit columns of the examples.
struct BitsEvalParams {
  const uint32_t* lit_t;     // [o + 2][Gs]: bit e of word g = x_f of example 32g + e; row o ones, o + 1 zeros
  uint32_t Gs;               // words per lit_t row (lit_t_stride(q))
  const uint32_t* lists;     // per clause: positive-literal features (padded to 4 with o), then
                             // negated-literal features (padded to 4 with o + 1)
  const int4* meta;          // [m*n_loc] {list offset / 4, list length, positive-part length, 0}
  uint32_t* prev;            // refresh mode: [m*n_loc][Wq]
  int32_t n_loc, j_begin, m, Wq;
  int32_t cta_clauses, chunks;  // clauses per CTA (<= 2040), CTAs per class
  int32_t dynamic;              // long lists: clauses handed out through a shared counter, two
                                // folds of 16 loads; short lists: by stride, one fold of 8 loads
  int32_t all_positive;         // regression head: every clause votes +1
  int64_t q;
  int32_t* sums;  // [q][m], accumulated with atomics
};

// B (plane count) and NW (words per lane per part) instantiations.
bool train_async_launch(const TrainParams& p, int B, int NW, cudaStream_t s, int* blocks);
bool train_async_smem_launch(const TrainParams& p, int B, int NW, cudaStream_t s, int* blocks);
// Clause warps the async kernel for this shape keeps resident on the device
// at once (one wave), and the warps per CTA (waves are cut at CTA multiples).
int train_async_resident_warps(const TrainParams& p, int B, int NW, int* warps_per_cta);
int train_async_smem_resident_warps(const TrainParams& p, int B, int NW, int* warps_per_cta);
bool train_mirror_launch(const TrainParams& p, const MirrorParams& mp, int B, int NW, cudaStream_t s);
bool type_i_async_once_launch(const TrainParams& p, uint32_t* state, uint32_t g, uint32_t i, int out, int B, int NW,
                              cudaStream_t s);
bool type_i_smem_once_launch(const TrainParams& p, uint32_t* state, uint32_t g, uint32_t i, int out, int B, int NW,
                             cudaStream_t s);
bool feedback_rates_launch(const TrainParams& p, const uint32_t* state0, int out, uint32_t trials, int B, int NW,
                           unsigned long long* inc, unsigned long long* dec, cudaStream_t s);
// Include counts, padded list lengths and offsets; returns the total list length (-1 on a CUDA error; syncs).
int64_t build_lists_launch(const uint32_t* state, int clauses, int B, int Wp, int Wx, int32_t* inc_count,
                           int32_t* lens, int32_t* npos, int64_t* offs, cudaStream_t s);
void fill_lists_launch(const uint32_t* state, int clauses, int B, int Wp, int Wx, int o, const int64_t* offs,
                       const int32_t* npos, uint32_t* lists, int4* meta, cudaStream_t s);
int64_t lit_t_stride(int64_t q);
void transpose_literals_launch(const uint32_t* xplane, int64_t row_stride, int64_t q, int o, uint32_t* lit_t,
                               cudaStream_t s);
void eval_bits_launch(const BitsEvalParams& p, bool train_mode, cudaStream_t s);
void counters_to_planes_launch(const uint16_t* counters, uint32_t* state, int clauses, int o, int B,
                               int Wp, int N, cudaStream_t s);
void planes_to_counters_launch(const uint32_t* state, uint16_t* counters, int clauses, int o, int B,
                               int Wp, int N, cudaStream_t s);
void pack_planes_launch(const uint8_t* bits, uint32_t* xplane, uint32_t* nplane, int64_t q, int o,
                        int Wp, int* err, cudaStream_t s);
void check_labels_launch(const int32_t* labels, int64_t q, int m, int* err, cudaStream_t s);
void unpack_ref_literals_launch(const uint64_t* lits, uint32_t* xplane, uint32_t* nplane, int64_t q,
                                int o, int Wp, cudaStream_t s);
void argmax_launch(const int32_t* sums, int32_t* pred, int64_t q, int m, cudaStream_t s);
void init_state_launch(uint32_t* state, int clauses, int B, int Wp, cudaStream_t s);
void clamp_launch(const int32_t* sums, int32_t* out, int64_t q, int T, cudaStream_t s);
void apply_remote_delta_launch(int32_t* tallies, const int32_t* reduced, int32_t* own, int64_t count,
                               cudaStream_t s);
void apply_snapshot_launch(int32_t* tallies, const int32_t* reduced, const int32_t* snap, int64_t count,
                           cudaStream_t s);
// Integer-pipe peak micro-benchmark: returns thread-ops/s for LOP3-only and LOP3+IMAD streams.
bool int_peak_launch(int sms, double* lop3_ops, double* mixed_ops);

}  // namespace tmg
