/*
 * tmgpu.h — C ABI of the B200-native asynchronous Tsetlin Machine engine
 * (libtmgpu.so). Plain pointers and sizes only; no C++ or torch types.
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (tsetlin-cpp, /root/reference/proj) exposes a statically linked C++ header
 * API with no FFI; each entry below names the reference function or member it
 * replaces (file:line under proj/). The C++ facade in include/tsetlin/*.hpp
 * re-exposes the reference's own class and function names on top of this ABI
 * (see INTEGRATION.md).
 *
 * Conventions
 *   - Every function returns TMG_OK (0) or an error code; the message of the
 *     last error on the calling thread is available from tmg_last_error().
 *     Error classes mirror the reference's exceptions:
 *       TMG_EINVAL  <- std::invalid_argument (core.cpp:48-74, pool.cpp:29-55,
 *                      trainer.cpp:46-53,106,110,184)
 *       TMG_ERANGE  <- std::out_of_range    (core.cpp:26-29, pool.cpp:95-98)
 *       TMG_ERUNTIME<- std::runtime_error / CUDA failures
 *   - Host buffers are caller-owned and only borrowed for the call.
 *   - All calls are synchronous (they return after the device work is done)
 *     and a handle must not be used from two threads at once — the
 *     reference's threading contract (pool.hpp:92-93).
 *   - Layouts at the boundary are the reference's: counters n x 2o uint16 in
 *     [1, 2N] per bank (core.hpp:200), literal rows ceil(2o/64) uint64 with
 *     features then negations (core.cpp:34-46), tallies q x m int32
 *     (pool.hpp:66-69), previous outputs n x ceil(q/64) uint64 per bank
 *     (core.hpp:203).
 */
#ifndef TMGPU_H_
#define TMGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMG_OK 0
#define TMG_EINVAL 1
#define TMG_ERANGE 2
#define TMG_ERUNTIME 3

#define TMG_ABI_VERSION 1

/* Training modes of tmg_train_epoch. */
#define TMG_MODE_ASYNC 0       /* Algorithm 1, every clause concurrently (GPU) */
#define TMG_MODE_SYNC_MIRROR 1 /* bit-exact replay of train_epoch_parallel's
                                  W-worker schedule (exact reference for W=1) */
#define TMG_MODE_AUTO 2        /* what the drop-in train_epoch_parallel uses (C++
                                  facade and Python alike): TMG_MODE_ASYNC for any
                                  `workers`, unless workers == 1 and the environment
                                  sets TSETLIN_DETERMINISTIC=1, which selects the
                                  bit-exact single-worker replay */

/* Evaluation modes (core.hpp:33-35). */
#define TMG_EVAL_TRAIN 0
#define TMG_EVAL_PREDICT 1

typedef struct tmg_machine tmg_machine;
typedef struct tmg_pool tmg_pool;

/* TMConfig (core.hpp:85-97). */
typedef struct tmg_config {
  int32_t clauses;     /* n per class, even */
  int32_t margin;      /* T */
  double specificity;  /* s */
  int32_t state_depth; /* N */
  int32_t boost_true_positive;
  int32_t epochs;
  int32_t workers; /* 0 = hardware concurrency; recorded, see tmg_train_epoch */
  uint64_t seed;
} tmg_config;

/* EpochReport (trainer.hpp:31-43). feedback_events points to caller memory
 * of num_classes entries. */
typedef struct tmg_epoch_report {
  int32_t epoch;
  double seconds;        /* wall time of the epoch call */
  double device_seconds; /* CUDA-event time of the epoch's kernels */
  uint64_t* feedback_events;
  uint64_t* type_i_events; /* optional (may be NULL): Type I share, async mode */
} tmg_epoch_report;

typedef struct tmg_machine_info {
  int32_t feature_count, num_classes, clauses, state_depth;
  int32_t clause_begin, clause_end; /* this shard's slice of every class */
  int32_t planes;                   /* bit planes per automaton (B) */
  int32_t words_per_lane;           /* NW: 32-bit words per lane per part */
  int32_t bound_examples;           /* ClassBank::bound_examples (core.hpp:183) shared by every
                                       bank; -1 when the banks are bound to different counts */
  int32_t device;
  uint64_t device_bytes;
} tmg_machine_info;

int tmg_abi_version(void);
const char* tmg_last_error(void);
int tmg_device_count(int32_t* count);
/* Kernels launched by this library so far (process-wide counter). */
unsigned long long tmg_kernel_launches(void);
/* Device time of the last class-sum kernel of this machine (CUDA events
 * around the eval_bits_kernel launch alone: bench.py's inference roofline). */
int tmg_last_eval_kernel_ms(tmg_machine* tm, float* ms);
/* The CUDA stream (cudaStream_t) a machine's work runs on. */
int tmg_machine_stream(tmg_machine* tm, void** stream);
/* Statistical probe of the asynchronous Type I path (criterion
 * 1): applies it `trials` times to fresh copies of clause j of `bank` on one
 * literal row with the given clause output, counting per literal k (2o
 * entries, reference order) the +1 (inc) and -1 (dec) transitions. */
int tmg_debug_feedback_rates(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals,
                             int32_t clause_output, uint32_t trials, uint64_t* inc, uint64_t* dec);
/* One asynchronous Type I feedback (the epoch kernel's type_i_async: Philox
 * key of `epoch`, counters (global clause g = bank*clauses + j, example)) applied
 * in place to clause j of `bank` on one literal row (reference layout) with the
 * given clause output. Deterministic; register-resident shapes (feature_count
 * <= 4096) and the shared-memory path of wider rows. Replaces one call of
 * detail::type_i_with_output (feedback.cpp:32-70) under the async RNG. */
int tmg_debug_type_i_async(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals,
                           int32_t clause_output, uint32_t example, int32_t epoch);
/* Instrumentation counters of a TMG_STATS build (zeros otherwise): copies
 * `count` (<= 256) of them to `out`, then zeroes them if `reset`. */
int tmg_debug_counters(tmg_machine* tm, uint64_t* out, int32_t count, int32_t reset);
/* The async engine's alias table for the clause-output-0 Type I draw: 256
 * entries (threshold24 << 8 | alias) of the law of 8 independent literals
 * firing with probability threshold / 2^32 (host-side, no GPU needed). */
int tmg_alias8_table(uint32_t threshold, uint32_t* out);
/* Integer-pipe roofline probe: LOP3-only and LOP3+IMAD thread-ops per second. */
int tmg_bench_int_peak(int32_t device, double* lop3_ops_per_s, double* mixed_ops_per_s);
/* Host probe of the xoshiro256 jump-ahead used by the bit-exact replays
 * (train_epoch_sequential, W = 1): state <- M^k state, M the GF(2) matrix of
 * one state update of rng.hpp next(). Must equal k calls of next(). */
int tmg_debug_xoshiro_jump(uint64_t* state, uint64_t k);

/* Defaults of TMConfig (core.hpp:86-93). */
void tmg_config_default(tmg_config* cfg);
/* TMConfig::validate (core.cpp:48-74). */
int tmg_config_validate(const tmg_config* cfg);
/* effective_workers (core.cpp:76-80). */
int32_t tmg_effective_workers(const tmg_config* cfg);

/* ---- machine (MultiClassTM, trainer.cpp:89-100; ClassBank, core.cpp:82-105) */
int tmg_machine_create(const tmg_config* cfg, int32_t feature_count, int32_t num_classes,
                       int32_t device, tmg_machine** out);
/* Clause shard for multi-GPU: this machine holds clauses [clause_begin,
 * clause_end) of every class (even-aligned so polarity balance is kept). */
int tmg_machine_create_shard(const tmg_config* cfg, int32_t feature_count, int32_t num_classes,
                             int32_t device, int32_t clause_begin, int32_t clause_end,
                             tmg_machine** out);
int tmg_machine_destroy(tmg_machine* tm);
int tmg_machine_info_get(const tmg_machine* tm, tmg_machine_info* info);
int tmg_machine_config(const tmg_machine* tm, tmg_config* cfg);
/* Resets every automaton to N and clears previous outputs (fresh machine). */
int tmg_machine_reset(tmg_machine* tm);

/* ClassBank::counters / mutable_counters+rebuild_masks / set_counter
 * (core.hpp:126-133, 192-195; core.cpp:107-115,128-139). bank = class index;
 * out/in: n_shard x 2o uint16 in [1, 2N]. */
int tmg_get_counters(const tmg_machine* tm, int32_t bank, uint16_t* out);
int tmg_set_counters(tmg_machine* tm, int32_t bank, const uint16_t* in);
/* ClassBank::include_mask / include_count (core.hpp:147-156): n x W64 u64, n i32. */
int tmg_get_include_masks(const tmg_machine* tm, int32_t bank, uint64_t* out);
int tmg_get_include_counts(const tmg_machine* tm, int32_t bank, int32_t* out);
/* ClassBank::bind_examples (core.cpp:117-126) on every bank of the machine:
 * zeroes all previous outputs. */
int tmg_bind_examples(tmg_machine* tm, int64_t example_count);
/* ClassBank::bind_examples (core.cpp:117-126) on ONE bank: zeroes that bank's
 * previous outputs only; the other banks keep theirs. */
int tmg_bind_bank(tmg_machine* tm, int32_t bank, int64_t example_count);
/* ClassBank::bound_examples (core.hpp:183) of one bank. */
int tmg_bank_bound_examples(const tmg_machine* tm, int32_t bank, int64_t* example_count);
/* ClassBank::prev_output / set_prev_output (core.hpp:184-191):
 * n x ceil(bound/64) uint64 per bank (bound = that bank's bound_examples). */
int tmg_get_prev_outputs(const tmg_machine* tm, int32_t bank, uint64_t* out);
int tmg_set_prev_outputs(tmg_machine* tm, int32_t bank, const uint64_t* in);

/* ---- example pool (ExamplePool, pool.hpp:30-78; pool.cpp:23-80) */
/* bits: q x o uint8 in {0,1} (row-major), labels: q int32. Validation and
 * errors follow the ExamplePool constructor (pool.cpp:29-55). */
int tmg_pool_create(int32_t device, int32_t feature_count, const uint8_t* bits,
                    const int32_t* labels, int64_t q, int32_t num_classes, tmg_pool** out);
/* Same, from device pointers already resident on `device` (no host copy). */
int tmg_pool_create_device(int32_t device, int32_t feature_count, const uint8_t* d_bits,
                           const int32_t* d_labels, int64_t q, int32_t num_classes,
                           tmg_pool** out);
int tmg_pool_destroy(tmg_pool* pool);
int tmg_pool_size(const tmg_pool* pool, int64_t* q);
/* ExamplePool::literals (pool.hpp:43-48): q x ceil(2o/64) uint64. */
int tmg_pool_get_literals(const tmg_pool* pool, uint64_t* out);
/* ExamplePool::tally / set_tally / reset_tallies (pool.hpp:54-62): q x m int32. */
int tmg_pool_get_tallies(const tmg_pool* pool, int32_t* out);
int tmg_pool_set_tallies(tmg_pool* pool, const int32_t* in);
int tmg_pool_reset_tallies(tmg_pool* pool);
/* Device pointer of the q x m int32 tally array (for collectives / interop). */
int tmg_pool_tally_device_ptr(tmg_pool* pool, void** ptr);
/* Device pointer of the q x m int32 tally-delta buffer (multi-GPU windows). */
int tmg_pool_delta_device_ptr(tmg_pool* pool, void** ptr);
/* Multi-GPU over peer memory (replaces the window exchange
 * of the reference's shared atomic tallies, pool.hpp:66-69, across GPUs):
 * every rank keeps a full q x m tally replica, and the training kernels add
 * each tally change into the local replica AND, over NVLink, into every
 * peer's — the collective is fused into the clause kernel, no windows.
 * tmg_pool_tally_ipc_handle moves the replica to IPC-exportable memory (once)
 * and writes its 64-byte cudaIpcMemHandle_t; tmg_pool_set_peers opens the
 * other ranks' handles (npeers <= 7, concatenated 64-byte handles; 0
 * detaches). Callers reset every replica and barrier before an epoch, and
 * barrier after it. */
int tmg_pool_tally_ipc_handle(tmg_pool* pool, unsigned char* handle);
int tmg_pool_set_peers(tmg_pool* pool, const unsigned char* handles, int32_t npeers);

/* ---- training */
/* train_epoch_parallel (trainer.cpp:181-242).
 *   TMG_MODE_ASYNC: Algorithm 1 over every clause of the machine at once on
 *     the GPU (workers is recorded only; parallelism is the device's).
 *   TMG_MODE_SYNC_MIRROR: replays the reference's schedule for `workers`
 *     workers one after another with the reference xoshiro streams; for
 *     workers == 1 the result is bit-identical to the reference. */
int tmg_train_epoch(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                    tmg_epoch_report* report);
/* train_epoch_sequential (trainer.cpp:138-179): the classic trainer replayed
 * bit-exactly (one CTA; clause evaluation in parallel, the reference's single
 * xoshiro stream serial). feedback_events: num_classes entries. */
int tmg_train_epoch_sequential(tmg_machine* tm, tmg_pool* pool, int32_t epoch, double* seconds,
                               uint64_t* feedback_events);
/* ---- clause-sharded machines (the reference's W worker
 * threads sharing atomic tallies inside one train_epoch_parallel call,
 * trainer.cpp:210-231, pool.hpp:57-59, spread over GPUs).
 *
 * One process, several GPUs: tmg_machine_create_devices splits the clause
 * pairs of every class evenly over `devices` (repeats allowed: several shards
 * on one GPU). The handle is used like any machine: counters, include masks,
 * previous outputs, binding, tmg_train_epoch (TMG_MODE_ASYNC / AUTO),
 * tmg_refresh_tallies, class sums and predictions cover the whole machine;
 * calls that replay the reference's serial streams (sequential trainer,
 * update_clause, feedback, the W = 1 replay, regression) need one device and
 * fail with TMG_EINVAL. An epoch is one kernel launch per shard on its own
 * device; while they run, the shards' cumulative tally deltas are exchanged
 * about `windows` times per epoch (tmg_machine_set_windows, default 16) on
 * high-priority side streams: NCCL all-reduce when the devices are distinct
 * and libnccl.so.2 loads (TSETLIN_EXCHANGE=peer forces the other path), else
 * a peer-memory reduction kernel. Pools are replicated to the shards' devices
 * on first use. ndev == 1 creates a plain machine. */
int tmg_machine_create_devices(const tmg_config* cfg, int32_t o, int32_t m, const int32_t* devices, int32_t ndev,
                               tmg_machine** out);
/* Tally exchanges per epoch of a sharded machine (the interval adapts to the
 * previous epoch's length). */
int tmg_machine_set_windows(tmg_machine* tm, int32_t windows);
/* Tallies of the pool's replica for shard k of the last sharded machine that
 * used it (q x m int32; test hook: every replica holds the same tallies). */
int tmg_pool_replica_tallies(const tmg_pool* pool, int32_t k, int32_t* out);
/* shards held (group) or ranks (communicator); whether the exchange uses NCCL. */
int tmg_machine_exchange_info(const tmg_machine* tm, int32_t* shards, int32_t* uses_nccl);
/* 1 when libnccl.so.2 could be loaded; else 0 and the reason in `why`. */
int tmg_nccl_available(char* why, int32_t len);
/* One process per GPU: rank 0 makes a 128-byte NCCL id, the caller sends it
 * to every rank, each rank creates its communicator on its device and
 * attaches it to its shard (tmg_machine_create_shard with the even-aligned
 * slice of its rank). tmg_train_epoch then trains this rank's clauses with
 * the streaming tally exchange over NCCL and reports every rank's feedback events;
 * tmg_class_sums / tmg_predict / tmg_refresh_tallies return whole-machine
 * results on every rank. These calls are collective: every rank makes them
 * in the same order with the same arguments. Attach NULL to detach. */
typedef struct tmg_comm tmg_comm;
int tmg_comm_unique_id(unsigned char* id128);
int tmg_comm_create(const unsigned char* id128, int32_t nranks, int32_t rank, int32_t device, tmg_comm** out);
int tmg_comm_destroy(tmg_comm* comm);
/* The same without NCCL, over CUDA IPC (one node): every rank maps the
 * others' snapshot slots and pulls them with the copy engine (NVLink), so no
 * exchange kernel needs to be co-scheduled across ranks. Create with the
 * largest q x m any pool of the machine will have, export the 192-byte
 * handle, gather every rank's handles (rank order, nranks x 192 bytes) over
 * your transport, connect, attach. */
int tmg_comm_create_ipc(int32_t nranks, int32_t rank, int32_t device, int64_t capacity, tmg_comm** out);
int tmg_comm_ipc_handle(tmg_comm* comm, unsigned char* handle192);
int tmg_comm_ipc_connect(tmg_comm* comm, const unsigned char* handles);
int tmg_machine_attach_comm(tmg_machine* tm, tmg_comm* comm);

/* Multi-GPU building blocks: one asynchronous window [t_begin, t_end) of every
 * clause's pass of `epoch`. Deltas are also accumulated in the pool's delta
 * buffer; after an allreduce of that buffer call tmg_pool_apply_reduced. */
int tmg_train_window(tmg_machine* tm, tmg_pool* pool, int32_t epoch, int64_t t_begin,
                     int64_t t_end, uint64_t* feedback_events);
int tmg_epoch_begin(tmg_machine* tm, tmg_pool* pool, int32_t epoch);
/* tallies += reduced - own_delta; own_delta = 0. d_reduced: q x m int32 on device. */
int tmg_pool_apply_reduced(tmg_pool* pool, const void* d_reduced);
/* Overlapped windows (double-buffered exchange). All three
 * only ENQUEUE on the machine's stream (tmg_machine_stream) and return:
 *   tmg_train_window_async     one window, events accumulate since tmg_epoch_begin;
 *   tmg_window_delta_snapshot  d_snapshot = own delta, own delta = 0;
 *   tmg_window_apply_remote    tallies += d_reduced - d_snapshot (the remote share
 *                              of an earlier window, once its all-reduce is done).
 * tmg_epoch_events synchronises the stream and reads the per-class events. */
int tmg_train_window_async(tmg_machine* tm, tmg_pool* pool, int32_t epoch, int64_t t_begin, int64_t t_end);
int tmg_window_delta_snapshot(tmg_machine* tm, tmg_pool* pool, void* d_snapshot);
int tmg_window_apply_remote(tmg_machine* tm, tmg_pool* pool, const void* d_reduced, const void* d_snapshot);
int tmg_epoch_events(tmg_machine* tm, uint64_t* feedback_events);
/* update_clause (trainer.cpp:102-136) with the reference stream: rng_state is
 * the 4-word xoshiro256++ state, advanced in place. order may be NULL (natural
 * order) or hold order_len == q indices. */
int tmg_update_clause(tmg_machine* tm, tmg_pool* pool, int32_t class_idx, int32_t j,
                      const int32_t* order, int64_t order_len, int64_t offset, int64_t batch,
                      int32_t margin, double s, int32_t boost, uint64_t* rng_state,
                      uint64_t* events);

/* type_i_feedback / type_ii_feedback (feedback.cpp:87-99) on clause j of
 * `bank` for one reference-layout literal row: type 1 = Type I (draws 2o
 * uniforms from rng_state, advanced in place), type 2 = Type II.
 * clause_output: -1 evaluates the clause first (type_i/ii_feedback);
 * 0 or 1 uses the given output (detail::type_i/ii_with_output,
 * feedback.cpp:32-83). */
int tmg_feedback(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals, int32_t type,
                 double s, int32_t boost, int32_t clause_output, uint64_t* rng_state);
/* evaluate_clause (core.hpp:208-219) of clause j of `bank` on one
 * reference-layout literal row; mode TMG_EVAL_TRAIN / TMG_EVAL_PREDICT. */
int tmg_evaluate_clause(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals,
                        int32_t mode, int32_t* out);

/* ---- inference */
/* refresh_tallies (pool.cpp:108-124): exact Train-mode sums + prev outputs. */
int tmg_refresh_tallies(tmg_machine* tm, tmg_pool* pool);
/* export_vote_sums (trainer.cpp:262-270) for every pool example: q x m int32. */
int tmg_class_sums(tmg_machine* tm, const tmg_pool* pool, int32_t mode, int32_t* out);
/* predict_all (trainer.cpp:272-279): q int32. */
int tmg_predict(tmg_machine* tm, const tmg_pool* pool, int32_t* out);
/* vote sums / classify on arbitrary reference-layout literal rows
 * (q x ceil(2o/64) uint64): vote_sum (pool.cpp:82-91), classify
 * (trainer.cpp:244-260). */
int tmg_class_sums_literals(tmg_machine* tm, const uint64_t* literals, int64_t q, int32_t mode,
                            int32_t* out);
int tmg_predict_literals(tmg_machine* tm, const uint64_t* literals, int64_t q, int32_t* out);
/* Device-resident variant for benchmarking: d_sums q x m int32 on device. */
int tmg_class_sums_device(tmg_machine* tm, const tmg_pool* pool, int32_t mode, int32_t* d_sums);

/* ---- regression head (proj/include/tsetlin/regression.hpp) */
/* RegressionHead ctor (regression.cpp:69-80): one all-positive bank of
 * cfg->clauses clauses. Pools for it have num_classes == 1 and hold scaled
 * integer targets t in [0, T] as labels (scaled_target, regression.cpp:82-89). */
int tmg_machine_create_regress(const tmg_config* cfg, int32_t feature_count, int32_t device,
                               tmg_machine** out);
/* train_epoch_regress_parallel (regression.cpp:163-227): TMG_MODE_ASYNC (all
 * clauses concurrently) or TMG_MODE_SYNC_MIRROR (the reference's W-worker
 * schedule and streams; bit-exact for W = 1). feedback_events: 1 entry. */
int tmg_train_epoch_regress(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers,
                            int32_t epoch, tmg_epoch_report* report);
/* train_epoch_regress_sequential (regression.cpp:125-161), bit-exact. */
int tmg_train_epoch_regress_sequential(tmg_machine* tm, tmg_pool* pool, int32_t epoch,
                                       double* seconds, uint64_t* feedback_events);
/* predict_scaled (regression.cpp:86-93): clause count clipped to [0, T], per
 * pool example or per reference-layout literal row. */
int tmg_regress_predict(tmg_machine* tm, const tmg_pool* pool, int32_t* out);
int tmg_regress_predict_literals(tmg_machine* tm, const uint64_t* literals, int64_t q, int32_t* out);
/* update_regress (regression.cpp:101-123) with a scaled target and the
 * caller's xoshiro stream (advanced in place). */
int tmg_update_regress(tmg_machine* tm, const uint64_t* literals, int32_t scaled_target,
                       uint64_t* rng_state, uint64_t* events);

/* ---- host-side RNG streams (tmgpu_rng.h), exported for FFI users */
/* Rng(seed, stream) (rng.hpp:39-42) -> 4-word xoshiro256++ state. */
void tmg_rng_state_init(uint64_t seed, uint64_t stream, uint64_t* state);
/* Rng::next (rng.hpp:44-54) on a 4-word state. */
uint64_t tmg_rng_state_next(uint64_t* state);
/* The epoch permutation of train_epoch_parallel (trainer.cpp:196-198). */
int tmg_epoch_order(uint64_t seed, int32_t epoch, int32_t q, int32_t* order);

/* ---- synthetic data (csrc/synth.c) */
int tmg_synth_xor(uint64_t seed, int64_t rows, int features, double noise, int with_noise,
                  uint8_t* bits, int32_t* labels);
int tmg_synth_mnist(uint64_t seed, int features, int classes, double r_class, double r_sub,
                    double flip, int64_t train_rows, int64_t test_rows, uint8_t* train_bits,
                    int32_t* train_labels, uint8_t* test_bits, int32_t* test_labels);
int tmg_synth_fmnist(uint64_t seed, int pixels, int classes, double r_class, double r_sub, int amp,
                     double mix, int64_t train_rows, int64_t test_rows, uint8_t* train_bits,
                     int32_t* train_labels, uint8_t* test_bits, int32_t* test_labels);
int tmg_synth_imdb(uint64_t seed, int vocab, int sentiment, double p_sent, double cross,
                   int64_t train_rows, int64_t test_rows, uint8_t* train_bits,
                   int32_t* train_labels, uint8_t* test_bits, int32_t* test_labels);
/* The canonical BASELINE.json datasets: kind 0 XOR12, 1 MNIST-, 2 FMNIST-,
 * 3 IMDb-shaped (features 12, 784, 2352, 10000). */
int tmg_synth_preset(int kind, uint64_t seed, double noise, int64_t train_rows, int64_t test_rows,
                     uint8_t* train_bits, int32_t* train_labels, uint8_t* test_bits,
                     int32_t* test_labels);

#ifdef __cplusplus
}
#endif

#endif /* TMGPU_H_ */
