// engine.h — internal host-side types of the engine (not part of the ABI):
// error plumbing, device buffers, the machine and pool objects behind the
// opaque handles of include/tmgpu.h, and the helpers the ABI translation
// units share (engine.cu: single-device machines; group.cu: clause shards
// over several devices / processes).
#pragma once

#include <atomic>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include "kernels.h"
#include "tmgpu.h"

#define TMG_API extern "C" __attribute__((visibility("default")))

namespace tmgx {

struct Error {
  int code;
  std::string msg;
};

extern thread_local std::string g_last_error;

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TMG_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TMG_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return TMG_ERUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TMG_ERUNTIME;
  }
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Keeps the current device's default memory pool from returning freed memory
// to the driver at every synchronisation (once per device).
void pool_init();

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  // Device memory comes from the device's stream-ordered pool, which keeps
  // freed blocks mapped (release threshold raised in pool_init): creating and
  // dropping example pools per call stays cheap. alloc/release keep
  // cudaMalloc/cudaFree's synchronous semantics.
  void alloc(size_t n) {
    release();
    if (n) {
      pool_init();
      CK(cudaMallocAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T), cudaStreamPerThread));
      CK(cudaStreamSynchronize(cudaStreamPerThread));
    }
    count = n;
  }
  // Plain cudaMalloc memory instead (IPC-exportable: the stream-ordered
  // pool's blocks cannot be shared with cudaIpcGetMemHandle).
  void alloc_plain(size_t n) {
    release();
    if (n) CK(cudaMalloc(reinterpret_cast<void**>(&ptr), n * sizeof(T)));
    count = n;
    plain = n != 0;
  }
  void release() {
    if (ptr) {
      cudaDeviceSynchronize();
      if (plain) {
        cudaFree(ptr);
      } else {
        cudaFreeAsync(ptr, cudaStreamPerThread);
        cudaStreamSynchronize(cudaStreamPerThread);
      }
    }
    ptr = nullptr;
    count = 0;
    plain = false;
  }
  void swap(DevBuf& o) {
    std::swap(ptr, o.ptr);
    std::swap(count, o.count);
    std::swap(plain, o.plain);
  }
  bool plain = false;
  size_t bytes() const { return count * sizeof(T); }
};

struct Exchange;  // group.cu: the tally exchange of a sharded machine

}  // namespace tmgx

struct tmg_pool {
  int device = 0;
  int o = 0, m = 0, Wp = 0;
  int64_t q = 0;
  cudaStream_t stream = nullptr;
  tmgx::DevBuf<uint32_t> rows;  // [q][2][Wp]: x-plane words, then !x-plane words
  uint32_t* xplane() const { return rows.ptr; }
  uint32_t* nplane() const { return rows.ptr + Wp; }
  tmgx::DevBuf<int32_t> labels, tallies, delta, order;
  // Feature-major example columns for evaluation (eval.cu), built on first
  // use: the rows never change after creation.
  mutable tmgx::DevBuf<uint32_t> lit_t;
  std::vector<int32_t> host_labels;
  // Tally replicas of the other ranks (multi-GPU over peer memory): every
  // tally change is also added into each of them by the training kernels.
  std::vector<int32_t*> peers;
  // Sharded machines (group.cu): one tally replica per shard (replicas[k]
  // may be this pool itself); a replica points back at its primary.
  std::vector<tmg_pool*> replicas;
  tmg_pool* primary = nullptr;
  void close_peers() {
    for (int32_t* p : peers) cudaIpcCloseMemHandle(p);
    peers.clear();
  }
};

struct tmg_machine {
  tmg_config cfg{};
  int o = 0, m = 0, n = 0, j_begin = 0, j_end = 0, n_loc = 0;
  int N = 0, B = 0, NW = 0, Wx = 0, Wp = 0, Wq = 0;
  int device = 0;
  int64_t q_bound = 0;          // examples every bank is bound to, -1 when the banks differ
  std::vector<int64_t> bank_q;  // per bank (ClassBank::bound_examples); prev stride Wq covers the largest
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t eval0 = nullptr, eval1 = nullptr;  // around the last class-sum kernel
  tmgx::DevBuf<uint32_t> state, prev;
  tmgx::DevBuf<int32_t> inc_count, lens, npos, sums;
  tmgx::DevBuf<int64_t> offs;      // [clauses + 1] literal-list offsets
  tmgx::DevBuf<int4> meta;         // [clauses] eval list descriptors
  tmgx::DevBuf<uint32_t> lists;    // included-literal lists (eval.cu)
  tmgx::DevBuf<uint32_t> lit_t;    // scratch: feature-major example columns of non-pool rows
  tmgx::DevBuf<unsigned long long> events;
  tmgx::DevBuf<unsigned long long> dbg;  // instrumentation counters (TMG_STATS builds)
  tmgx::DevBuf<int32_t> work;            // clause counter of the persistent shared-memory kernel
  tmgx::DevBuf<uint32_t> alias8;         // alias table of the clause-output-0 Type I draw
  tmgx::DevBuf<uint16_t> scratch16;
  // sequential-trainer jump matrices (M^chunk, M^(2o)) and per-clause states
  tmgx::DevBuf<uint32_t> seq_jump;
  tmgx::DevBuf<uint64_t> seq_tstate;
  tmgx::DevBuf<uint32_t> seq_scratch;  // grid-wide replay: output / gated bits, votes, negative class
  bool entries_dirty = true;
  int64_t lists_total = 0;  // padded included-literal list entries over all clauses
  // current async epoch
  int32_t cur_epoch = -1;
  uint32_t key0 = 0, key1 = 0;
  int all_positive = 0;  // regression head bank (PolarityScheme::AllPositive)
  bool regress_mode = false;  // current call trains the regression head
  // Sharded machine (group.cu): clause shards on devices of this process
  // (parts non-empty: this handle owns no device state itself), or a shard
  // of a multi-process machine attached to a communicator (xchg, parts empty).
  std::vector<tmg_machine*> parts;
  tmgx::Exchange* xchg = nullptr;
  bool owns_xchg = false;
  int windows = 16;  // tally-exchange windows per sharded epoch
  int clauses() const { return m * n_loc; }
};

namespace tmgx {

// engine.cu
void validate_config(const tmg_config& c);
void check_compatible(const tmg_machine* tm, const tmg_pool* pool);
void bind(tmg_machine* tm, int64_t q);
void bind_bank(tmg_machine* tm, int c, int64_t q);
void bind_for(tmg_machine* tm, int64_t q);
void rebuild_entries(tmg_machine* tm);
void reset_state(tmg_machine* tm);
tmg_machine* create_machine(const tmg_config* cfg, int o, int m, int device, int jb, int je, int all_positive = 0);
void upload_order(tmg_machine* tm, tmg_pool* pool, int32_t epoch);
void epoch_keys(tmg_machine* tm, int32_t epoch);
// Steps [t0, t1) of every clause's pass — of the clause-order warps
// [w_begin, w_end) only when w_end >= 0 (one wave of a sharded epoch).
void run_async_window(tmg_machine* tm, tmg_pool* pool, int64_t t0, int64_t t1, bool with_delta, int w_begin = 0,
                      int w_end = -1);
// Clause warps one launch keeps resident on tm's device, and the CTA width.
int resident_clause_warps(tmg_machine* tm, tmg_pool* pool, int* warps_per_cta);
void class_sums_device(tmg_machine* tm, const uint32_t* xplane, int64_t q, bool train_mode, int32_t* d_out,
                       uint32_t* prev, const uint32_t* lit_t = nullptr);
const uint32_t* pool_lit_t(tmg_machine* tm, const tmg_pool* pool);
void literals_to_planes(tmg_machine* tm, const uint64_t* lits, int64_t q, DevBuf<uint32_t>& xs);
tmg_pool* create_pool_common(int device, int o, int64_t q, int m);
int32_t resolve_mode(int32_t mode, int32_t workers);

// group.cu — sharded machines. The group_* entry points implement the ABI
// call of the same name for a machine with parts (or an attached comm).
inline bool is_group(const tmg_machine* tm) { return tm && !tm->parts.empty(); }
inline bool is_sharded(const tmg_machine* tm) { return tm && (!tm->parts.empty() || tm->xchg); }
void need_single(const tmg_machine* tm, const char* what);
void destroy_group(tmg_machine* tm);
void destroy_replicas(tmg_pool* pool);
int group_info(const tmg_machine* tm, tmg_machine_info* info);
int group_reset(tmg_machine* tm);
int group_counters(const tmg_machine* tm, int32_t bank, uint16_t* out, const uint16_t* in);
int group_include(const tmg_machine* tm, int32_t bank, uint64_t* masks, int32_t* counts);
int group_bind(tmg_machine* tm, int32_t bank, int64_t q);  // bank < 0: every bank
int group_prev(const tmg_machine* tm, int32_t bank, uint64_t* out, const uint64_t* in);
tmg_machine* group_owner(const tmg_machine* tm, int32_t j);  // shard holding clause j, or null
int group_update_clause(tmg_machine* tm, tmg_pool* pool, int32_t c, int32_t j, const int32_t* order,
                        int64_t order_len, int64_t offset, int64_t batch, int32_t margin, double s, int32_t boost,
                        uint64_t* rng_state, uint64_t* events);
int group_train_epoch(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                      tmg_epoch_report* report);
// Class sums over every shard into host memory (train mode also refreshes
// the shards' previous outputs and, with set_tallies, the pool's tallies).
int group_class_sums(tmg_machine* tm, const tmg_pool* pool, const uint64_t* lits, int64_t q, int32_t mode,
                     int32_t* out, bool set_tallies);

}  // namespace tmgx
