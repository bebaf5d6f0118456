// group.cu — clause-sharded machines over several GPUs.
//
// The reference runs all of its parallelism inside one call,
// train_epoch_parallel(tm, pool, workers, epoch) (trainer.cpp:181-242): W
// threads update disjoint clauses and share the q x m tallies through
// relaxed atomics (pool.hpp:57-59, pool.cpp:93-106). Here the clause pairs of
// every class are split over GPUs; each shard's epoch is one kernel launch
// over its clauses that updates its own tally replica and a cumulative delta
// buffer, and while the kernels run, a host loop on high-priority side streams
// exchanges the deltas (sharded_epoch): every other shard's changes reach a
// replica one exchange interval (~1/16 of an epoch) after they happen — the
// same relaxed, lock-free tally semantics as the reference's threads.
//
// Two ways to hold the shards:
//   * one process, several devices (tmg_machine_create_devices; the C++
//     facade with $TSETLIN_DEVICES): the handle owns one shard per listed
//     device and the sum is an NCCL all-reduce over the devices
//     (ncclCommInitAll), or — for repeated devices or when NCCL cannot be
//     loaded — a peer-memory reduction kernel that reads every shard's
//     snapshot directly (same device or P2P over NVLink);
//   * one process per GPU (tmg_comm_create + tmg_machine_attach_comm): each
//     rank's shard sums over NCCL (ncclCommInitRank).
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy the process
// already loaded, e.g. torch's, else the system's), so the library loads and
// runs single-GPU without it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

#include "engine.h"

struct tmg_comm {
  tmgx::Exchange* x = nullptr;
};

namespace tmgx {

// ------------------------------------------------------------------ NCCL ---
struct Nccl {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (n.tried) return n;
  n.tried = true;
  // The copy the process already has (torch's, when torch is imported) —
  // loading a second, older libnccl.so.2 first would make the later
  // libtorch_cuda.so bind to it by SONAME and fail on newer symbols. Else
  // $TMG_NCCL_LIB (the Python package points it at the NCCL wheel torch
  // uses), else the system's.
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  const char* env = std::getenv("TMG_NCCL_LIB");
  if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    n.why = e ? e : "dlopen(libnccl.so.2) failed";
    return n;
  }
  auto sym = [&](auto& fn, const char* name) {
    fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
    if (!fn && n.why.empty()) n.why = std::string("libnccl.so.2 lacks ") + name;
  };
  sym(n.GetUniqueId, "ncclGetUniqueId");
  sym(n.CommInitRank, "ncclCommInitRank");
  sym(n.CommInitAll, "ncclCommInitAll");
  sym(n.CommDestroy, "ncclCommDestroy");
  sym(n.AllReduce, "ncclAllReduce");
  sym(n.GroupStart, "ncclGroupStart");
  sym(n.GroupEnd, "ncclGroupEnd");
  sym(n.GetErrorString, "ncclGetErrorString");
  n.ok = n.why.empty();
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(TMG_ERUNTIME, std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

// ------------------------------------------------------------- exchange ---
struct PeerSrc {
  const int32_t* p[16];
  int32_t n;
};

__global__ void peer_sum_kernel(int32_t* __restrict__ out, PeerSrc s, int64_t count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int32_t v = 0;
    for (int j = 0; j < s.n; ++j) v += __ldcg(s.p[j] + i);
    out[i] = v;
  }
}

// tallies += (other shards' deltas since the last exchange) =
// (sum_new - sum_prev) - (own_new - own_prev), atomically: the epoch kernel
// is adding to the same tallies meanwhile.
__global__ void stream_apply_kernel(int32_t* __restrict__ tallies, const int32_t* __restrict__ red_new,
                                    const int32_t* __restrict__ red_prev, const int32_t* __restrict__ own_new,
                                    const int32_t* __restrict__ own_prev, int64_t count) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = (red_new[i] - red_prev[i]) - (own_new[i] - own_prev[i]);
    if (v) atomicAdd(tallies + i, v);
  }
}

struct Exchange {
  bool use_nccl = false;
  int nranks = 1, rank = 0;           // processes (tmg_comm); 1 for a one-process group
  std::vector<int> devices;           // one per shard held by this process
  std::vector<ncclComm_t> comms;      // use_nccl: one per local shard
  std::vector<cudaStream_t> cstreams;  // side stream per local shard
  struct Slot {
    // snap[b]: the shard's cumulative tally deltas of this epoch as copied at
    // exchange b, plus one trailing element: 1 once the shard's kernel has
    // finished; red[b]: its sum over every shard
    DevBuf<int32_t> snap[2], red[2];
    cudaEvent_t snap_ev[2] = {nullptr, nullptr}, red_ev[2] = {nullptr, nullptr};
    cudaEvent_t done = nullptr;  // the shard's epoch kernel finished
    int32_t* flag = nullptr;     // pinned host: [0] done flag to send, [1] reduced done count
  };
  std::vector<std::unique_ptr<Slot>> slots;
  int64_t count = 0;
  double interval_s = 0.002;  // time between exchanges (adapted to the epoch length)
  // IPC mode (one process per GPU, no NCCL): every rank's snapshot slots and
  // control words are mapped into every other rank (CUDA IPC over NVLink);
  // each rank PULLS the others' snapshots with the copy engine and sums
  // locally, so no exchange kernel has to be co-scheduled across ranks.
  // ctl = [ready seq of slot 0, 1][consumed seq: slot 0 by rank 0..N-1][slot 1 by 0..N-1]
  bool use_ipc = false;
  int64_t seq = 0;                         // exchange sequence number, identical on every rank
  int64_t ipc_count = 0;                   // capacity of the exported snapshot slots
  DevBuf<int64_t> ctl;
  std::vector<int32_t*> peer_snap[2];      // [slot][rank] (own rank: null)
  std::vector<int64_t*> peer_ctl;          // [rank]
  std::vector<std::unique_ptr<DevBuf<int32_t>>> recv;  // [rank] pulled snapshots
  cudaStream_t pstream = nullptr;          // polling copies
  int64_t* hpoll = nullptr;                // pinned host words for polling / flag writes
  DevBuf<unsigned long long> scratch64;  // cross-rank event / sum reductions
  DevBuf<int32_t> scratch32;

  void init_streams() {
    for (size_t k = slots.size(); k < devices.size(); ++k) slots.push_back(std::make_unique<Slot>());
    cstreams.resize(devices.size());
    for (size_t k = 0; k < devices.size(); ++k) {
      DeviceGuard dg(devices[k]);
      // the exchange's copies, sums and applies run beside the epoch kernel,
      // which fills every SM: the highest priority puts them on the next free slot
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&cstreams[k], cudaStreamNonBlocking, hi));
      for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&slots[k]->snap_ev[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&slots[k]->red_ev[b], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&slots[k]->done, cudaEventDisableTiming));
      CK(cudaMallocHost(reinterpret_cast<void**>(&slots[k]->flag), 2 * sizeof(int32_t)));
      // Load the exchange's kernels now: with lazy module loading a first
      // launch beside a running epoch kernel would wait for the device to
      // drain, i.e. the first epoch's exchanges would all happen at its end.
      cudaFuncAttributes attr;
      CK(cudaFuncGetAttributes(&attr, peer_sum_kernel));
      CK(cudaFuncGetAttributes(&attr, stream_apply_kernel));
    }
  }

  void ensure(int64_t n) {
    if (n == count) return;
    if (use_ipc) {  // slots were exported with their capacity; only the count used changes
      if (n > ipc_count) fail(TMG_EINVAL, "pool larger than the IPC communicator's exported capacity");
      count = n;
      return;
    }
    for (size_t k = 0; k < devices.size(); ++k) {
      DeviceGuard dg(devices[k]);
      for (int b = 0; b < 2; ++b) {  // plain cudaMalloc: peer-accessible (stream-ordered pools are not)
        slots[k]->snap[b].alloc_plain(static_cast<size_t>(n));
        slots[k]->red[b].alloc_plain(static_cast<size_t>(n));
      }
    }
    count = n;
  }

  ~Exchange() {
    if (use_ipc && !devices.empty()) {
      cudaSetDevice(devices[0]);
      for (int b = 0; b < 2; ++b)
        for (int32_t* p : peer_snap[b])
          if (p) cudaIpcCloseMemHandle(p);
      for (int64_t* p : peer_ctl)
        if (p) cudaIpcCloseMemHandle(p);
      if (pstream) cudaStreamDestroy(pstream);
      if (hpoll) cudaFreeHost(hpoll);
    }
    for (size_t k = 0; k < devices.size(); ++k) {
      cudaSetDevice(devices[k]);
      if (k < cstreams.size() && cstreams[k]) cudaStreamSynchronize(cstreams[k]);
      if (k < slots.size())
        for (int b = 0; b < 2; ++b) {
          slots[k]->snap[b].release();
          slots[k]->red[b].release();
          if (slots[k]->snap_ev[b]) cudaEventDestroy(slots[k]->snap_ev[b]);
          if (slots[k]->red_ev[b]) cudaEventDestroy(slots[k]->red_ev[b]);
        }
      if (k < slots.size() && slots[k]->done) cudaEventDestroy(slots[k]->done);
      if (k < slots.size() && slots[k]->flag) cudaFreeHost(slots[k]->flag);
      if (k < comms.size() && comms[k] && nccl().CommDestroy) nccl().CommDestroy(comms[k]);
      if (k < cstreams.size() && cstreams[k]) cudaStreamDestroy(cstreams[k]);
    }
  }

  // Sum of the shards' snapshot b (all local shards and, with NCCL, all
  // ranks) into every local shard's red[b]; red_ev[b] marks completion.
  // Host-side poll of a device word (own or peer-mapped) until pred holds.
  template <typename Pred>
  void poll(const int64_t* dptr, Pred&& pred) {
    for (;;) {
      CK(cudaMemcpyAsync(hpoll, dptr, sizeof(int64_t), cudaMemcpyDeviceToHost, pstream));
      CK(cudaStreamSynchronize(pstream));
      if (pred(hpoll[0])) return;
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }

  // IPC exchange of slot b with sequence number sq (the snapshot is already
  // enqueued on cstreams[0]): publish ready, pull every other rank's
  // snapshot once it is ready, tell it so, sum locally.
  void reduce_ipc(int b, int64_t sq) {
    DeviceGuard dg(devices[0]);
    cudaStream_t cs = cstreams[0];
    int64_t* words = hpoll + 1;  // [1] = sq for the flag writes
    words[0] = sq;
    CK(cudaMemcpyAsync(ctl.ptr + b, words, sizeof(int64_t), cudaMemcpyHostToDevice, cs));  // ready[b] = sq
    PeerSrc src{};
    src.n = 0;
    src.p[src.n++] = slots[0]->snap[b].ptr;
    for (int j = 0; j < nranks; ++j) {
      if (j == rank) continue;
      poll(peer_ctl[j] + b, [&](int64_t v) { return v == sq; });
      CK(cudaMemcpyAsync(recv[j]->ptr, peer_snap[b][j], static_cast<size_t>(count) * 4, cudaMemcpyDeviceToDevice,
                         cs));
      CK(cudaMemcpyAsync(peer_ctl[j] + 2 + b * nranks + rank, words, sizeof(int64_t), cudaMemcpyHostToDevice, cs));
      src.p[src.n++] = recv[j]->ptr;
    }
    tmg::count_launch();
    peer_sum_kernel<<<64, 256, 0, cs>>>(slots[0]->red[b].ptr, src, count);
    CK(cudaGetLastError());
    CK(cudaEventRecord(slots[0]->red_ev[b], cs));
    CK(cudaStreamSynchronize(cs));  // the flag words in hpoll are reused by the next exchange
  }

  // IPC: before overwriting own slot b, every other rank has pulled the
  // snapshot it held (sequence number >= sq).
  void wait_consumed(int b, int64_t sq) {
    DeviceGuard dg(devices[0]);
    for (int j = 0; j < nranks; ++j)
      if (j != rank) poll(ctl.ptr + 2 + b * nranks + j, [&](int64_t v) { return v >= sq; });
  }

  void reduce(int b) {
    const size_t n = devices.size();
    if (use_nccl) {
      for (size_t k = 0; k < n; ++k) {
        DeviceGuard dg(devices[k]);
        CK(cudaStreamWaitEvent(cstreams[k], slots[k]->snap_ev[b], 0));
      }
      nccl_check(nccl().GroupStart(), "ncclGroupStart");
      for (size_t k = 0; k < n; ++k)
        nccl_check(nccl().AllReduce(slots[k]->snap[b].ptr, slots[k]->red[b].ptr, static_cast<size_t>(count),
                                    ncclInt32, ncclSum, comms[k], cstreams[k]),
                   "ncclAllReduce");
      nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
      for (size_t k = 0; k < n; ++k) {
        DeviceGuard dg(devices[k]);
        CK(cudaEventRecord(slots[k]->red_ev[b], cstreams[k]));
      }
      return;
    }
    PeerSrc src{};
    src.n = static_cast<int32_t>(n);
    for (size_t j = 0; j < n; ++j) src.p[j] = slots[j]->snap[b].ptr;
    for (size_t k = 0; k < n; ++k) {
      DeviceGuard dg(devices[k]);
      for (size_t j = 0; j < n; ++j) CK(cudaStreamWaitEvent(cstreams[k], slots[j]->snap_ev[b], 0));
      tmg::count_launch();
      peer_sum_kernel<<<296, 256, 0, cstreams[k]>>>(slots[k]->red[b].ptr, src, count);
      CK(cudaGetLastError());
      CK(cudaEventRecord(slots[k]->red_ev[b], cstreams[k]));
    }
  }

  // Host-side sum over ranks through the IPC slots (events, class sums):
  // each value split into int32 words in own slot 0, one exchange round.
  template <typename T>
  void allreduce_host_ipc(T* v, size_t n) {
    const size_t words = n * sizeof(T) / 4;
    if (static_cast<int64_t>(words) > ipc_count) fail(TMG_EINVAL, "host all-reduce larger than the IPC slots");
    DeviceGuard dg(devices[0]);
    const int64_t sq = seq++;
    const int b = static_cast<int>(sq & 1);
    wait_consumed(b, sq - 2);
    std::vector<uint32_t> lo(words);
    std::memcpy(lo.data(), v, words * 4);
    const int64_t keep = count;
    count = static_cast<int64_t>(words);
    CK(cudaMemcpyAsync(slots[0]->snap[b].ptr, lo.data(), words * 4, cudaMemcpyHostToDevice, cstreams[0]));
    // pull the raw words of every rank and add on the host (exact for uint64 too)
    DeviceGuard dg2(devices[0]);
    int64_t* w = hpoll + 1;
    w[0] = sq;
    CK(cudaMemcpyAsync(ctl.ptr + b, w, sizeof(int64_t), cudaMemcpyHostToDevice, cstreams[0]));
    CK(cudaStreamSynchronize(cstreams[0]));
    std::vector<T> acc(v, v + n), part(n);
    for (int j = 0; j < nranks; ++j) {
      if (j == rank) continue;
      poll(peer_ctl[j] + b, [&](int64_t x) { return x == sq; });
      CK(cudaMemcpyAsync(part.data(), peer_snap[b][j], words * 4, cudaMemcpyDeviceToHost, cstreams[0]));
      CK(cudaMemcpyAsync(peer_ctl[j] + 2 + b * nranks + rank, w, sizeof(int64_t), cudaMemcpyHostToDevice,
                         cstreams[0]));
      CK(cudaStreamSynchronize(cstreams[0]));
      for (size_t i = 0; i < n; ++i) acc[i] += part[i];
    }
    std::memcpy(v, acc.data(), n * sizeof(T));
    count = keep;
    wait_consumed(b, sq);
  }

  // Before shard k touches snapshot b again: its own sum is done and (peer
  // mode) so is every other shard's read of its snapshot.
  void wait_reduced(size_t k, int b, cudaStream_t s) {
    if (use_nccl) {
      CK(cudaStreamWaitEvent(s, slots[k]->red_ev[b], 0));
      return;
    }
    for (size_t j = 0; j < devices.size(); ++j) CK(cudaStreamWaitEvent(s, slots[j]->red_ev[b], 0));
  }

  // Host-side sum over ranks (multi-process); identity for one process.
  template <typename T>
  void allreduce_host(T* v, size_t n) {
    if (nranks == 1) return;
    if (use_ipc) return allreduce_host_ipc(v, n);
    static_assert(sizeof(T) == 4 || sizeof(T) == 8, "int32 / uint64 only");
    DeviceGuard dg(devices[0]);
    void* d = nullptr;
    if (sizeof(T) == 8) {
      if (scratch64.count < n) scratch64.alloc(n);
      d = scratch64.ptr;
    } else {
      if (scratch32.count < n) scratch32.alloc(n);
      d = scratch32.ptr;
    }
    CK(cudaMemcpyAsync(d, v, n * sizeof(T), cudaMemcpyHostToDevice, cstreams[0]));
    nccl_check(nccl().AllReduce(d, d, n, sizeof(T) == 8 ? ncclUint64 : ncclInt32, ncclSum, comms[0], cstreams[0]),
               "ncclAllReduce");
    CK(cudaMemcpyAsync(v, d, n * sizeof(T), cudaMemcpyDeviceToHost, cstreams[0]));
    CK(cudaStreamSynchronize(cstreams[0]));
  }
};

// Even-aligned slice of n clauses for shard k of s (pairs are never split,
// so each shard keeps the alternating polarity; distributed.shard_range).
std::pair<int, int> shard_range(int n, int k, int s) {
  const int pairs = n / 2, base = pairs / s, extra = pairs % s;
  const int start = k * base + std::min(k, extra), cnt = base + (k < extra ? 1 : 0);
  return {2 * start, 2 * (start + cnt)};
}

void need_single(const tmg_machine* tm, const char* what) {
  if (is_sharded(tm))
    fail(TMG_EINVAL, std::string(what) + " needs a single-device machine (this one is clause-sharded)");
}

void destroy_group(tmg_machine* tm) {
  for (tmg_machine* p : tm->parts) tmg_machine_destroy(p);
  tm->parts.clear();
  if (tm->owns_xchg) delete tm->xchg;
  tm->xchg = nullptr;
}

// -------------------------------------------------------- pool replicas ---
tmg_pool* make_replica(tmg_pool* src, int device) {
  tmg_pool* r = create_pool_common(device, src->o, src->q, src->m);
  try {
    DeviceGuard dg(device);
    CK(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    const size_t rows = static_cast<size_t>(src->q);
    r->rows.alloc(rows * 2 * r->Wp);
    r->labels.alloc(rows);
    r->tallies.alloc(rows * r->m);
    r->delta.alloc(rows * r->m);
    r->order.alloc(rows);
    CK(cudaMemcpyPeerAsync(r->rows.ptr, device, src->rows.ptr, src->device, r->rows.bytes(), r->stream));
    CK(cudaMemcpyPeerAsync(r->labels.ptr, device, src->labels.ptr, src->device, r->labels.bytes(), r->stream));
    CK(cudaMemsetAsync(r->delta.ptr, 0, r->delta.bytes(), r->stream));
    CK(cudaStreamSynchronize(r->stream));
    r->host_labels = src->host_labels;
    r->primary = src;
  } catch (...) {
    tmg_pool_destroy(r);
    throw;
  }
  return r;
}

void destroy_replicas(tmg_pool* pool) {
  for (tmg_pool* r : pool->replicas)
    if (r != pool) tmg_pool_destroy(r);
  pool->replicas.clear();
}

// One tally replica per shard, holding the primary's current tallies.
std::vector<tmg_pool*> replicas_for(tmg_machine* g, tmg_pool* pool) {
  const size_t n = g->parts.size();
  bool ok = pool->replicas.size() == n;
  for (size_t k = 0; ok && k < n; ++k) ok = pool->replicas[k]->device == g->parts[k]->device;
  if (!ok) {
    destroy_replicas(pool);
    for (size_t k = 0; k < n; ++k)
      pool->replicas.push_back(k == 0 && g->parts[0]->device == pool->device ? pool
                                                                             : make_replica(pool, g->parts[k]->device));
  }
  CK(cudaStreamSynchronize(pool->stream));
  for (tmg_pool* r : pool->replicas)
    if (r != pool) {
      DeviceGuard dg(r->device);
      CK(cudaMemcpyPeerAsync(r->tallies.ptr, r->device, pool->tallies.ptr, pool->device, pool->tallies.bytes(),
                             r->stream));
      CK(cudaStreamSynchronize(r->stream));
    }
  return pool->replicas;
}

// ----------------------------------------------------------- the epoch ---
// One asynchronous epoch of every shard, with the tally replicas exchanged
// while the epochs run. Each shard's epoch is ONE launch over all its clauses
// — the schedule of a single-GPU epoch (clause warps retire and the next take
// their place), which learns measurably better than cutting every clause's
// pass into lock-step windows. The kernels add every tally
// change to their own replica and to a cumulative delta buffer that is never
// reset during the epoch; a host loop on high-priority side streams copies the
// cumulative deltas (copy engine), sums them over all shards (NCCL or the
// peer-memory kernel) and adds to each replica the others' growth since the
// previous exchange. A 32-bit copy of a word that kernels are RED-adding to
// reads some prefix of those adds, so every change is counted exactly once
// over the epoch; the loop ends with an exchange taken after every shard's
// kernel has finished (a done flag rides in the sums).
void sharded_epoch(Exchange& X, const std::vector<tmg_machine*>& shards, const std::vector<tmg_pool*>& pools,
                   int32_t epoch, int windows, std::vector<uint64_t>& events) {
  const size_t n = shards.size();
  const int64_t q = pools[0]->q;
  const int m = shards[0]->m;
  const int64_t cnt = q * m;
  X.ensure(cnt + 1);
  const auto t_begin = std::chrono::steady_clock::now();
  for (size_t k = 0; k < n; ++k) {
    tmg_machine* tm = shards[k];
    DeviceGuard dg(tm->device);
    bind_for(tm, q);
    upload_order(tm, pools[k], epoch);
    epoch_keys(tm, epoch);
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    CK(cudaMemsetAsync(pools[k]->delta.ptr, 0, pools[k]->delta.bytes(), tm->stream));
    for (int b = 0; b < 2; ++b) {  // the "previous" snapshot and sum of exchange 0 are zero
      CK(cudaMemsetAsync(X.slots[k]->snap[b].ptr, 0, X.slots[k]->snap[b].bytes(), tm->stream));
      CK(cudaMemsetAsync(X.slots[k]->red[b].ptr, 0, X.slots[k]->red[b].bytes(), tm->stream));
    }
    CK(cudaStreamSynchronize(tm->stream));
  }
  for (size_t k = 0; k < n; ++k) {  // the epochs: one launch per shard
    tmg_machine* tm = shards[k];
    DeviceGuard dg(tm->device);
    run_async_window(tm, pools[k], 0, q, true);
    CK(cudaEventRecord(X.slots[k]->done, tm->stream));
  }
  const int total = static_cast<int>(n) * X.nranks;
  const auto interval = std::chrono::duration<double>(X.interval_s);
  int64_t last_sq = -1;
  for (int64_t it = 0;; ++it) {
    const int64_t sq = X.seq++;  // the same on every rank: all ranks run the same exchanges
    const int b = static_cast<int>(sq & 1), p = b ^ 1;
    last_sq = sq;
    // wait for the interval or for every local shard to finish
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      bool all = true;
      for (size_t k = 0; k < n && all; ++k) all = cudaEventQuery(X.slots[k]->done) == cudaSuccess;
      if (all || std::chrono::steady_clock::now() - t0 >= interval) break;
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    for (size_t k = 0; k < n; ++k) {  // snapshot the cumulative deltas (+ done flag)
      DeviceGuard dg(shards[k]->device);
      Exchange::Slot& sl = *X.slots[k];
      sl.flag[0] = cudaEventQuery(sl.done) == cudaSuccess ? 1 : 0;  // before the copy: a done shard's copy is final
      if (X.use_ipc) X.wait_consumed(b, sq - 2);  // the other ranks pulled what slot b held
      else X.wait_reduced(k, b, X.cstreams[k]);   // slot b's last readers (two exchanges ago) are done
      CK(cudaMemcpyAsync(sl.snap[b].ptr, pools[k]->delta.ptr, static_cast<size_t>(cnt) * 4, cudaMemcpyDeviceToDevice,
                         X.cstreams[k]));
      CK(cudaMemcpyAsync(sl.snap[b].ptr + cnt, sl.flag, 4, cudaMemcpyHostToDevice, X.cstreams[k]));
      CK(cudaEventRecord(sl.snap_ev[b], X.cstreams[k]));
    }
    if (X.use_ipc) X.reduce_ipc(b, sq);
    else X.reduce(b);
    for (size_t k = 0; k < n; ++k) {  // replica += the other shards' growth since the last exchange
      DeviceGuard dg(shards[k]->device);
      Exchange::Slot& sl = *X.slots[k];
      X.wait_reduced(k, b, X.cstreams[k]);
      tmg::count_launch();
      stream_apply_kernel<<<148, 256, 0, X.cstreams[k]>>>(pools[k]->tallies.ptr, sl.red[b].ptr, sl.red[p].ptr,
                                                          sl.snap[b].ptr, sl.snap[p].ptr, cnt);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(sl.flag + 1, sl.red[b].ptr + cnt, 4, cudaMemcpyDeviceToHost, X.cstreams[k]));
    }
    for (size_t k = 0; k < n; ++k) {  // (also frees the pinned flags for the next exchange)
      DeviceGuard dg(shards[k]->device);
      CK(cudaStreamSynchronize(X.cstreams[k]));
    }
    if (X.slots[0]->flag[1] >= total) break;  // every shard's final deltas are in this exchange
  }
  for (size_t k = 0; k < n; ++k) {
    DeviceGuard dg(shards[k]->device);
    CK(cudaStreamSynchronize(X.cstreams[k]));
    CK(cudaStreamSynchronize(shards[k]->stream));
  }
  if (X.use_ipc) {  // no rank may zero its slots for the next epoch while another still pulls
    X.wait_consumed(static_cast<int>(last_sq & 1), last_sq);
    X.wait_consumed(static_cast<int>((last_sq - 1) & 1), last_sq - 1);
  }
  // aim at `windows` exchanges in the next epoch of similar length
  const double took = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_begin).count();
  X.interval_s = std::max(2e-4, took / std::max(1, windows));
  events.assign(static_cast<size_t>(2 * m), 0);
  std::vector<unsigned long long> ev(static_cast<size_t>(2 * m));
  for (size_t k = 0; k < n; ++k) {
    DeviceGuard dg(shards[k]->device);
    CK(cudaMemcpyAsync(ev.data(), shards[k]->events.ptr, shards[k]->events.bytes(), cudaMemcpyDeviceToHost,
                       shards[k]->stream));
    CK(cudaStreamSynchronize(shards[k]->stream));
    for (size_t c = 0; c < ev.size(); ++c) events[c] += ev[c];
  }
  X.allreduce_host(events.data(), events.size());
}

int group_train_epoch(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                      tmg_epoch_report* report) {
  return guarded([&] {
    check_compatible(tm, pool);
    if (workers < 1) fail(TMG_EINVAL, "workers must be >= 1");  // trainer.cpp:184
    if (resolve_mode(mode, workers) != TMG_MODE_ASYNC)
      fail(TMG_EINVAL, "a clause-sharded machine trains asynchronously only (the W = 1 replay needs one device)");
    if (tm->regress_mode || tm->all_positive) fail(TMG_EINVAL, "regression heads are single-device");
    const auto wall0 = std::chrono::steady_clock::now();
    std::vector<tmg_machine*> shards;
    std::vector<tmg_pool*> pools;
    if (is_group(tm)) {
      shards = tm->parts;
      pools = replicas_for(tm, pool);
    } else {  // this rank's shard of a multi-process machine
      if (!pool->peers.empty()) fail(TMG_EINVAL, "pool has peer tally replicas attached; detach them first");
      shards = {tm};
      pools = {pool};
    }
    std::vector<uint64_t> ev;
    sharded_epoch(*tm->xchg, shards, pools, epoch, tm->windows, ev);
    if (is_group(tm) && pools[0] != pool) {  // the primary holds the trained tallies
      DeviceGuard dg(pool->device);
      CK(cudaMemcpyPeerAsync(pool->tallies.ptr, pool->device, pools[0]->tallies.ptr, pools[0]->device,
                             pool->tallies.bytes(), pool->stream));
      CK(cudaStreamSynchronize(pool->stream));
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
    if (report) {
      report->epoch = epoch;
      report->seconds = std::max(secs, 1e-9);
      report->device_seconds = secs;
      for (int c = 0; c < tm->m; ++c) {
        if (report->feedback_events) report->feedback_events[c] = ev[static_cast<size_t>(c)];
        if (report->type_i_events) report->type_i_events[c] = ev[static_cast<size_t>(tm->m + c)];
      }
    }
  });
}

// --------------------------------------------------------- class sums ---
int group_class_sums(tmg_machine* tm, const tmg_pool* cpool, const uint64_t* lits, int64_t q, int32_t mode,
                     int32_t* out, bool set_tallies) {
  return guarded([&] {
    auto* pool = const_cast<tmg_pool*>(cpool);
    if (pool) {
      check_compatible(tm, pool);
      q = pool->q;
    }
    if (q <= 0) return;
    const bool train = mode == TMG_EVAL_TRAIN;
    const size_t cnt = static_cast<size_t>(q) * tm->m;
    std::fill(out, out + cnt, 0);
    std::vector<int32_t> part(cnt);
    std::vector<tmg_machine*> shards = is_group(tm) ? tm->parts : std::vector<tmg_machine*>{tm};
    std::vector<tmg_pool*> pools;
    if (pool) pools = is_group(tm) ? replicas_for(tm, pool) : std::vector<tmg_pool*>{pool};
    for (size_t k = 0; k < shards.size(); ++k) {
      tmg_machine* s = shards[k];
      DeviceGuard dg(s->device);
      DevBuf<int32_t> d;
      d.alloc(cnt);
      if (pool) {
        if (set_tallies) bind_for(s, q);  // refresh_tallies binds (pool.cpp:113)
        class_sums_device(s, pools[k]->xplane(), q, train, d.ptr, set_tallies ? s->prev.ptr : nullptr,
                          pool_lit_t(s, pools[k]));
      } else {
        DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
        literals_to_planes(s, lits, q, xs);
        class_sums_device(s, xs.ptr, q, train, d.ptr, nullptr);
      }
      CK(cudaMemcpyAsync(part.data(), d.ptr, cnt * 4, cudaMemcpyDeviceToHost, s->stream));
      CK(cudaStreamSynchronize(s->stream));
      for (size_t i = 0; i < cnt; ++i) out[i] += part[i];
    }
    tm->xchg->allreduce_host(out, cnt);
    if (set_tallies && pool && tmg_pool_set_tallies(pool, out) != TMG_OK) fail(TMG_ERUNTIME, tmg_last_error());
  });
}

// ------------------------------------------------- state in slices ---
int group_info(const tmg_machine* tm, tmg_machine_info* info) {
  return guarded([&] {
    if (tmg_machine_info_get(tm->parts[0], info) != TMG_OK) fail(TMG_ERUNTIME, tmg_last_error());
    uint64_t bytes = 0;
    for (tmg_machine* p : tm->parts) {
      tmg_machine_info pi{};
      if (tmg_machine_info_get(p, &pi) != TMG_OK) fail(TMG_ERUNTIME, tmg_last_error());
      bytes += pi.device_bytes;
    }
    info->clause_begin = 0;
    info->clause_end = tm->n;
    info->device_bytes = bytes;
  });
}

int group_reset(tmg_machine* tm) {
  return guarded([&] {
    for (tmg_machine* p : tm->parts)
      if (tmg_machine_reset(p) != TMG_OK) fail(TMG_ERUNTIME, tmg_last_error());
  });
}

int group_counters(const tmg_machine* tm, int32_t bank, uint16_t* out, const uint16_t* in) {
  return guarded([&] {
    if (bank < 0 || bank >= tm->m) fail(TMG_ERANGE, "bank index out of range");
    const size_t row = 2 * static_cast<size_t>(tm->o);
    for (tmg_machine* p : tm->parts) {
      const size_t off = static_cast<size_t>(p->j_begin) * row;
      const int rc = out ? tmg_get_counters(p, bank, out + off) : tmg_set_counters(p, bank, in + off);
      if (rc != TMG_OK) fail(rc, tmg_last_error());
    }
  });
}

int group_include(const tmg_machine* tm, int32_t bank, uint64_t* masks, int32_t* counts) {
  return guarded([&] {
    if (bank < 0 || bank >= tm->m) fail(TMG_ERANGE, "bank index out of range");
    const size_t w64 = static_cast<size_t>((2 * tm->o + 63) / 64);
    for (tmg_machine* p : tm->parts) {
      const int rc = masks ? tmg_get_include_masks(p, bank, masks + static_cast<size_t>(p->j_begin) * w64)
                           : tmg_get_include_counts(p, bank, counts + p->j_begin);
      if (rc != TMG_OK) fail(rc, tmg_last_error());
    }
  });
}

int group_bind(tmg_machine* tm, int32_t bank, int64_t q) {
  return guarded([&] {
    for (tmg_machine* p : tm->parts) {
      const int rc = bank < 0 ? tmg_bind_examples(p, q) : tmg_bind_bank(p, bank, q);
      if (rc != TMG_OK) fail(rc, tmg_last_error());
    }
    tm->q_bound = tm->parts[0]->q_bound;
    tm->bank_q = tm->parts[0]->bank_q;
  });
}

int group_prev(const tmg_machine* tm, int32_t bank, uint64_t* out, const uint64_t* in) {
  return guarded([&] {
    if (bank < 0 || bank >= tm->m) fail(TMG_ERANGE, "bank index out of range");
    const size_t w = static_cast<size_t>((tm->parts[0]->bank_q[static_cast<size_t>(bank)] + 63) / 64);
    for (tmg_machine* p : tm->parts) {
      const size_t off = static_cast<size_t>(p->j_begin) * w;
      const int rc = out ? tmg_get_prev_outputs(p, bank, out + off) : tmg_set_prev_outputs(p, bank, in + off);
      if (rc != TMG_OK) fail(rc, tmg_last_error());
    }
  });
}

tmg_machine* group_owner(const tmg_machine* tm, int32_t j) {
  for (tmg_machine* p : tm->parts)
    if (j >= p->j_begin && j < p->j_end) return p;
  return nullptr;
}

// update_clause (trainer.cpp:102-136) on the shard that owns clause j, with
// that shard's tally replica; the pool's tallies are the replica's after.
int group_update_clause(tmg_machine* tm, tmg_pool* pool, int32_t c, int32_t j, const int32_t* order,
                        int64_t order_len, int64_t offset, int64_t batch, int32_t margin, double s, int32_t boost,
                        uint64_t* rng_state, uint64_t* events) {
  tmg_machine* part = group_owner(tm, j);
  if (!part) return guarded([&] { fail(TMG_ERANGE, "clause index outside this machine"); });
  if (!pool) return guarded([&] { fail(TMG_EINVAL, "null handle"); });
  size_t k = 0;
  while (tm->parts[k] != part) ++k;
  tmg_pool* rep = nullptr;
  const int rc0 = guarded([&] {
    if (c < 0 || c >= tm->m) fail(TMG_ERANGE, "class index out of range");
    for (tmg_machine* p : tm->parts)  // the bank spans every shard: rebind it everywhere (trainer.cpp:107)
      if (p->bank_q[static_cast<size_t>(c)] != pool->q && tmg_bind_bank(p, c, pool->q) != TMG_OK)
        fail(TMG_ERUNTIME, tmg_last_error());
    tm->bank_q = tm->parts[0]->bank_q;
    tm->q_bound = tm->parts[0]->q_bound;
    rep = replicas_for(tm, pool)[k];
  });
  if (rc0 != TMG_OK) return rc0;
  const int rc = tmg_update_clause(part, rep, c, j, order, order_len, offset, batch, margin, s, boost, rng_state,
                                   events);
  if (rc != TMG_OK || rep == pool) return rc;
  return guarded([&] {
    DeviceGuard dg(pool->device);
    CK(cudaMemcpyPeerAsync(pool->tallies.ptr, pool->device, rep->tallies.ptr, rep->device, pool->tallies.bytes(),
                           pool->stream));
    CK(cudaStreamSynchronize(pool->stream));
  });
}

}  // namespace tmgx

using namespace tmgx;

// ===================================================================== ABI ===

TMG_API int tmg_machine_create_devices(const tmg_config* cfg, int32_t o, int32_t m, const int32_t* devices,
                                       int32_t ndev, tmg_machine** out) {
  return guarded([&] {
    if (!cfg) fail(TMG_EINVAL, "null config");
    if (ndev < 1 || ndev > 16 || !devices) fail(TMG_EINVAL, "1 to 16 devices");
    if (ndev == 1) {  // a plain machine
      *out = create_machine(cfg, o, m, devices[0], 0, cfg->clauses);
      return;
    }
    validate_config(*cfg);
    if (cfg->clauses / 2 < ndev) fail(TMG_EINVAL, "fewer clause pairs than devices");
    auto g = new tmg_machine();
    try {
      g->cfg = *cfg;
      g->o = o;
      g->m = m;
      g->n = cfg->clauses;
      g->j_begin = 0;
      g->j_end = g->n;
      g->n_loc = g->n;
      g->device = devices[0];
      for (int k = 0; k < ndev; ++k) {
        const auto r = shard_range(g->n, k, ndev);
        g->parts.push_back(create_machine(cfg, o, m, devices[k], r.first, r.second));
      }
      g->N = g->parts[0]->N;
      g->B = g->parts[0]->B;
      g->NW = g->parts[0]->NW;
      g->Wx = g->parts[0]->Wx;
      g->Wp = g->parts[0]->Wp;
      g->bank_q = g->parts[0]->bank_q;
      auto* x = new Exchange();
      g->xchg = x;
      g->owns_xchg = true;
      x->devices.assign(devices, devices + ndev);
      std::vector<int> sorted(x->devices);
      std::sort(sorted.begin(), sorted.end());
      const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
      const char* pref = std::getenv("TSETLIN_EXCHANGE");
      const bool want_peer = pref && std::strcmp(pref, "peer") == 0;
      x->use_nccl = distinct && !want_peer && nccl().ok;
      if (!x->use_nccl) {  // peer-memory sums: every shard must reach every other's buffers
        for (int a : sorted)
          for (int b : sorted) {
            if (a == b) continue;
            int can = 0;
            CK(cudaDeviceCanAccessPeer(&can, a, b));
            if (!can) fail(TMG_ERUNTIME, "no peer access between devices " + std::to_string(a) + " and " +
                                             std::to_string(b) + (nccl().ok ? "" : " and NCCL unavailable: " + nccl().why));
            DeviceGuard dg(a);
            const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
            cudaGetLastError();
          }
      }
      x->init_streams();
      if (x->use_nccl) {
        x->comms.resize(static_cast<size_t>(ndev));
        nccl_check(nccl().CommInitAll(x->comms.data(), ndev, x->devices.data()), "ncclCommInitAll");
      }
    } catch (...) {
      tmg_machine_destroy(g);
      throw;
    }
    *out = g;
  });
}

TMG_API int tmg_pool_replica_tallies(const tmg_pool* pool, int32_t k, int32_t* out) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    if (k < 0 || k >= static_cast<int32_t>(pool->replicas.size())) fail(TMG_ERANGE, "no such replica");
    const tmg_pool* r = pool->replicas[static_cast<size_t>(k)];
    DeviceGuard dg(r->device);
    CK(cudaMemcpy(out, r->tallies.ptr, r->tallies.bytes(), cudaMemcpyDeviceToHost));
  });
}

TMG_API int tmg_machine_set_windows(tmg_machine* tm, int32_t windows) {
  return guarded([&] {
    if (!tm) fail(TMG_EINVAL, "null machine handle");
    if (windows < 1) fail(TMG_EINVAL, "windows must be >= 1");
    tm->windows = windows;
  });
}

TMG_API int tmg_machine_exchange_info(const tmg_machine* tm, int32_t* shards, int32_t* uses_nccl) {
  return guarded([&] {
    if (!tm) fail(TMG_EINVAL, "null machine handle");
    *shards = is_group(tm) ? static_cast<int32_t>(tm->parts.size()) : (tm->xchg ? tm->xchg->nranks : 1);
    *uses_nccl = tm->xchg && tm->xchg->use_nccl ? 1 : 0;
  });
}

TMG_API int tmg_nccl_available(char* why, int32_t len) {
  Nccl& n = nccl();
  if (why && len > 0) {
    std::strncpy(why, n.ok ? "" : n.why.c_str(), static_cast<size_t>(len - 1));
    why[len - 1] = '\0';
  }
  return n.ok ? 1 : 0;
}

TMG_API int tmg_comm_unique_id(unsigned char* id) {
  return guarded([&] {
    if (!nccl().ok) fail(TMG_ERUNTIME, "NCCL unavailable: " + nccl().why);
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, sizeof u);
  });
}

TMG_API int tmg_comm_create(const unsigned char* id, int32_t nranks, int32_t rank, int32_t device, tmg_comm** out) {
  return guarded([&] {
    if (!nccl().ok) fail(TMG_ERUNTIME, "NCCL unavailable: " + nccl().why);
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(TMG_EINVAL, "bad rank / rank count");
    auto c = new tmg_comm();
    c->x = new Exchange();
    try {
      c->x->use_nccl = true;
      c->x->nranks = nranks;
      c->x->rank = rank;
      c->x->devices = {device};
      c->x->init_streams();
      ncclUniqueId u;
      std::memcpy(&u, id, sizeof u);
      c->x->comms.resize(1);
      DeviceGuard dg(device);
      nccl_check(nccl().CommInitRank(&c->x->comms[0], nranks, u, rank), "ncclCommInitRank");
    } catch (...) {
      delete c->x;
      delete c;
      throw;
    }
    *out = c;
  });
}

TMG_API int tmg_comm_create_ipc(int32_t nranks, int32_t rank, int32_t device, int64_t capacity, tmg_comm** out) {
  return guarded([&] {
    if (nranks < 1 || nranks > 16 || rank < 0 || rank >= nranks) fail(TMG_EINVAL, "bad rank / rank count (1-16)");
    if (capacity < 1) fail(TMG_EINVAL, "capacity (q x m) must be >= 1");
    auto c = new tmg_comm();
    c->x = new Exchange();
    try {
      Exchange& x = *c->x;
      x.use_ipc = true;
      x.nranks = nranks;
      x.rank = rank;
      x.devices = {device};
      x.init_streams();
      DeviceGuard dg(device);
      x.ipc_count = capacity + 1;  // + the done flag
      for (int b = 0; b < 2; ++b) {
        x.slots[0]->snap[b].alloc_plain(static_cast<size_t>(x.ipc_count));
        x.slots[0]->red[b].alloc_plain(static_cast<size_t>(x.ipc_count));
      }
      x.ctl.alloc_plain(2 + 2 * static_cast<size_t>(nranks));
      CK(cudaMemset(x.ctl.ptr, 0xFF, x.ctl.bytes()));  // every sequence word -1: nothing ready, nothing pulled
      x.recv.resize(static_cast<size_t>(nranks));
      for (int j = 0; j < nranks; ++j) {
        if (j == rank) continue;
        x.recv[static_cast<size_t>(j)] = std::make_unique<DevBuf<int32_t>>();
        x.recv[static_cast<size_t>(j)]->alloc_plain(static_cast<size_t>(x.ipc_count));
      }
      CK(cudaStreamCreateWithFlags(&x.pstream, cudaStreamNonBlocking));
      CK(cudaMallocHost(reinterpret_cast<void**>(&x.hpoll), 4 * sizeof(int64_t)));
    } catch (...) {
      delete c->x;
      delete c;
      throw;
    }
    *out = c;
  });
}

TMG_API int tmg_comm_ipc_handle(tmg_comm* comm, unsigned char* out) {
  return guarded([&] {
    if (!comm || !comm->x->use_ipc) fail(TMG_EINVAL, "not an IPC communicator");
    Exchange& x = *comm->x;
    DeviceGuard dg(x.devices[0]);
    cudaIpcMemHandle_t h[3];
    CK(cudaIpcGetMemHandle(&h[0], x.slots[0]->snap[0].ptr));
    CK(cudaIpcGetMemHandle(&h[1], x.slots[0]->snap[1].ptr));
    CK(cudaIpcGetMemHandle(&h[2], x.ctl.ptr));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "64-byte IPC handles");
    std::memcpy(out, h, sizeof h);
  });
}

TMG_API int tmg_comm_ipc_connect(tmg_comm* comm, const unsigned char* all) {
  return guarded([&] {
    if (!comm || !comm->x->use_ipc) fail(TMG_EINVAL, "not an IPC communicator");
    Exchange& x = *comm->x;
    DeviceGuard dg(x.devices[0]);
    x.peer_snap[0].assign(static_cast<size_t>(x.nranks), nullptr);
    x.peer_snap[1].assign(static_cast<size_t>(x.nranks), nullptr);
    x.peer_ctl.assign(static_cast<size_t>(x.nranks), nullptr);
    for (int j = 0; j < x.nranks; ++j) {
      if (j == x.rank) continue;
      cudaIpcMemHandle_t h[3];
      std::memcpy(h, all + static_cast<size_t>(j) * sizeof h, sizeof h);
      void* p = nullptr;
      for (int b = 0; b < 2; ++b) {
        CK(cudaIpcOpenMemHandle(&p, h[b], cudaIpcMemLazyEnablePeerAccess));
        x.peer_snap[b][static_cast<size_t>(j)] = static_cast<int32_t*>(p);
      }
      CK(cudaIpcOpenMemHandle(&p, h[2], cudaIpcMemLazyEnablePeerAccess));
      x.peer_ctl[static_cast<size_t>(j)] = static_cast<int64_t*>(p);
    }
  });
}

TMG_API int tmg_comm_destroy(tmg_comm* comm) {
  if (!comm) return TMG_OK;
  delete comm->x;
  delete comm;
  return TMG_OK;
}

TMG_API int tmg_machine_attach_comm(tmg_machine* tm, tmg_comm* comm) {
  return guarded([&] {
    if (!tm) fail(TMG_EINVAL, "null machine handle");
    if (is_group(tm)) fail(TMG_EINVAL, "a multi-device machine has its own exchange");
    if (tm->owns_xchg) fail(TMG_EINVAL, "machine owns an exchange");
    if (!comm) {  // detach
      tm->xchg = nullptr;
      return;
    }
    if (comm->x->devices[0] != tm->device) fail(TMG_EINVAL, "communicator and machine are on different devices");
    if (tm->all_positive) fail(TMG_EINVAL, "regression heads are single-device");
    tm->xchg = comm->x;
  });
}
