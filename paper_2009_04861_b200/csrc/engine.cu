// engine.cu — host runtime of the B200 Tsetlin engine and the C ABI
// (include/tmgpu.h). Owns device memory, one CUDA stream per machine/pool,
// the epoch orchestration (permutation, Philox keys, thresholds) and the
// conversions between the reference's host layouts and the device layouts.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "engine.h"
#include "kernels.h"
#include "tmgpu.h"
#include "tmgpu_rng.h"

namespace tmg {
unsigned long long g_launches = 0;
}

namespace tmgx {

thread_local std::string g_last_error;

// Keeps the current device's default memory pool from returning freed memory
// to the driver at every synchronisation (once per device).
void pool_init() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  static std::atomic<bool> done[64];
  if (done[dev].load(std::memory_order_acquire)) return;
  cudaMemPool_t mp;
  if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev].store(true, std::memory_order_release);
}


// Supported words-per-lane instantiations of the training kernels.
int round_nw(int nw) {
  // Compiled widths first (register-held rows); wider rows take the
  // runtime-width shared-memory kernel (train_smem.cu, NW = 0) as they are.
  static const int kNW[] = {1, 2, 3, 4, 6, 8, 10, 12, 16};
  for (int v : kNW)
    if (nw <= v) return v;
  return nw;
}

int planes_for(int N) {
  // 2^(B-1) >= N so Include is the top plane; instantiated B in {4, 8, 15}.
  if (N <= 8) return 4;
  if (N <= 128) return 8;
  return 15;
}

uint32_t prob_threshold(double p) {  // P(u < p) as 32-bit fixed point
  if (!(p > 0.0)) return 0u;
  const double v = std::ldexp(p, 32);
  if (v >= 4294967295.0) return 0xFFFFFFFFu;
  return static_cast<uint32_t>(std::llround(v));
}

// Walker/Vose alias table of the law of an 8-literal Type I pattern when
// every literal fires independently with probability p = P / 2^32 (the
// clause-output-0 draw of the async sampler, tm_device.cuh alias_words).
// Built exactly in integer units of 2^-32: each pattern's mass is its
// product-law probability rounded by largest remainders (error < 2^-32,
// total exactly 1), 256 columns of 2^24 units, so the sampled law equals
// the rounded masses exactly. Entry = threshold24 << 8 | alias; a column
// whose own pattern always wins is stored as (0 << 8 | itself).
void build_alias8(uint32_t P, uint32_t out[256]) {
  const double p = std::ldexp(static_cast<double>(P), -32);
  int64_t mass[256];
  double frac[256];
  int64_t total = 0;
  for (int i = 0; i < 256; ++i) {
    const int k = __builtin_popcount(static_cast<unsigned>(i));
    const double units = std::ldexp(std::pow(p, k) * std::pow(1.0 - p, 8 - k), 32);
    mass[i] = static_cast<int64_t>(std::floor(units));
    frac[i] = units - static_cast<double>(mass[i]);
    total += mass[i];
  }
  int order[256];
  for (int i = 0; i < 256; ++i) order[i] = i;
  std::stable_sort(order, order + 256, [&](int a, int b) { return frac[a] > frac[b]; });
  for (int r = 0; total < (int64_t(1) << 32); ++r, ++total) ++mass[order[r % 256]];
  for (int r = 255; total > (int64_t(1) << 32); --r, --total)  // (float slack only)
    if (mass[order[r]] > 0) --mass[order[r]];
  constexpr int64_t kCol = int64_t(1) << 24;
  int alias[256];
  int64_t thr[256];
  int small[256], large[256], ns = 0, nl = 0;
  for (int i = 0; i < 256; ++i) {
    alias[i] = i;
    thr[i] = kCol;
    (mass[i] < kCol ? small[ns++] : large[nl++]) = i;
  }
  while (ns > 0 && nl > 0) {
    const int a = small[--ns], b = large[--nl];
    thr[a] = mass[a];
    alias[a] = b;
    mass[b] -= kCol - mass[a];
    (mass[b] < kCol ? small[ns++] : large[nl++]) = b;
  }
  for (int i = 0; i < 256; ++i)
    out[i] = (alias[i] == i || thr[i] >= kCol) ? static_cast<uint32_t>(i)
                                               : (static_cast<uint32_t>(thr[i]) << 8) | static_cast<uint32_t>(alias[i]);
}


}  // namespace tmgx

using namespace tmgx;

namespace tmgx {

void validate_config(const tmg_config& c) {  // core.cpp:48-74
  if (c.clauses < 2 || c.clauses % 2 != 0)
    fail(TMG_EINVAL, "clauses must be even and >= 2, got " + std::to_string(c.clauses));
  if (c.margin < 1) fail(TMG_EINVAL, "margin must be >= 1, got " + std::to_string(c.margin));
  if (!(c.specificity >= 1.0)) fail(TMG_EINVAL, "specificity must be >= 1, got " + std::to_string(c.specificity));
  if (c.state_depth < 1) fail(TMG_EINVAL, "state depth must be >= 1, got " + std::to_string(c.state_depth));
  if (c.state_depth > 16383) fail(TMG_EINVAL, "state depth too large for 16-bit counters");
  if (c.epochs < 0) fail(TMG_EINVAL, "epochs must be >= 0");
  if (c.workers < 0) fail(TMG_EINVAL, "workers must be >= 0 (0 = auto)");
}

int words_x(int o) { return (o + 31) / 32; }
int wp_for(int o) { return 32 * round_nw((words_x(o) + 31) / 32); }

void check_compatible(const tmg_machine* tm, const tmg_pool* pool) {  // trainer.cpp:46-53
  if (!tm || !pool) fail(TMG_EINVAL, "null handle");
  if (tm->o != pool->o) fail(TMG_EINVAL, "model/pool feature count mismatch");
  if (tm->m != pool->m) fail(TMG_EINVAL, "model/pool class count mismatch");
  if (tm->device != pool->device) fail(TMG_EINVAL, "model and pool live on different devices");
}

void check_bind_count(int64_t q) {
  if (q < 0) fail(TMG_EINVAL, "example count must be >= 0");
  if (q > (int64_t(1) << 31) - 64) fail(TMG_EINVAL, "example count too large");
}

// bind_examples on every bank (core.cpp:117-126): all bitmaps cleared.
void bind(tmg_machine* tm, int64_t q) {
  check_bind_count(q);
  tm->q_bound = q;
  tm->bank_q.assign(static_cast<size_t>(tm->m), q);
  tm->Wq = static_cast<int>(2 * ((q + 63) / 64));
  tm->prev.alloc(static_cast<size_t>(tm->clauses()) * tm->Wq);
  if (tm->prev.bytes()) CK(cudaMemsetAsync(tm->prev.ptr, 0, tm->prev.bytes(), tm->stream));
  CK(cudaStreamSynchronize(tm->stream));
}

// bind_examples on ONE bank: only its bitmap is cleared, the other banks keep
// theirs (the buffer's row stride grows to the widest binding).
void bind_bank(tmg_machine* tm, int c, int64_t q) {
  check_bind_count(q);
  const int need = static_cast<int>(2 * ((q + 63) / 64));
  const size_t rows = static_cast<size_t>(tm->clauses());
  if (need > tm->Wq) {
    DevBuf<uint32_t> grown;
    grown.alloc(rows * need);
    CK(cudaMemsetAsync(grown.ptr, 0, grown.bytes(), tm->stream));
    if (tm->Wq > 0 && rows)
      CK(cudaMemcpy2DAsync(grown.ptr, static_cast<size_t>(need) * 4, tm->prev.ptr, static_cast<size_t>(tm->Wq) * 4,
                           static_cast<size_t>(tm->Wq) * 4, rows, cudaMemcpyDeviceToDevice, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    tm->prev.swap(grown);
    tm->Wq = need;
  }
  const size_t bank_words = static_cast<size_t>(tm->n_loc) * tm->Wq;
  if (bank_words)
    CK(cudaMemsetAsync(tm->prev.ptr + static_cast<size_t>(c) * bank_words, 0, bank_words * 4, tm->stream));
  tm->bank_q[static_cast<size_t>(c)] = q;
  tm->q_bound = q;
  for (int64_t b : tm->bank_q)
    if (b != q) tm->q_bound = -1;
  CK(cudaStreamSynchronize(tm->stream));
}

// What every trainer does first (trainer.cpp:150,192-194; pool.cpp:113):
// rebind only the banks whose bound count differs from the pool's.
void bind_for(tmg_machine* tm, int64_t q) {
  if (tm->q_bound == q) return;
  bool none = true;
  for (int64_t b : tm->bank_q) none = none && b != q;
  if (none) return bind(tm, q);
  for (int c = 0; c < tm->m; ++c)
    if (tm->bank_q[static_cast<size_t>(c)] != q) bind_bank(tm, c, q);
}

// Include counts and the per-clause included-literal lists of the current
// state (rebuilt lazily after any state change).
void rebuild_entries(tmg_machine* tm) {
  if (!tm->entries_dirty) return;
  const int64_t total = tmg::build_lists_launch(tm->state.ptr, tm->clauses(), tm->B, tm->Wp, tm->Wx,
                                                tm->inc_count.ptr, tm->lens.ptr, tm->npos.ptr, tm->offs.ptr,
                                                tm->stream);
  if (total < 0) CK(cudaGetLastError());
  tm->lists_total = total;
  if (tm->lists.count < static_cast<size_t>(total) + 8) {
    // grow with headroom: lists get longer as clauses learn
    tm->lists.alloc(static_cast<size_t>(total + total / 4) + 64);
  }
  tmg::fill_lists_launch(tm->state.ptr, tm->clauses(), tm->B, tm->Wp, tm->Wx, tm->o, tm->offs.ptr, tm->npos.ptr,
                         tm->lists.ptr, tm->meta.ptr, tm->stream);
  CK(cudaGetLastError());
  tm->entries_dirty = false;
}

void reset_state(tmg_machine* tm) {  // ClassBank ctor: counters = N (core.cpp:96-100)
  tmg::init_state_launch(tm->state.ptr, tm->clauses(), tm->B, tm->Wp, tm->stream);
  CK(cudaGetLastError());
  if (tm->prev.bytes()) CK(cudaMemsetAsync(tm->prev.ptr, 0, tm->prev.bytes(), tm->stream));
  CK(cudaMemsetAsync(tm->inc_count.ptr, 0, tm->inc_count.bytes(), tm->stream));
  tm->entries_dirty = true;
  CK(cudaStreamSynchronize(tm->stream));
}

tmg_machine* create_machine(const tmg_config* cfg, int o, int m, int device, int jb, int je, int all_positive) {
  if (!cfg) fail(TMG_EINVAL, "null config");
  validate_config(*cfg);
  if (m < 1) fail(TMG_EINVAL, "class count must be >= 1");
  if (o < 1) fail(TMG_EINVAL, "feature count must be >= 1");
  if (jb < 0 || je > cfg->clauses || jb >= je || (jb % 2) || (je % 2))
    fail(TMG_EINVAL, "clause shard must be a non-empty even-aligned sub-range of [0, clauses)");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) fail(TMG_EINVAL, "no such CUDA device " + std::to_string(device));
  DeviceGuard dg(device);
  auto tm = new tmg_machine();
  try {
    tm->cfg = *cfg;
    tm->o = o;
    tm->m = m;
    tm->n = cfg->clauses;
    tm->j_begin = jb;
    tm->j_end = je;
    tm->n_loc = je - jb;
    tm->N = cfg->state_depth;
    tm->B = planes_for(tm->N);
    tm->Wx = words_x(o);
    tm->Wp = wp_for(o);
    tm->NW = tm->Wp / 32;
    // Rows wider than 4 words per lane keep a clause's automata in shared
    // memory (train_smem.cu), or in place in HBM beyond what shared memory holds.
    tm->device = device;
    tm->all_positive = all_positive ? 1 : 0;
    CK(cudaStreamCreateWithFlags(&tm->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&tm->ev0));
    CK(cudaEventCreate(&tm->ev1));
    const size_t cl = static_cast<size_t>(tm->clauses());
    tm->state.alloc(cl * tm->B * 2 * tm->Wp);
    tm->inc_count.alloc(cl);
    tm->lens.alloc(cl);
    tm->npos.alloc(cl);
    tm->meta.alloc(cl);
    tm->offs.alloc(cl + 1);
    tm->events.alloc(2 * static_cast<size_t>(m));  // all events, then Type I events
    tm->dbg.alloc(tmg::kDebugCounters);
    CK(cudaMemsetAsync(tm->dbg.ptr, 0, tm->dbg.bytes(), tm->stream));
    tm->work.alloc(1);
    {
      uint32_t tab[256];
      build_alias8(prob_threshold(1.0 / cfg->specificity), tab);
      tm->alias8.alloc(256);
      CK(cudaMemcpy(tm->alias8.ptr, tab, sizeof tab, cudaMemcpyHostToDevice));
    }
    bind(tm, 0);
    reset_state(tm);
  } catch (...) {
    tmg_machine_destroy(tm);
    throw;
  }
  return tm;
}

void upload_order(tmg_machine* tm, tmg_pool* pool, int32_t epoch) {
  // The epoch permutation of train_epoch_parallel (trainer.cpp:196-198).
  tmg_rng r;
  // regression epochs use their own stream kinds (regression.cpp:29-31)
  tmg_rng_seed(&r, tm->cfg.seed,
               tmg_mix_stream(tm->regress_mode ? 5 : TMG_STREAM_PERMUTATION, static_cast<uint64_t>(epoch), 0));
  std::vector<int32_t> order(static_cast<size_t>(pool->q));
  tmg_shuffled_indices(static_cast<int32_t>(pool->q), &r, order.data());
  CK(cudaMemcpyAsync(pool->order.ptr, order.data(), order.size() * 4, cudaMemcpyHostToDevice, tm->stream));
  CK(cudaStreamSynchronize(tm->stream));
}

tmg::TrainParams make_params(tmg_machine* tm, tmg_pool* pool) {
  tmg::TrainParams p{};
  p.state = tm->state.ptr;
  p.inc_count = tm->inc_count.ptr;
  p.prev = tm->prev.ptr;
  p.n = tm->n;
  p.n_loc = tm->n_loc;
  p.j_begin = tm->j_begin;
  p.m = tm->m;
  p.w_begin = 0;
  p.w_end = tm->m * tm->n_loc;
  p.o = tm->o;
  p.Wp = tm->Wp;
  p.Wq = tm->Wq;
  p.lo = (1u << (tm->B - 1)) - static_cast<uint32_t>(tm->N);
  p.hi = (1u << (tm->B - 1)) + static_cast<uint32_t>(tm->N) - 1u;
  p.xplane = pool->xplane();
  p.nplane = pool->nplane();
  p.labels = pool->labels.ptr;
  p.tallies = pool->tallies.ptr;
  p.tally_delta = nullptr;
  p.npeers = static_cast<int32_t>(pool->peers.size());
  for (int k = 0; k < tmg::kMaxPeers; ++k) p.peer_tallies[k] = k < p.npeers ? pool->peers[k] : nullptr;
  p.q = pool->q;
  p.order = pool->order.ptr;
  p.margin = tm->cfg.margin;
  p.boost = tm->cfg.boost_true_positive ? 1 : 0;
  p.all_positive = tm->all_positive;
  p.regress = tm->regress_mode ? 1 : 0;
  {  // clause order over the grid's waves (kernels.h TrainParams::interleave)
    const char* o = std::getenv("TMG_CLAUSE_ORDER");
    p.interleave = o && o[0] == 'c' ? 0 : (o && o[0] == 'w' ? 1 : 2);
  }
  const double s = tm->cfg.specificity;
  p.thr_high = prob_threshold((s - 1.0) / s);
  p.thr_low = prob_threshold(1.0 / s);
  for (int b = 0; b < 8; ++b) {
    p.bern.hi_mask[b] = ((p.thr_high >> (31 - b)) & 1u) ? 0xFFFFFFFFu : 0u;
    p.bern.lo_mask[b] = ((p.thr_low >> (31 - b)) & 1u) ? 0xFFFFFFFFu : 0u;
  }
  p.bern.hi_rest = p.thr_high & 0x00FFFFFFu;
  p.bern.lo_rest = p.thr_low & 0x00FFFFFFu;
  p.bern.one = 1u;
  p.key0 = tm->key0;
  p.key1 = tm->key1;
  for (int r = 0; r < tmg::kMaxPhiloxRounds; ++r) {
    p.rkey[0][r] = tm->key0 + static_cast<uint32_t>(r) * 0x9E3779B9u;
    p.rkey[1][r] = tm->key1 + static_cast<uint32_t>(r) * 0xBB67AE85u;
  }
  p.t_begin = 0;
  p.t_end = pool->q;
  p.events = tm->events.ptr;
  p.alias8 = tm->alias8.ptr;
  p.alias_sel = (static_cast<uint64_t>(p.thr_high) + p.thr_low == (uint64_t(1) << 32)) ? 1 : 0;
#ifdef TMG_STATS
  p.dbg = tm->dbg.ptr;
#endif
  p.work = tm->work.ptr;
  return p;
}

// ---- xoshiro256 jump-ahead matrices for the parallel sequential replay.
// The state update of rng.hpp next() (everything but the output scrambler)
// is linear over GF(2): state' = M * state, state bit 64k + t = bit t of s_k.
struct Gf2 {
  uint64_t r[256][4];  // row i: the input bits whose parity is output bit i
};

void xo_update(uint64_t s[4]) {  // rng.hpp next(), state part
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

Gf2 gf2_step() {
  static Gf2 m{};
  static bool done = false;
  if (!done) {
    for (int b = 0; b < 256; ++b) {  // column b = the update of unit vector b
      uint64_t e[4] = {0, 0, 0, 0};
      e[b >> 6] = uint64_t(1) << (b & 63);
      xo_update(e);
      for (int i = 0; i < 256; ++i)
        if ((e[i >> 6] >> (i & 63)) & 1) m.r[i][b >> 6] |= uint64_t(1) << (b & 63);
    }
    done = true;
  }
  return m;
}

Gf2 gf2_mul(const Gf2& a, const Gf2& b) {  // (a * b) x = a (b x)
  Gf2 c{};
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 256; ++j)
      if ((a.r[i][j >> 6] >> (j & 63)) & 1)
        for (int w = 0; w < 4; ++w) c.r[i][w] ^= b.r[j][w];
  return c;
}

Gf2 gf2_pow(uint64_t k) {
  Gf2 result{}, base = gf2_step();
  for (int i = 0; i < 256; ++i) result.r[i][i >> 6] = uint64_t(1) << (i & 63);
  while (k) {
    if (k & 1) result = gf2_mul(base, result);
    base = gf2_mul(base, base);
    k >>= 1;
  }
  return result;
}

// Device layout of tm_device.cuh gf2_apply: nibble tables, entry (pos, v) =
// the 8 words of m * (v << 4 pos) = XOR of the columns of m for v's bits.
void gf2_layout(const Gf2& m, uint32_t* out) {
  uint32_t col[256][8] = {};
  for (int i = 0; i < 256; ++i)
    for (int b = 0; b < 256; ++b)
      if ((m.r[i][b >> 6] >> (b & 63)) & 1) col[b][i >> 5] |= 1u << (i & 31);
  for (int pos = 0; pos < 64; ++pos)
    for (int v = 0; v < 16; ++v) {
      uint32_t* e = out + (pos * 16 + v) * 8;
      for (int w = 0; w < 8; ++w) e[w] = 0;
      for (int bit = 0; bit < 4; ++bit)
        if ((v >> bit) & 1)
          for (int w = 0; w < 8; ++w) e[w] ^= col[4 * pos + bit][w];
    }
}

// The parallel replay pays off once a bank has enough clauses to spread over
// the warps or the rows are wide enough for the draw segments to matter
// (XOR12, 20 clauses of 24 literals: serial 0.048 s vs parallel 0.085 s per
// 2 000 examples; MNIST-shaped: 29.0 s vs 2.4 s per 500). TMG_SEQ_SERIAL=1
// forces the serial replay, =0 the parallel one (A/B checks).
bool seq_parallel_enabled(const tmg_machine* tm) {
  const char* e = std::getenv("TMG_SEQ_SERIAL");
  if (e && e[0] == '1') return false;
  if (e && e[0] == '0') return true;
  return tm->n >= 64 || 2 * tm->o >= 128;
}

// TMG_SEQ_GRID=0 keeps the parallel replay on one CTA (A/B checks).
bool seq_grid_enabled() {
  const char* e = std::getenv("TMG_SEQ_GRID");
  return !(e && e[0] == '0');
}

// M^ceil(2o/32) and M^(2o), built once per machine.
void ensure_jumps(tmg_machine* tm) {
  const int L = 2 * tm->o;
  const int chunk = (L + 31) / 32;
  constexpr size_t kTab = tmg::kGf2TabWords;
  if (tm->seq_jump.count != 2 * kTab) {
    std::vector<uint32_t> host(2 * kTab);
    gf2_layout(gf2_pow(static_cast<uint64_t>(chunk)), host.data());
    gf2_layout(gf2_pow(static_cast<uint64_t>(L)), host.data() + kTab);
    tm->seq_jump.alloc(2 * kTab);
    CK(cudaMemcpy(tm->seq_jump.ptr, host.data(), host.size() * 4, cudaMemcpyHostToDevice));
  }
}

// The W = 1 replay (train_mirror_kernel) draws a Type I step's 2o uniforms
// by jump-ahead once 2o is large enough for 32 matrix applications to beat
// 2o serial draws. TMG_SEQ_SERIAL=1 keeps them serial (A/B checks).
void mirror_jumps(tmg_machine* tm, tmg::MirrorParams& mp) {
  const char* e = std::getenv("TMG_SEQ_SERIAL");
  if ((e && e[0] == '1') || 2 * tm->o < 256) return;
  ensure_jumps(tm);
  mp.jump_chunk = tm->seq_jump.ptr;
  mp.jump_lits = tm->seq_jump.ptr + tmg::kGf2TabWords;
  mp.chunk = (2 * tm->o + 31) / 32;
}

// Fills the parallel-replay fields of sp (matrices cached on the machine).
void seq_jumps(tmg_machine* tm, tmg::SeqParams& sp) {
  const int L = 2 * tm->o;
  const int chunk = (L + 31) / 32;
  ensure_jumps(tm);
  if (tm->seq_tstate.count != static_cast<size_t>(tm->n) * 4) tm->seq_tstate.alloc(static_cast<size_t>(tm->n) * 4);
  sp.jump_chunk = tm->seq_jump.ptr;
  sp.jump_lits = tm->seq_jump.ptr + tmg::kGf2TabWords;
  sp.chunk = chunk;
  sp.tstate = tm->seq_tstate.ptr;
  if (seq_grid_enabled()) {
    const size_t nwords = (static_cast<size_t>(tm->n) + 31) / 32;
    if (tm->seq_scratch.count != 3 * nwords + 3) tm->seq_scratch.alloc(3 * nwords + 3);
    CK(cudaMemsetAsync(tm->seq_scratch.ptr, 0, tm->seq_scratch.bytes(), tm->stream));
    sp.g_outs = tm->seq_scratch.ptr;
    sp.g_gbits = tm->seq_scratch.ptr + 2 * nwords;
    sp.g_misc = reinterpret_cast<int32_t*>(tm->seq_scratch.ptr + 3 * nwords);
  }
}

void epoch_keys(tmg_machine* tm, int32_t epoch) {
  // Philox key per (seed, epoch); stream kind 4 is disjoint from the
  // reference's kinds 1-3 (trainer.cpp:29-31).
  const uint64_t k = tmg_mix_stream(4, static_cast<uint64_t>(epoch), tm->cfg.seed);
  tm->key0 = static_cast<uint32_t>(k);
  tm->key1 = static_cast<uint32_t>(k >> 32);
  tm->cur_epoch = epoch;
}

void run_async_window(tmg_machine* tm, tmg_pool* pool, int64_t t0, int64_t t1, bool with_delta, int w_begin,
                      int w_end) {
  tmg::TrainParams p = make_params(tm, pool);
  p.t_begin = t0;
  p.t_end = t1;
  if (w_end >= 0) {  // one wave of the clause order
    p.w_begin = w_begin;
    p.w_end = w_end;
  }
  if (with_delta && !pool->peers.empty())
    fail(TMG_EINVAL, "pool has peer tally replicas attached: the windowed exchange would count every change twice "
                     "(detach with tmg_pool_set_peers(pool, NULL, 0))");
  if (with_delta) p.tally_delta = pool->delta.ptr;
  int blocks = 0;
  // Register-resident clauses up to 4 words per lane per part (o <= 4096);
  // wider rows keep the automata in shared memory (FMNIST's 3-word rows on
  // the shared-memory kernel: 1203 vs 627 ms, round 2). (A variant splitting each
  // wide clause over 2-4 warps with register-resident slices measured 3-11 %
  // slower at IMDb shape, round 1, and was dropped.)
  const bool ok = tm->NW <= 4 ? tmg::train_async_launch(p, tm->B, tm->NW, tm->stream, &blocks)
                              : tmg::train_async_smem_launch(p, tm->B, tm->NW, tm->stream, &blocks);
  if (!ok) fail(TMG_ERUNTIME, "no async kernel instantiation for this shape");
  CK(cudaGetLastError());
  tm->entries_dirty = true;
}

int resident_clause_warps(tmg_machine* tm, tmg_pool* pool, int* warps_per_cta) {
  const tmg::TrainParams p = make_params(tm, pool);
  DeviceGuard dg(tm->device);
  return tmg::train_async_resident_warps(p, tm->B, tm->NW, warps_per_cta);
}

// Class sums of q literal rows (x-plane words at xplane, row stride 2*Wp)
// into d_out [q][m]; train mode writes previous-output bitmaps to prev when
// given. lit_t: the rows' feature-major columns if already built (pools cache
// theirs), else they are built into the machine's scratch.
void class_sums_device(tmg_machine* tm, const uint32_t* xplane, int64_t q, bool train_mode, int32_t* d_out,
                       uint32_t* prev, const uint32_t* lit_t) {
  rebuild_entries(tm);
  const int64_t Gs = tmg::lit_t_stride(q);
  if (!lit_t) {
    const size_t need = static_cast<size_t>(tm->o + 2) * Gs;
    if (tm->lit_t.count < need) tm->lit_t.alloc(need);
    tmg::transpose_literals_launch(xplane, 2 * tm->Wp, q, tm->o, tm->lit_t.ptr, tm->stream);
    lit_t = tm->lit_t.ptr;
  }
  tmg::BitsEvalParams e{};
  e.lit_t = lit_t;
  e.Gs = static_cast<uint32_t>(Gs);
  e.lists = tm->lists.ptr;
  e.meta = tm->meta.ptr;
  e.prev = prev;
  e.n_loc = tm->n_loc;
  e.j_begin = tm->j_begin;
  e.m = tm->m;
  e.Wq = tm->Wq;
  e.q = q;
  e.sums = d_out;
  e.all_positive = tm->all_positive;
  // 2 to 6 resident waves of 5 CTAs (40 warps) per SM, by the literal loads
  // to do (~1k per warp and wave); at most 2040 clauses per CTA (the
  // bit-sliced counters' range), >= 4 per warp.
  const int64_t blocks = (q + 1023) / 1024;
  const int64_t resident = int64_t(148) * 5;
  const int64_t steps = blocks * tm->lists_total;  // warp-level literal loads
  const char* wv = std::getenv("TMG_EVAL_MINWAVES");
  const int64_t min_waves = wv ? std::atoi(wv) : 3;
  const int64_t waves = std::min<int64_t>(6, std::max<int64_t>(min_waves, steps / (resident * 8 * 1024)));
  int64_t chunks = (resident * waves + blocks * tm->m - 1) / (blocks * tm->m);
  chunks = std::max<int64_t>(chunks, (tm->n_loc + 2039) / 2040);
  chunks = std::min<int64_t>(chunks, std::max(1, tm->n_loc / 32));
  chunks = std::max<int64_t>(chunks, (tm->n_loc + 2039) / 2040);
  chunks = std::min<int64_t>(chunks, 65535 / tm->m);
  e.cta_clauses = static_cast<int32_t>((tm->n_loc + chunks - 1) / chunks);
  {
    const char* dyn = std::getenv("TMG_EVAL_DYNAMIC");
    const int64_t avg = tm->lists_total / std::max(1, tm->clauses());
    e.dynamic = dyn ? (dyn[0] == '1') : (avg > 16 ? 1 : 0);
  }
  e.chunks = static_cast<int32_t>((tm->n_loc + e.cta_clauses - 1) / e.cta_clauses);
  CK(cudaMemsetAsync(d_out, 0, static_cast<size_t>(q) * tm->m * 4, tm->stream));
  if (!tm->eval0) {
    CK(cudaEventCreate(&tm->eval0));
    CK(cudaEventCreate(&tm->eval1));
  }
  CK(cudaEventRecord(tm->eval0, tm->stream));
  tmg::eval_bits_launch(e, train_mode, tm->stream);
  CK(cudaEventRecord(tm->eval1, tm->stream));
  CK(cudaGetLastError());
}

const uint32_t* pool_lit_t(tmg_machine* tm, const tmg_pool* pool) {
  if (!pool->lit_t.ptr) {
    pool->lit_t.alloc(static_cast<size_t>(pool->o + 2) * tmg::lit_t_stride(pool->q));
    tmg::transpose_literals_launch(pool->xplane(), 2 * pool->Wp, pool->q, pool->o, pool->lit_t.ptr, tm->stream);
    CK(cudaGetLastError());
  }
  return pool->lit_t.ptr;
}

void ensure_sums(tmg_machine* tm, int64_t q) {
  if (tm->sums.count < static_cast<size_t>(q) * tm->m) tm->sums.alloc(static_cast<size_t>(q) * tm->m);
}

tmg_pool* create_pool_common(int device, int o, int64_t q, int m) {
  if (o < 1) fail(TMG_EINVAL, "feature count must be >= 1");
  if (m < 1) fail(TMG_EINVAL, "class count must be >= 1");
  if (q <= 0) fail(TMG_EINVAL, "example pool must not be empty");
  if (q > (int64_t(1) << 31) - 64) fail(TMG_EINVAL, "example pool too large");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) fail(TMG_EINVAL, "no such CUDA device " + std::to_string(device));
  auto pool = new tmg_pool();
  pool->device = device;
  pool->o = o;
  pool->m = m;
  pool->q = q;
  pool->Wp = wp_for(o);
  return pool;
}

void finish_pool(tmg_pool* pool, const uint8_t* d_bits, const int32_t* d_labels) {
  const size_t rows = static_cast<size_t>(pool->q);
  pool->rows.alloc(rows * 2 * pool->Wp);
  pool->labels.alloc(rows);
  pool->tallies.alloc(rows * pool->m);
  pool->delta.alloc(rows * pool->m);
  pool->order.alloc(rows);
  // Pack and validate on the device (ExamplePool ctor checks, pool.cpp:40-55).
  DevBuf<int> err;
  err.alloc(2);
  CK(cudaMemsetAsync(err.ptr, 0, 8, pool->stream));
  tmg::pack_planes_launch(d_bits, pool->xplane(), pool->nplane(), pool->q, pool->o, pool->Wp, err.ptr,
                          pool->stream);
  CK(cudaGetLastError());
  if (pool->m > 1) tmg::check_labels_launch(d_labels, pool->q, pool->m, err.ptr, pool->stream);
  CK(cudaMemcpyAsync(pool->labels.ptr, d_labels, rows * 4, cudaMemcpyDeviceToDevice, pool->stream));
  CK(cudaMemsetAsync(pool->tallies.ptr, 0, pool->tallies.bytes(), pool->stream));  // pool.cpp:71
  CK(cudaMemsetAsync(pool->delta.ptr, 0, pool->delta.bytes(), pool->stream));
  int herr[2] = {0, 0};
  CK(cudaMemcpyAsync(herr, err.ptr, 8, cudaMemcpyDeviceToHost, pool->stream));
  CK(cudaStreamSynchronize(pool->stream));
  err.release();
  if (herr[0] & 1) fail(TMG_EINVAL, "inputs must be 0/1");
  if (herr[0] & 2)
    fail(TMG_EINVAL, "label " + std::to_string(herr[1]) + " outside [0, " + std::to_string(pool->m) + ")");
}

tmg_machine* M(tmg_machine* tm) {
  if (!tm) fail(TMG_EINVAL, "null machine handle");
  return tm;
}
const tmg_machine* M(const tmg_machine* tm) {
  if (!tm) fail(TMG_EINVAL, "null machine handle");
  return tm;
}

void check_bank(const tmg_machine* tm, int32_t bank) {
  if (bank < 0 || bank >= tm->m) fail(TMG_ERANGE, "bank index out of range");
}

}  // namespace tmgx

// ===================================================================== ABI ===

TMG_API int tmg_abi_version(void) { return TMG_ABI_VERSION; }
TMG_API const char* tmg_last_error(void) { return g_last_error.c_str(); }

TMG_API int tmg_device_count(int32_t* count) {
  return guarded([&] {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    *count = n;
  });
}

TMG_API void tmg_config_default(tmg_config* cfg) {
  cfg->clauses = 100;
  cfg->margin = 15;
  cfg->specificity = 3.0;
  cfg->state_depth = 128;
  cfg->boost_true_positive = 0;
  cfg->epochs = 100;
  cfg->workers = 0;
  cfg->seed = 42;
}

TMG_API int tmg_config_validate(const tmg_config* cfg) {
  return guarded([&] {
    if (!cfg) fail(TMG_EINVAL, "null config");
    validate_config(*cfg);
  });
}

TMG_API int32_t tmg_effective_workers(const tmg_config* cfg) {
  if (cfg->workers > 0) return cfg->workers;
  return 1;  // the GPU engine's parallelism is the device, not host threads
}

TMG_API int tmg_machine_create(const tmg_config* cfg, int32_t o, int32_t m, int32_t device, tmg_machine** out) {
  return guarded([&] { *out = create_machine(cfg, o, m, device, 0, cfg ? cfg->clauses : 0); });
}

TMG_API int tmg_machine_create_shard(const tmg_config* cfg, int32_t o, int32_t m, int32_t device, int32_t jb,
                                     int32_t je, tmg_machine** out) {
  return guarded([&] { *out = create_machine(cfg, o, m, device, jb, je); });
}

TMG_API int tmg_machine_destroy(tmg_machine* tm) {
  if (!tm) return TMG_OK;
  if (is_group(tm) || tm->owns_xchg) destroy_group(tm);
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(tm->device);
  if (tm->stream) cudaStreamSynchronize(tm->stream);
  tm->state.release();
  tm->prev.release();
  tm->inc_count.release();
  tm->lens.release();
  tm->npos.release();
  tm->meta.release();
  tm->offs.release();
  tm->lit_t.release();
  tm->sums.release();
  tm->lists.release();
  tm->events.release();
  tm->dbg.release();
  tm->work.release();
  tm->alias8.release();
  tm->scratch16.release();
  if (tm->eval0) cudaEventDestroy(tm->eval0);
  if (tm->eval1) cudaEventDestroy(tm->eval1);
  if (tm->ev0) cudaEventDestroy(tm->ev0);
  if (tm->ev1) cudaEventDestroy(tm->ev1);
  if (tm->stream) cudaStreamDestroy(tm->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete tm;
  return TMG_OK;
}

TMG_API int tmg_machine_info_get(const tmg_machine* tm, tmg_machine_info* info) {
  if (is_group(tm)) return group_info(tm, info);
  return guarded([&] {
    M(tm);
    info->feature_count = tm->o;
    info->num_classes = tm->m;
    info->clauses = tm->n;
    info->state_depth = tm->N;
    info->clause_begin = tm->j_begin;
    info->clause_end = tm->j_end;
    info->planes = tm->B;
    info->words_per_lane = tm->NW;
    info->bound_examples = static_cast<int32_t>(tm->q_bound);
    info->device = tm->device;
    info->device_bytes = tm->state.bytes() + tm->prev.bytes() + tm->inc_count.bytes() + tm->lists.bytes() +
                         tm->lens.bytes() + tm->npos.bytes() + tm->offs.bytes() + tm->lit_t.bytes() + tm->sums.bytes();
  });
}

TMG_API int tmg_machine_config(const tmg_machine* tm, tmg_config* cfg) {
  return guarded([&] { *cfg = M(tm)->cfg; });
}

TMG_API int tmg_machine_reset(tmg_machine* tm) {
  if (is_group(tm)) return group_reset(tm);
  return guarded([&] {
    DeviceGuard dg(M(tm)->device);
    reset_state(tm);
  });
}

TMG_API int tmg_get_counters(const tmg_machine* ctm, int32_t bank, uint16_t* out) {
  if (is_group(ctm)) return group_counters(ctm, bank, out, nullptr);
  return guarded([&] {
    auto tm = const_cast<tmg_machine*>(M(ctm));
    check_bank(tm, bank);
    DeviceGuard dg(tm->device);
    const size_t count = static_cast<size_t>(tm->n_loc) * 2 * tm->o;
    if (tm->scratch16.count < count) tm->scratch16.alloc(count);
    tmg::planes_to_counters_launch(tm->state.ptr + static_cast<size_t>(bank) * tm->n_loc * tm->B * 2 * tm->Wp,
                                   tm->scratch16.ptr, tm->n_loc, tm->o, tm->B, tm->Wp, tm->N, tm->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, tm->scratch16.ptr, count * 2, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_set_counters(tmg_machine* tm, int32_t bank, const uint16_t* in) {
  if (is_group(tm)) return group_counters(tm, bank, nullptr, in);
  return guarded([&] {
    check_bank(M(tm), bank);
    DeviceGuard dg(tm->device);
    const size_t count = static_cast<size_t>(tm->n_loc) * 2 * tm->o;
    for (size_t k = 0; k < count; ++k)
      if (in[k] < 1 || in[k] > 2 * tm->N)
        fail(TMG_EINVAL, "automaton counter outside [1, 2N]");
    if (tm->scratch16.count < count) tm->scratch16.alloc(count);
    CK(cudaMemcpyAsync(tm->scratch16.ptr, in, count * 2, cudaMemcpyHostToDevice, tm->stream));
    tmg::counters_to_planes_launch(tm->scratch16.ptr,
                                   tm->state.ptr + static_cast<size_t>(bank) * tm->n_loc * tm->B * 2 * tm->Wp,
                                   tm->n_loc, tm->o, tm->B, tm->Wp, tm->N, tm->stream);
    CK(cudaGetLastError());
    tm->entries_dirty = true;
    rebuild_entries(tm);  // refreshes include counts too
    CK(cudaStreamSynchronize(tm->stream));
  });
}

namespace {
std::vector<uint32_t> top_planes(tmg_machine* tm, int32_t bank) {
  // [n_loc][2][Wp] include bits of one bank.
  std::vector<uint32_t> out(static_cast<size_t>(tm->n_loc) * 2 * tm->Wp);
  const size_t stride = static_cast<size_t>(tm->B) * 2 * tm->Wp;
  for (int jl = 0; jl < tm->n_loc; ++jl) {
    const uint32_t* src = tm->state.ptr + (static_cast<size_t>(bank) * tm->n_loc + jl) * stride +
                          static_cast<size_t>(tm->B - 1) * 2 * tm->Wp;
    CK(cudaMemcpyAsync(out.data() + static_cast<size_t>(jl) * 2 * tm->Wp, src, 2 * tm->Wp * 4,
                       cudaMemcpyDeviceToHost, tm->stream));
  }
  CK(cudaStreamSynchronize(tm->stream));
  return out;
}
}  // namespace

TMG_API int tmg_get_include_masks(const tmg_machine* ctm, int32_t bank, uint64_t* out) {
  if (is_group(ctm)) return group_include(ctm, bank, out, nullptr);
  return guarded([&] {
    auto tm = const_cast<tmg_machine*>(M(ctm));
    check_bank(tm, bank);
    DeviceGuard dg(tm->device);
    const auto top = top_planes(tm, bank);
    const int W64 = (2 * tm->o + 63) / 64;
    for (int jl = 0; jl < tm->n_loc; ++jl) {
      uint64_t* row = out + static_cast<size_t>(jl) * W64;
      std::fill(row, row + W64, 0);
      const uint32_t* t = top.data() + static_cast<size_t>(jl) * 2 * tm->Wp;
      for (int part = 0; part < 2; ++part)
        for (int f = 0; f < tm->o; ++f)
          if ((t[part * tm->Wp + (f >> 5)] >> (f & 31)) & 1u) {
            const int k = part * tm->o + f;
            row[k >> 6] |= 1ULL << (k & 63);
          }
    }
  });
}

TMG_API int tmg_get_include_counts(const tmg_machine* ctm, int32_t bank, int32_t* out) {
  if (is_group(ctm)) return group_include(ctm, bank, nullptr, out);
  return guarded([&] {
    auto tm = const_cast<tmg_machine*>(M(ctm));
    check_bank(tm, bank);
    DeviceGuard dg(tm->device);
    rebuild_entries(tm);
    CK(cudaMemcpyAsync(out, tm->inc_count.ptr + static_cast<size_t>(bank) * tm->n_loc, tm->n_loc * 4,
                       cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_bind_examples(tmg_machine* tm, int64_t q) {
  if (is_group(tm)) return group_bind(tm, -1, q);
  return guarded([&] {
    DeviceGuard dg(M(tm)->device);
    bind(tm, q);
  });
}

TMG_API int tmg_bind_bank(tmg_machine* tm, int32_t bank, int64_t q) {
  if (is_group(tm)) return group_bind(tm, bank, q);
  return guarded([&] {
    check_bank(M(tm), bank);
    DeviceGuard dg(tm->device);
    bind_bank(tm, bank, q);
  });
}

TMG_API int tmg_bank_bound_examples(const tmg_machine* tm, int32_t bank, int64_t* q) {
  if (is_group(tm)) return tmg_bank_bound_examples(tm->parts[0], bank, q);
  return guarded([&] {
    check_bank(M(tm), bank);
    *q = tm->bank_q[static_cast<size_t>(bank)];
  });
}

// Previous outputs of one bank in the reference layout: per clause
// ceil(bound/64) u64 words (the device rows are Wq u32 words apart).
TMG_API int tmg_get_prev_outputs(const tmg_machine* ctm, int32_t bank, uint64_t* out) {
  if (is_group(ctm)) return group_prev(ctm, bank, out, nullptr);
  return guarded([&] {
    auto tm = const_cast<tmg_machine*>(M(ctm));
    check_bank(tm, bank);
    DeviceGuard dg(tm->device);
    const size_t w = 2 * static_cast<size_t>((tm->bank_q[static_cast<size_t>(bank)] + 63) / 64);
    const size_t rows = static_cast<size_t>(tm->n_loc);
    if (w && rows)
      CK(cudaMemcpy2DAsync(out, w * 4, tm->prev.ptr + static_cast<size_t>(bank) * rows * tm->Wq,
                           static_cast<size_t>(tm->Wq) * 4, w * 4, rows, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_set_prev_outputs(tmg_machine* tm, int32_t bank, const uint64_t* in) {
  if (is_group(tm)) return group_prev(tm, bank, nullptr, in);
  return guarded([&] {
    check_bank(M(tm), bank);
    DeviceGuard dg(tm->device);
    const size_t w = 2 * static_cast<size_t>((tm->bank_q[static_cast<size_t>(bank)] + 63) / 64);
    const size_t rows = static_cast<size_t>(tm->n_loc);
    if (w && rows)
      CK(cudaMemcpy2DAsync(tm->prev.ptr + static_cast<size_t>(bank) * rows * tm->Wq, static_cast<size_t>(tm->Wq) * 4,
                           in, w * 4, w * 4, rows, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

// ------------------------------------------------------------------ pool ---

TMG_API int tmg_pool_create(int32_t device, int32_t o, const uint8_t* bits, const int32_t* labels, int64_t q,
                            int32_t m, tmg_pool** out) {
  return guarded([&] {
    tmg_pool* pool = create_pool_common(device, o, q, m);
    try {
      DeviceGuard dg(device);
      CK(cudaStreamCreateWithFlags(&pool->stream, cudaStreamNonBlocking));
      DevBuf<uint8_t> dbits;
      DevBuf<int32_t> dlab;
      dbits.alloc(static_cast<size_t>(q) * o);
      dlab.alloc(static_cast<size_t>(q));
      CK(cudaMemcpyAsync(dbits.ptr, bits, dbits.bytes(), cudaMemcpyHostToDevice, pool->stream));
      CK(cudaMemcpyAsync(dlab.ptr, labels, dlab.bytes(), cudaMemcpyHostToDevice, pool->stream));
      finish_pool(pool, dbits.ptr, dlab.ptr);
      dbits.release();
      dlab.release();
      pool->host_labels.assign(labels, labels + q);
    } catch (...) {
      tmg_pool_destroy(pool);
      throw;
    }
    *out = pool;
  });
}

TMG_API int tmg_pool_create_device(int32_t device, int32_t o, const uint8_t* d_bits, const int32_t* d_labels,
                                   int64_t q, int32_t m, tmg_pool** out) {
  return guarded([&] {
    tmg_pool* pool = create_pool_common(device, o, q, m);
    try {
      DeviceGuard dg(device);
      CK(cudaStreamCreateWithFlags(&pool->stream, cudaStreamNonBlocking));
      finish_pool(pool, d_bits, d_labels);
    } catch (...) {
      tmg_pool_destroy(pool);
      throw;
    }
    *out = pool;
  });
}

TMG_API int tmg_pool_destroy(tmg_pool* pool) {
  if (!pool) return TMG_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(pool->device);
  if (pool->stream) cudaStreamSynchronize(pool->stream);
  pool->close_peers();
  destroy_replicas(pool);
  pool->rows.release();
  pool->labels.release();
  pool->tallies.release();
  pool->delta.release();
  pool->order.release();
  if (pool->stream) cudaStreamDestroy(pool->stream);
  if (prev >= 0) cudaSetDevice(prev);
  delete pool;
  return TMG_OK;
}

TMG_API int tmg_pool_size(const tmg_pool* pool, int64_t* q) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    *q = pool->q;
  });
}

TMG_API int tmg_pool_get_literals(const tmg_pool* pool, uint64_t* out) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    DeviceGuard dg(pool->device);
    const size_t rows = static_cast<size_t>(pool->q);
    std::vector<uint32_t> rw(rows * 2 * pool->Wp);
    CK(cudaMemcpyAsync(rw.data(), pool->xplane(), rw.size() * 4, cudaMemcpyDeviceToHost, pool->stream));
    CK(cudaStreamSynchronize(pool->stream));
    const int o = pool->o, W64 = (2 * o + 63) / 64;
    for (size_t i = 0; i < rows; ++i) {
      uint64_t* row = out + i * W64;
      std::fill(row, row + W64, 0);
      const uint32_t* xs = rw.data() + i * 2 * pool->Wp;
      const uint32_t* ns = xs + pool->Wp;
      for (int f = 0; f < o; ++f) {
        if ((xs[f >> 5] >> (f & 31)) & 1u) row[f >> 6] |= 1ULL << (f & 63);
        if ((ns[f >> 5] >> (f & 31)) & 1u) row[(o + f) >> 6] |= 1ULL << ((o + f) & 63);
      }
    }
  });
}

TMG_API int tmg_pool_get_tallies(const tmg_pool* pool, int32_t* out) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    DeviceGuard dg(pool->device);
    CK(cudaMemcpyAsync(out, pool->tallies.ptr, pool->tallies.bytes(), cudaMemcpyDeviceToHost, pool->stream));
    CK(cudaStreamSynchronize(pool->stream));
  });
}

TMG_API int tmg_pool_set_tallies(tmg_pool* pool, const int32_t* in) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    DeviceGuard dg(pool->device);
    CK(cudaMemcpyAsync(pool->tallies.ptr, in, pool->tallies.bytes(), cudaMemcpyHostToDevice, pool->stream));
    CK(cudaStreamSynchronize(pool->stream));
  });
}

TMG_API int tmg_pool_reset_tallies(tmg_pool* pool) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    DeviceGuard dg(pool->device);
    CK(cudaMemsetAsync(pool->tallies.ptr, 0, pool->tallies.bytes(), pool->stream));
    CK(cudaMemsetAsync(pool->delta.ptr, 0, pool->delta.bytes(), pool->stream));
    CK(cudaStreamSynchronize(pool->stream));
  });
}

// Host check of the jump-ahead matrices (sequential.cu / draw_type_i_bits):
// state <- M^k state for the xoshiro256 state update.
TMG_API int tmg_debug_xoshiro_jump(uint64_t* state, uint64_t k) {
  return guarded([&] {
    if (!state) fail(TMG_EINVAL, "null state");
    const Gf2 m = gf2_pow(k);
    uint64_t out[4] = {0, 0, 0, 0};
    for (int i = 0; i < 256; ++i) {
      uint64_t acc = 0;
      for (int w = 0; w < 4; ++w) acc ^= m.r[i][w] & state[w];
      if (__builtin_popcountll(acc) & 1) out[i >> 6] |= uint64_t(1) << (i & 63);
    }
    for (int w = 0; w < 4; ++w) state[w] = out[w];
  });
}

TMG_API int tmg_pool_tally_ipc_handle(tmg_pool* pool, unsigned char* handle) {
  return guarded([&] {
    if (!pool || !handle) fail(TMG_EINVAL, "null argument");
    DeviceGuard dg(pool->device);
    CK(cudaStreamSynchronize(pool->stream));
    if (!pool->tallies.plain && pool->tallies.count) {  // move the replica to exportable memory
      DevBuf<int32_t> t;
      t.alloc_plain(pool->tallies.count);
      CK(cudaMemcpy(t.ptr, pool->tallies.ptr, t.bytes(), cudaMemcpyDeviceToDevice));
      pool->tallies.swap(t);
    }
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, pool->tallies.ptr));
    std::memcpy(handle, &h, sizeof(h));
  });
}

TMG_API int tmg_pool_set_peers(tmg_pool* pool, const unsigned char* handles, int32_t npeers) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    if (npeers < 0 || npeers > tmg::kMaxPeers)
      fail(TMG_EINVAL, "peer count must be in [0, " + std::to_string(tmg::kMaxPeers) + "]");
    if (npeers > 0 && !handles) fail(TMG_EINVAL, "null handles");
    DeviceGuard dg(pool->device);
    CK(cudaStreamSynchronize(pool->stream));
    pool->close_peers();
    for (int k = 0; k < npeers; ++k) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + static_cast<size_t>(k) * sizeof(h), sizeof(h));
      void* ptr = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        pool->close_peers();
        fail(TMG_ERUNTIME, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      pool->peers.push_back(static_cast<int32_t*>(ptr));
    }
  });
}

TMG_API int tmg_pool_tally_device_ptr(tmg_pool* pool, void** ptr) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    *ptr = pool->tallies.ptr;
  });
}

TMG_API int tmg_pool_delta_device_ptr(tmg_pool* pool, void** ptr) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    *ptr = pool->delta.ptr;
  });
}

TMG_API int tmg_pool_apply_reduced(tmg_pool* pool, const void* d_reduced) {
  return guarded([&] {
    if (!pool) fail(TMG_EINVAL, "null pool handle");
    DeviceGuard dg(pool->device);
    tmg::apply_remote_delta_launch(pool->tallies.ptr, static_cast<const int32_t*>(d_reduced), pool->delta.ptr,
                                   pool->q * pool->m, pool->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(pool->stream));
  });
}

// -------------------------------------------------------------- training ---

TMG_API int tmg_epoch_begin(tmg_machine* tm, tmg_pool* pool, int32_t epoch) {
  return guarded([&] {
    need_single(tm, "tmg_epoch_begin");
    check_compatible(M(tm), pool);
    DeviceGuard dg(tm->device);
    bind_for(tm, pool->q);
    upload_order(tm, pool, epoch);
    epoch_keys(tm, epoch);
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
  });
}

TMG_API int tmg_train_window_async(tmg_machine* tm, tmg_pool* pool, int32_t epoch, int64_t t0, int64_t t1) {
  return guarded([&] {
    need_single(tm, "tmg_train_window_async");
    check_compatible(M(tm), pool);
    if (tm->cur_epoch != epoch || tm->q_bound != pool->q) fail(TMG_EINVAL, "call tmg_epoch_begin first");
    if (t0 < 0 || t1 > pool->q || t0 > t1) fail(TMG_ERANGE, "window outside [0, q]");
    DeviceGuard dg(tm->device);
    run_async_window(tm, pool, t0, t1, true);
  });
}

TMG_API int tmg_window_delta_snapshot(tmg_machine* tm, tmg_pool* pool, void* d_snapshot) {
  return guarded([&] {
    need_single(tm, "tmg_window_delta_snapshot");
    check_compatible(M(tm), pool);
    if (!d_snapshot) fail(TMG_EINVAL, "null snapshot buffer");
    DeviceGuard dg(tm->device);
    CK(cudaMemcpyAsync(d_snapshot, pool->delta.ptr, pool->delta.bytes(), cudaMemcpyDeviceToDevice, tm->stream));
    CK(cudaMemsetAsync(pool->delta.ptr, 0, pool->delta.bytes(), tm->stream));
  });
}

TMG_API int tmg_window_apply_remote(tmg_machine* tm, tmg_pool* pool, const void* d_reduced, const void* d_snapshot) {
  return guarded([&] {
    need_single(tm, "tmg_window_apply_remote");
    check_compatible(M(tm), pool);
    if (!d_reduced || !d_snapshot) fail(TMG_EINVAL, "null buffer");
    DeviceGuard dg(tm->device);
    tmg::apply_snapshot_launch(pool->tallies.ptr, static_cast<const int32_t*>(d_reduced),
                               static_cast<const int32_t*>(d_snapshot), pool->q * pool->m, tm->stream);
    CK(cudaGetLastError());
  });
}

TMG_API int tmg_epoch_events(tmg_machine* tm, uint64_t* feedback_events) {
  return guarded([&] {
    need_single(tm, "tmg_epoch_events");
    DeviceGuard dg(M(tm)->device);
    std::vector<unsigned long long> ev(2 * static_cast<size_t>(tm->m));
    CK(cudaMemcpyAsync(ev.data(), tm->events.ptr, tm->events.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    if (feedback_events)
      for (int c = 0; c < tm->m; ++c) feedback_events[c] = ev[static_cast<size_t>(c)];
  });
}

TMG_API int tmg_train_window(tmg_machine* tm, tmg_pool* pool, int32_t epoch, int64_t t0, int64_t t1,
                             uint64_t* feedback_events) {
  return guarded([&] {
    need_single(tm, "tmg_train_window");
    check_compatible(M(tm), pool);
    if (tm->cur_epoch != epoch || tm->q_bound != pool->q) fail(TMG_EINVAL, "call tmg_epoch_begin first");
    if (t0 < 0 || t1 > pool->q || t0 > t1) fail(TMG_ERANGE, "window outside [0, q]");
    DeviceGuard dg(tm->device);
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    run_async_window(tm, pool, t0, t1, true);
    std::vector<unsigned long long> ev(2 * static_cast<size_t>(tm->m));
    CK(cudaMemcpyAsync(ev.data(), tm->events.ptr, tm->events.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    if (feedback_events)
      for (int c = 0; c < tm->m; ++c) feedback_events[c] = ev[static_cast<size_t>(c)];
  });
}

static int train_epoch_impl(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                            tmg_epoch_report* report);

TMG_API int tmg_train_epoch(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                            tmg_epoch_report* report) {
  if (is_sharded(tm)) return group_train_epoch(tm, pool, mode, workers, epoch, report);
  if (tm && tm->all_positive) {
    g_last_error = "regression machine: use tmg_train_epoch_regress";
    return TMG_EINVAL;
  }
  return train_epoch_impl(tm, pool, mode, workers, epoch, report);
}

TMG_API int tmg_train_epoch_regress(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                                    tmg_epoch_report* report) {
  if (is_sharded(tm)) {
    g_last_error = "train_epoch_regress_parallel needs a single-device machine";
    return TMG_EINVAL;
  }
  // train_epoch_regress_parallel (regression.cpp:163-227)
  if (!tm || !tm->all_positive) {
    g_last_error = "not a regression machine (create it with tmg_machine_create_regress)";
    return TMG_EINVAL;
  }
  if (pool && pool->m != 1) {
    g_last_error = "regression pool must have one tally class";
    return TMG_EINVAL;
  }
  tm->regress_mode = true;
  const int rc = train_epoch_impl(tm, pool, mode, workers, epoch, report);
  tm->regress_mode = false;
  return rc;
}

// TMG_MODE_AUTO (include/tmgpu.h): one rule for every drop-in caller.
int32_t tmgx::resolve_mode(int32_t mode, int32_t workers) {
  if (mode != TMG_MODE_AUTO) return mode;
  const char* det = std::getenv("TSETLIN_DETERMINISTIC");
  return workers == 1 && det && det[0] == '1' ? TMG_MODE_SYNC_MIRROR : TMG_MODE_ASYNC;
}

static int train_epoch_impl(tmg_machine* tm, tmg_pool* pool, int32_t mode, int32_t workers, int32_t epoch,
                            tmg_epoch_report* report) {
  return guarded([&] {
    check_compatible(M(tm), pool);
    if (workers < 1) fail(TMG_EINVAL, "workers must be >= 1");  // trainer.cpp:184
    mode = resolve_mode(mode, workers);
    if (mode != TMG_MODE_ASYNC && mode != TMG_MODE_SYNC_MIRROR) fail(TMG_EINVAL, "unknown training mode");
    DeviceGuard dg(tm->device);
    const auto wall0 = std::chrono::steady_clock::now();
    bind_for(tm, pool->q);  // trainer.cpp:192-194
    upload_order(tm, pool, epoch);
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    CK(cudaEventRecord(tm->ev0, tm->stream));
    if (mode == TMG_MODE_ASYNC) {
      epoch_keys(tm, epoch);
      run_async_window(tm, pool, 0, pool->q, false);
    } else if (mode == TMG_MODE_SYNC_MIRROR) {
      if (tm->n_loc != tm->n) fail(TMG_EINVAL, "sync mirror mode needs the full (unsharded) machine");
      // Worker w owns g = w, w+W, ... (trainer.cpp:214-227), run one after another.
      std::vector<tmg::MirrorJob> jobs;
      const int64_t total = static_cast<int64_t>(tm->m) * tm->n;
      jobs.reserve(static_cast<size_t>(total));
      std::vector<uint64_t> rng(static_cast<size_t>(workers) * 4);
      for (int w = 0; w < workers; ++w) {
        tmg_rng r;
        tmg_rng_seed(&r, tm->cfg.seed,
                     tmg_mix_stream(tm->regress_mode ? 6 : TMG_STREAM_WORKER, static_cast<uint64_t>(epoch),
                                    static_cast<uint64_t>(w)));
        std::memcpy(&rng[static_cast<size_t>(w) * 4], r.s, 32);
        for (int64_t g = w; g < total; g += workers) {
          tmg::MirrorJob jb{};
          jb.c = static_cast<int32_t>(g / tm->n);
          jb.j = static_cast<int32_t>(g % tm->n);
          jb.worker = w;
          jb.offset = static_cast<int64_t>(tmg_clause_offset(static_cast<uint64_t>(g), pool->q));
          jb.batch = pool->q;
          jobs.push_back(jb);
        }
      }
      DevBuf<tmg::MirrorJob> djobs;
      DevBuf<uint64_t> drng;
      djobs.alloc(jobs.size());
      drng.alloc(rng.size());
      CK(cudaMemcpyAsync(djobs.ptr, jobs.data(), djobs.bytes(), cudaMemcpyHostToDevice, tm->stream));
      CK(cudaMemcpyAsync(drng.ptr, rng.data(), drng.bytes(), cudaMemcpyHostToDevice, tm->stream));
      tmg::TrainParams p = make_params(tm, pool);
      tmg::MirrorParams mp{};
      mp.jobs = djobs.ptr;
      mp.njobs = static_cast<int32_t>(jobs.size());
      mp.rng = drng.ptr;
      mp.p_high = (tm->cfg.specificity - 1.0) / tm->cfg.specificity;
      mp.p_low = 1.0 / tm->cfg.specificity;
      mirror_jumps(tm, mp);
      if (!tmg::train_mirror_launch(p, mp, tm->B, tm->NW, tm->stream))
        fail(TMG_ERUNTIME, "no mirror kernel instantiation for this shape");
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(tm->stream));
      tm->entries_dirty = true;
    } else {
      fail(TMG_EINVAL, "unknown training mode");
    }
    CK(cudaEventRecord(tm->ev1, tm->stream));
    std::vector<unsigned long long> ev(2 * static_cast<size_t>(tm->m));
    CK(cudaMemcpyAsync(ev.data(), tm->events.ptr, tm->events.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, tm->ev0, tm->ev1));
    if (report) {
      report->epoch = epoch;
      report->device_seconds = ms * 1e-3;
      double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
      report->seconds = secs > 0 ? secs : 1e-9;
      if (report->feedback_events)
        for (int c = 0; c < tm->m; ++c) report->feedback_events[c] = ev[static_cast<size_t>(c)];
      if (report->type_i_events)
        for (int c = 0; c < tm->m; ++c)
          report->type_i_events[c] = mode == TMG_MODE_ASYNC ? ev[static_cast<size_t>(tm->m + c)] : 0;
    }
  });
}

TMG_API int tmg_train_epoch_regress_sequential(tmg_machine* tm, tmg_pool* pool, int32_t epoch, double* seconds,
                                               uint64_t* feedback_events) {
  if (is_sharded(tm)) {
    g_last_error = "train_epoch_regress_sequential needs a single-device machine";
    return TMG_EINVAL;
  }
  // train_epoch_regress_sequential (regression.cpp:125-161)
  if (!tm || !tm->all_positive) {
    g_last_error = "not a regression machine (create it with tmg_machine_create_regress)";
    return TMG_EINVAL;
  }
  tm->regress_mode = true;
  const int rc = tmg_train_epoch_sequential(tm, pool, epoch, seconds, feedback_events);
  tm->regress_mode = false;
  return rc;
}

TMG_API int tmg_train_epoch_sequential(tmg_machine* tm, tmg_pool* pool, int32_t epoch, double* seconds,
                                       uint64_t* feedback_events) {
  return guarded([&] {
    need_single(tm, "train_epoch_sequential");
    if (tm && tm->regress_mode) {
      if (!pool || tm->o != pool->o) fail(TMG_EINVAL, "head/pool feature count mismatch");
      if (tm->device != pool->device) fail(TMG_EINVAL, "model and pool live on different devices");
    } else {
      check_compatible(M(tm), pool);
      if (tm->all_positive) fail(TMG_EINVAL, "regression machine: use tmg_train_epoch_regress_sequential");
      if (tm->m < 2) fail(TMG_EINVAL, "classification needs at least two banks");  // trainer.cpp:141-143
    }
    if (tm->n_loc != tm->n) fail(TMG_EINVAL, "the sequential trainer needs the full (unsharded) machine");
    DeviceGuard dg(tm->device);
    const auto wall0 = std::chrono::steady_clock::now();
    // Rng(seed, mix_stream(1, epoch)) shuffles, then keeps feeding the epoch
    // (regression: stream kind 4, regression.cpp:133-135).
    tmg_rng r;
    tmg_rng_seed(&r, tm->cfg.seed,
                 tmg_mix_stream(tm->regress_mode ? 4 : TMG_STREAM_SEQUENTIAL, static_cast<uint64_t>(epoch), 0));
    std::vector<int32_t> order(static_cast<size_t>(pool->q));
    tmg_shuffled_indices(static_cast<int32_t>(pool->q), &r, order.data());
    CK(cudaMemcpyAsync(pool->order.ptr, order.data(), order.size() * 4, cudaMemcpyHostToDevice, tm->stream));
    DevBuf<uint64_t> drng;
    drng.alloc(4);
    CK(cudaMemcpyAsync(drng.ptr, r.s, 32, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    tmg::TrainParams p = make_params(tm, pool);
    tmg::SeqParams sp{};
    sp.rng = drng.ptr;
    sp.p_high = (tm->cfg.specificity - 1.0) / tm->cfg.specificity;
    sp.p_low = 1.0 / tm->cfg.specificity;
    sp.events = tm->events.ptr;
    if (seq_parallel_enabled(tm)) seq_jumps(tm, sp);
    if (!tmg::train_sequential_launch(p, sp, tm->B, tm->stream)) fail(TMG_ERUNTIME, "no sequential kernel for B");
    CK(cudaGetLastError());
    std::vector<unsigned long long> ev(2 * static_cast<size_t>(tm->m));
    CK(cudaMemcpyAsync(ev.data(), tm->events.ptr, tm->events.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    tm->entries_dirty = true;
    if (feedback_events)
      for (int c = 0; c < tm->m; ++c) feedback_events[c] = ev[static_cast<size_t>(c)];
    if (seconds) {
      const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
      *seconds = secs > 0 ? secs : 1e-9;
    }
  });
}

TMG_API int tmg_debug_feedback_rates(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals,
                                     int32_t clause_output, uint32_t trials, uint64_t* inc, uint64_t* dec) {
  return guarded([&] {
    need_single(tm, "tmg_debug_feedback_rates");
    check_bank(M(tm), bank);
    if (j < tm->j_begin || j >= tm->j_end) fail(TMG_ERANGE, "clause index outside this machine");
    DeviceGuard dg(tm->device);
    const int W64 = (2 * tm->o + 63) / 64;
    DevBuf<uint64_t> dl;
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    DevBuf<unsigned long long> dinc, ddec;
    dl.alloc(W64);
    xs.alloc(2 * tm->Wp);
    dinc.alloc(2 * static_cast<size_t>(tm->o));
    ddec.alloc(2 * static_cast<size_t>(tm->o));
    CK(cudaMemcpyAsync(dl.ptr, literals, W64 * 8, cudaMemcpyHostToDevice, tm->stream));
    tmg::unpack_ref_literals_launch(dl.ptr, xs.ptr, xs.ptr + tm->Wp, 1, tm->o, tm->Wp, tm->stream);
    CK(cudaMemsetAsync(dinc.ptr, 0, dinc.bytes(), tm->stream));
    CK(cudaMemsetAsync(ddec.ptr, 0, ddec.bytes(), tm->stream));
    epoch_keys(tm, 0);
    tmg::TrainParams p{};
    // same thresholds/keys as an async epoch; literal row 0 = the given row
    tmg_pool fake;
    fake.o = tm->o;
    fake.m = tm->m;
    fake.q = 1;
    p = make_params(tm, &fake);
    p.xplane = xs.ptr;
    p.nplane = xs.ptr + tm->Wp;
    const size_t lc = static_cast<size_t>(bank) * tm->n_loc + (j - tm->j_begin);
    if (!tmg::feedback_rates_launch(p, tm->state.ptr + lc * tm->B * 2 * tm->Wp, clause_output ? 1 : 0, trials,
                                    tm->B, tm->NW, dinc.ptr, ddec.ptr, tm->stream))
      fail(TMG_EINVAL, "feedback-rate probe not instantiated for this shape");
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(inc, dinc.ptr, dinc.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaMemcpyAsync(dec, ddec.ptr, ddec.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_debug_type_i_async(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals,
                                   int32_t clause_output, uint32_t example, int32_t epoch) {
  return guarded([&] {
    need_single(tm, "tmg_debug_type_i_async");
    check_bank(M(tm), bank);
    if (j < tm->j_begin || j >= tm->j_end) fail(TMG_ERANGE, "clause index outside this machine");
    if (!literals) fail(TMG_EINVAL, "null literal row");
    DeviceGuard dg(tm->device);
    const int W64 = (2 * tm->o + 63) / 64;
    DevBuf<uint64_t> dl;
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    dl.alloc(W64);
    xs.alloc(2 * tm->Wp);
    CK(cudaMemcpyAsync(dl.ptr, literals, W64 * 8, cudaMemcpyHostToDevice, tm->stream));
    tmg::unpack_ref_literals_launch(dl.ptr, xs.ptr, xs.ptr + tm->Wp, 1, tm->o, tm->Wp, tm->stream);
    epoch_keys(tm, epoch);
    tmg_pool fake;
    fake.o = tm->o;
    fake.m = tm->m;
    fake.q = 1;
    tmg::TrainParams p = make_params(tm, &fake);
    p.xplane = xs.ptr;
    p.nplane = xs.ptr + tm->Wp;
    const size_t lc = static_cast<size_t>(bank) * tm->n_loc + (j - tm->j_begin);
    const uint32_t g = static_cast<uint32_t>(bank) * tm->n + j;
    uint32_t* st = tm->state.ptr + lc * tm->B * 2 * tm->Wp;
    const int out = clause_output ? 1 : 0;
    const bool ok = tm->NW <= 4 ? tmg::type_i_async_once_launch(p, st, g, example, out, tm->B, tm->NW, tm->stream)
                                : tmg::type_i_smem_once_launch(p, st, g, example, out, tm->B, tm->NW, tm->stream);
    if (!ok)
      fail(TMG_EINVAL, "async Type I probe not instantiated for this shape");
    CK(cudaGetLastError());
    tm->entries_dirty = true;
    rebuild_entries(tm);
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_debug_counters(tmg_machine* tm, uint64_t* out, int32_t count, int32_t reset) {
  return guarded([&] {
    need_single(tm, "tmg_debug_counters");
    M(tm);
    if (count < 0 || count > tmg::kDebugCounters) fail(TMG_EINVAL, "counter count out of range");
    DeviceGuard dg(tm->device);
    if (count) CK(cudaMemcpyAsync(out, tm->dbg.ptr, count * 8, cudaMemcpyDeviceToHost, tm->stream));
    if (reset) CK(cudaMemsetAsync(tm->dbg.ptr, 0, tm->dbg.bytes(), tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_alias8_table(uint32_t threshold, uint32_t* out) {
  return guarded([&] {
    if (!out) fail(TMG_EINVAL, "null output");
    build_alias8(threshold, out);
  });
}

TMG_API unsigned long long tmg_kernel_launches(void) {
  return __atomic_load_n(&tmg::g_launches, __ATOMIC_RELAXED);
}

TMG_API int tmg_last_eval_kernel_ms(tmg_machine* tm, float* ms) {
  return guarded([&] {
    M(tm);
    need_single(tm, "tmg_last_eval_kernel_ms");
    if (!tm->eval0) fail(TMG_EINVAL, "no class-sum kernel has run on this machine");
    DeviceGuard dg(tm->device);
    CK(cudaEventSynchronize(tm->eval1));
    CK(cudaEventElapsedTime(ms, tm->eval0, tm->eval1));
  });
}

TMG_API int tmg_machine_stream(tmg_machine* tm, void** stream) {
  if (is_group(tm)) return tmg_machine_stream(tm->parts[0], stream);
  return guarded([&] { *stream = M(tm)->stream; });
}

TMG_API int tmg_bench_int_peak(int32_t device, double* lop3_ops_per_s, double* mixed_ops_per_s) {
  return guarded([&] {
    DeviceGuard dg(device);
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (!tmg::int_peak_launch(prop.multiProcessorCount, lop3_ops_per_s, mixed_ops_per_s))
      fail(TMG_ERUNTIME, "integer peak probe failed");
  });
}

TMG_API int tmg_update_clause(tmg_machine* tm, tmg_pool* pool, int32_t c, int32_t j, const int32_t* order,
                              int64_t order_len, int64_t offset, int64_t batch, int32_t margin, double s,
                              int32_t boost, uint64_t* rng_state, uint64_t* events) {
  if (is_group(tm))
    return group_update_clause(tm, pool, c, j, order, order_len, offset, batch, margin, s, boost, rng_state, events);
  return guarded([&] {
    check_compatible(M(tm), pool);
    if (batch < 1) fail(TMG_EINVAL, "batch must be >= 1");  // trainer.cpp:106
    if (order && order_len != 0 && order_len != pool->q)
      fail(TMG_EINVAL, "example order length must equal pool size");  // trainer.cpp:109-111
    if (c < 0 || c >= tm->m) fail(TMG_ERANGE, "class index out of range");
    if (j < tm->j_begin || j >= tm->j_end) fail(TMG_ERANGE, "clause index outside this machine");
    if (offset < 0) fail(TMG_EINVAL, "offset must be >= 0");
    DeviceGuard dg(tm->device);
    if (tm->bank_q[static_cast<size_t>(c)] != pool->q) bind_bank(tm, c, pool->q);  // trainer.cpp:107
    const bool use_order = order && order_len == pool->q;
    if (use_order)  // record_output_and_tally's bounds check (pool.cpp:95-98), before any device write
      for (int64_t k = 0; k < pool->q; ++k)
        if (order[k] < 0 || order[k] >= pool->q)
          fail(TMG_ERANGE, "example index " + std::to_string(order[k]) + " out of range");
    if (use_order)
      CK(cudaMemcpyAsync(pool->order.ptr, order, pool->q * 4, cudaMemcpyHostToDevice, tm->stream));
    tmg::MirrorJob jb{};
    jb.c = c;
    jb.j = j;
    jb.worker = 0;
    jb.offset = offset % pool->q;
    jb.batch = batch;
    DevBuf<tmg::MirrorJob> djobs;
    DevBuf<uint64_t> drng;
    djobs.alloc(1);
    drng.alloc(4);
    CK(cudaMemcpyAsync(djobs.ptr, &jb, sizeof jb, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemcpyAsync(drng.ptr, rng_state, 32, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    tmg::TrainParams p = make_params(tm, pool);
    p.order = use_order ? pool->order.ptr : nullptr;
    p.margin = margin;
    p.boost = boost ? 1 : 0;
    tmg::MirrorParams mp{};
    mp.jobs = djobs.ptr;
    mp.njobs = 1;
    mp.rng = drng.ptr;
    mp.p_high = (s - 1.0) / s;
    mp.p_low = 1.0 / s;
    mirror_jumps(tm, mp);
    if (!tmg::train_mirror_launch(p, mp, tm->B, tm->NW, tm->stream))
      fail(TMG_ERUNTIME, "no mirror kernel instantiation for this shape");
    CK(cudaGetLastError());
    std::vector<unsigned long long> ev(2 * static_cast<size_t>(tm->m));
    CK(cudaMemcpyAsync(ev.data(), tm->events.ptr, tm->events.bytes(), cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaMemcpyAsync(rng_state, drng.ptr, 32, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    tm->entries_dirty = true;
    if (events) *events = ev[static_cast<size_t>(c)];
  });
}

TMG_API int tmg_feedback(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals, int32_t type,
                         double s, int32_t boost, int32_t clause_output, uint64_t* rng_state) {
  if (is_group(tm)) {  // the shard that owns clause j
    tmg_machine* part = group_owner(tm, j);
    if (!part) return guarded([&] { fail(TMG_ERANGE, "clause index outside this machine"); });
    return tmg_feedback(part, bank, j, literals, type, s, boost, clause_output, rng_state);
  }
  return guarded([&] {
    check_bank(M(tm), bank);
    if (j < tm->j_begin || j >= tm->j_end) fail(TMG_ERANGE, "clause index outside this machine");
    if (type != 1 && type != 2) fail(TMG_EINVAL, "feedback type must be 1 (Type I) or 2 (Type II)");
    DeviceGuard dg(tm->device);
    const int W64 = (2 * tm->o + 63) / 64;
    DevBuf<uint64_t> dl;
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    dl.alloc(W64);
    xs.alloc(2 * tm->Wp);
    CK(cudaMemcpyAsync(dl.ptr, literals, W64 * 8, cudaMemcpyHostToDevice, tm->stream));
    tmg::unpack_ref_literals_launch(dl.ptr, xs.ptr, xs.ptr + tm->Wp, 1, tm->o, tm->Wp, tm->stream);
    tmg::MirrorJob jb{};
    jb.c = bank;
    jb.j = j;
    jb.forced = type;
    jb.out_override = clause_output < 0 ? -1 : (clause_output ? 1 : 0);
    jb.batch = 1;
    DevBuf<tmg::MirrorJob> djobs;
    DevBuf<uint64_t> drng;
    djobs.alloc(1);
    drng.alloc(4);
    CK(cudaMemcpyAsync(djobs.ptr, &jb, sizeof jb, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemcpyAsync(drng.ptr, rng_state, 32, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    tmg::TrainParams p{};
    p.state = tm->state.ptr;
    p.inc_count = tm->inc_count.ptr;
    p.prev = tm->prev.ptr;
    p.n = tm->n;
    p.n_loc = tm->n_loc;
    p.j_begin = tm->j_begin;
    p.m = tm->m;
    p.o = tm->o;
    p.Wp = tm->Wp;
    p.Wq = tm->Wq;
    p.lo = (1u << (tm->B - 1)) - static_cast<uint32_t>(tm->N);
    p.hi = (1u << (tm->B - 1)) + static_cast<uint32_t>(tm->N) - 1u;
    p.xplane = xs.ptr;
    p.nplane = xs.ptr + tm->Wp;
    p.q = 1;
    p.margin = 1;
    p.boost = boost ? 1 : 0;
    p.events = tm->events.ptr;
    tmg::MirrorParams mp{};
    mp.jobs = djobs.ptr;
    mp.njobs = 1;
    mp.rng = drng.ptr;
    mp.p_high = (s - 1.0) / s;
    mp.p_low = 1.0 / s;
    mirror_jumps(tm, mp);
    if (!tmg::train_mirror_launch(p, mp, tm->B, tm->NW, tm->stream))
      fail(TMG_ERUNTIME, "no mirror kernel instantiation for this shape");
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(rng_state, drng.ptr, 32, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    tm->entries_dirty = true;
  });
}

TMG_API int tmg_evaluate_clause(tmg_machine* tm, int32_t bank, int32_t j, const uint64_t* literals,
                                int32_t mode, int32_t* out) {
  if (is_group(tm)) {
    tmg_machine* part = group_owner(tm, j);
    if (!part) return guarded([&] { fail(TMG_ERANGE, "clause index outside this machine"); });
    return tmg_evaluate_clause(part, bank, j, literals, mode, out);
  }
  return guarded([&] {
    check_bank(M(tm), bank);
    if (j < tm->j_begin || j >= tm->j_end) fail(TMG_ERANGE, "clause index outside this machine");
    DeviceGuard dg(tm->device);
    const int W64 = (2 * tm->o + 63) / 64;
    DevBuf<uint64_t> dl;
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    DevBuf<int32_t> dout;
    dl.alloc(W64);
    xs.alloc(2 * tm->Wp);
    dout.alloc(1);
    CK(cudaMemcpyAsync(dl.ptr, literals, W64 * 8, cudaMemcpyHostToDevice, tm->stream));
    tmg::unpack_ref_literals_launch(dl.ptr, xs.ptr, xs.ptr + tm->Wp, 1, tm->o, tm->Wp, tm->stream);
    const int lc = bank * tm->n_loc + (j - tm->j_begin);
    tmg::eval_one_launch(tm->state.ptr, lc, tm->B, tm->Wp, xs.ptr, xs.ptr + tm->Wp, mode == TMG_EVAL_TRAIN ? 1 : 0,
                         dout.ptr, tm->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout.ptr, 4, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

// ------------------------------------------------------------- inference ---

TMG_API int tmg_refresh_tallies(tmg_machine* tm, tmg_pool* pool) {
  if (is_sharded(tm)) {  // sums over every shard; each shard rewrites its previous outputs
    if (!pool || !tm) return guarded([&] { fail(TMG_EINVAL, "null handle"); });
    std::vector<int32_t> sums(static_cast<size_t>(pool->q) * tm->m);
    return group_class_sums(tm, pool, nullptr, 0, TMG_EVAL_TRAIN, sums.data(), true);
  }
  return guarded([&] {
    check_compatible(M(tm), pool);
    if (tm->n_loc != tm->n)  // a shard's sums are partial: the pool's replicated tallies would be wrong
      fail(TMG_EINVAL, "refresh_tallies on a clause shard: use tmg_class_sums_device per shard and all-reduce");
    DeviceGuard dg(tm->device);
    bind_for(tm, pool->q);  // pool.cpp:113
    class_sums_device(tm, pool->xplane(), pool->q, true, pool->tallies.ptr, tm->prev.ptr, pool_lit_t(tm, pool));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_class_sums_device(tmg_machine* tm, const tmg_pool* pool, int32_t mode, int32_t* d_sums) {
  if (is_sharded(tm)) {
    if (!pool || !tm) return guarded([&] { fail(TMG_EINVAL, "null handle"); });
    std::vector<int32_t> sums(static_cast<size_t>(pool->q) * tm->m);
    const int rc = group_class_sums(tm, pool, nullptr, 0, mode, sums.data(), false);
    if (rc != TMG_OK) return rc;
    return guarded([&] {
      DeviceGuard dg(tm->device);
      CK(cudaMemcpy(d_sums, sums.data(), sums.size() * 4, cudaMemcpyHostToDevice));
    });
  }
  return guarded([&] {
    check_compatible(M(tm), pool);
    DeviceGuard dg(tm->device);
    class_sums_device(tm, pool->xplane(), pool->q, mode == TMG_EVAL_TRAIN, d_sums, nullptr, pool_lit_t(tm, pool));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_class_sums(tmg_machine* tm, const tmg_pool* pool, int32_t mode, int32_t* out) {
  if (is_sharded(tm)) return group_class_sums(tm, pool, nullptr, 0, mode, out, false);
  return guarded([&] {
    check_compatible(M(tm), pool);
    DeviceGuard dg(tm->device);
    ensure_sums(tm, pool->q);
    class_sums_device(tm, pool->xplane(), pool->q, mode == TMG_EVAL_TRAIN, tm->sums.ptr, nullptr,
                      pool_lit_t(tm, pool));
    CK(cudaMemcpyAsync(out, tm->sums.ptr, static_cast<size_t>(pool->q) * tm->m * 4, cudaMemcpyDeviceToHost,
                       tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

namespace {
void argmax_host(const int32_t* sums, int64_t q, int m, int32_t* pred) {  // classify, trainer.cpp:244-260
  for (int64_t i = 0; i < q; ++i) {
    const int32_t* row = sums + i * m;
    if (m == 1) {
      pred[i] = row[0] >= 0 ? 1 : 0;
      continue;
    }
    int best = 0;
    for (int c = 1; c < m; ++c)
      if (row[c] > row[best]) best = c;
    pred[i] = best;
  }
}
}  // namespace

TMG_API int tmg_predict(tmg_machine* tm, const tmg_pool* pool, int32_t* out) {
  if (is_sharded(tm)) {
    if (!pool || !tm) return guarded([&] { fail(TMG_EINVAL, "null handle"); });
    std::vector<int32_t> sums(static_cast<size_t>(pool->q) * tm->m);
    const int rc = group_class_sums(tm, pool, nullptr, 0, TMG_EVAL_PREDICT, sums.data(), false);
    if (rc == TMG_OK) argmax_host(sums.data(), pool->q, tm->m, out);
    return rc;
  }
  return guarded([&] {
    check_compatible(M(tm), pool);
    DeviceGuard dg(tm->device);
    if (tm->n_loc != tm->n) fail(TMG_EINVAL, "predict on a clause shard: reduce class sums across shards first");
    ensure_sums(tm, pool->q + (pool->q + tm->m - 1) / tm->m + 1);
    class_sums_device(tm, pool->xplane(), pool->q, false, tm->sums.ptr, nullptr, pool_lit_t(tm, pool));
    int32_t* pred = tm->sums.ptr + static_cast<size_t>(pool->q) * tm->m;
    tmg::argmax_launch(tm->sums.ptr, pred, pool->q, tm->m, tm->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, pred, static_cast<size_t>(pool->q) * 4, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

namespace tmgx {
void literals_to_planes(tmg_machine* tm, const uint64_t* lits, int64_t q, DevBuf<uint32_t>& xs) {
  const int W64 = (2 * tm->o + 63) / 64;
  DevBuf<uint64_t> dl;
  dl.alloc(static_cast<size_t>(q) * W64);
  xs.alloc(static_cast<size_t>(q) * 2 * tm->Wp);
  CK(cudaMemcpyAsync(dl.ptr, lits, dl.bytes(), cudaMemcpyHostToDevice, tm->stream));
  tmg::unpack_ref_literals_launch(dl.ptr, xs.ptr, xs.ptr + tm->Wp, q, tm->o, tm->Wp, tm->stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(tm->stream));
}
}  // namespace tmgx

TMG_API int tmg_class_sums_literals(tmg_machine* tm, const uint64_t* lits, int64_t q, int32_t mode, int32_t* out) {
  if (is_sharded(tm)) return group_class_sums(tm, nullptr, lits, q, mode, out, false);
  return guarded([&] {
    M(tm);
    if (q <= 0) return;
    DeviceGuard dg(tm->device);
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    literals_to_planes(tm, lits, q, xs);
    ensure_sums(tm, q);
    class_sums_device(tm, xs.ptr, q, mode == TMG_EVAL_TRAIN, tm->sums.ptr, nullptr);
    CK(cudaMemcpyAsync(out, tm->sums.ptr, static_cast<size_t>(q) * tm->m * 4, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

TMG_API int tmg_predict_literals(tmg_machine* tm, const uint64_t* lits, int64_t q, int32_t* out) {
  if (is_sharded(tm)) {
    if (q <= 0) return TMG_OK;
    std::vector<int32_t> sums(static_cast<size_t>(q) * tm->m);
    const int rc = group_class_sums(tm, nullptr, lits, q, TMG_EVAL_PREDICT, sums.data(), false);
    if (rc == TMG_OK) argmax_host(sums.data(), q, tm->m, out);
    return rc;
  }
  return guarded([&] {
    M(tm);
    if (q <= 0) return;
    if (tm->n_loc != tm->n) fail(TMG_EINVAL, "predict on a clause shard: reduce class sums across shards first");
    DeviceGuard dg(tm->device);
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    literals_to_planes(tm, lits, q, xs);
    ensure_sums(tm, q + (q + tm->m - 1) / tm->m + 1);
    class_sums_device(tm, xs.ptr, q, false, tm->sums.ptr, nullptr);
    int32_t* pred = tm->sums.ptr + static_cast<size_t>(q) * tm->m;
    tmg::argmax_launch(tm->sums.ptr, pred, q, tm->m, tm->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, pred, static_cast<size_t>(q) * 4, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
  });
}

// --------------------------------------------------------- regression head ---

TMG_API int tmg_machine_create_regress(const tmg_config* cfg, int32_t o, int32_t device, tmg_machine** out) {
  // RegressionHead ctor (regression.cpp:69-80): one all-positive bank.
  return guarded([&] { *out = create_machine(cfg, o, 1, device, 0, cfg ? cfg->clauses : 0, 1); });
}

namespace {
void regress_predict_planes(tmg_machine* tm, const uint32_t* xs, int64_t q, int32_t* out,
                            const uint32_t* lit_t = nullptr) {
  if (!tm->all_positive) fail(TMG_EINVAL, "not a regression machine");
  if (tm->n_loc != tm->n) fail(TMG_EINVAL, "predict on a clause shard: reduce clause counts across shards first");
  ensure_sums(tm, 2 * q);
  class_sums_device(tm, xs, q, false, tm->sums.ptr, nullptr, lit_t);
  tmg::clamp_launch(tm->sums.ptr, tm->sums.ptr + q, q, tm->cfg.margin, tm->stream);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, tm->sums.ptr + q, static_cast<size_t>(q) * 4, cudaMemcpyDeviceToHost, tm->stream));
  CK(cudaStreamSynchronize(tm->stream));
}
}  // namespace

TMG_API int tmg_regress_predict(tmg_machine* tm, const tmg_pool* pool, int32_t* out) {
  // predict_scaled over a pool (regression.cpp:86-93)
  return guarded([&] {
    need_single(tm, "predict_scaled");
    if (!M(tm) || !pool || tm->o != pool->o) fail(TMG_EINVAL, "head/pool feature count mismatch");
    DeviceGuard dg(tm->device);
    regress_predict_planes(tm, pool->xplane(), pool->q, out, pool_lit_t(tm, pool));
  });
}

TMG_API int tmg_regress_predict_literals(tmg_machine* tm, const uint64_t* lits, int64_t q, int32_t* out) {
  return guarded([&] {
    need_single(tm, "predict_scaled");
    M(tm);
    if (q <= 0) return;
    DeviceGuard dg(tm->device);
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    literals_to_planes(tm, lits, q, xs);
    regress_predict_planes(tm, xs.ptr, q, out);
  });
}

TMG_API int tmg_update_regress(tmg_machine* tm, const uint64_t* literals, int32_t scaled_target,
                               uint64_t* rng_state, uint64_t* events) {
  // update_regress (regression.cpp:101-123): one example through the
  // sequential regression kernel with the caller's stream.
  return guarded([&] {
    if (!M(tm)->all_positive) fail(TMG_EINVAL, "not a regression machine");
    if (tm->n_loc != tm->n) fail(TMG_EINVAL, "needs the full (unsharded) machine");
    DeviceGuard dg(tm->device);
    DevBuf<uint32_t> xs;  // literal rows [q][2][Wp]
    literals_to_planes(tm, literals, 1, xs);
    DevBuf<int32_t> lab, ord;
    DevBuf<uint64_t> drng;
    lab.alloc(1);
    ord.alloc(1);
    drng.alloc(4);
    const int32_t zero = 0;
    CK(cudaMemcpyAsync(lab.ptr, &scaled_target, 4, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemcpyAsync(ord.ptr, &zero, 4, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemcpyAsync(drng.ptr, rng_state, 32, cudaMemcpyHostToDevice, tm->stream));
    CK(cudaMemsetAsync(tm->events.ptr, 0, tm->events.bytes(), tm->stream));
    tmg_pool fake;
    fake.o = tm->o;
    fake.m = 1;
    fake.q = 1;
    tm->regress_mode = true;
    tmg::TrainParams p = make_params(tm, &fake);
    tm->regress_mode = false;
    p.xplane = xs.ptr;
    p.nplane = xs.ptr + tm->Wp;
    p.labels = lab.ptr;
    p.order = ord.ptr;
    tmg::SeqParams sp{};
    sp.rng = drng.ptr;
    sp.p_high = (tm->cfg.specificity - 1.0) / tm->cfg.specificity;
    sp.p_low = 1.0 / tm->cfg.specificity;
    sp.events = tm->events.ptr;
    if (seq_parallel_enabled(tm)) seq_jumps(tm, sp);
    if (!tmg::train_sequential_launch(p, sp, tm->B, tm->stream)) fail(TMG_ERUNTIME, "no sequential kernel for B");
    CK(cudaGetLastError());
    unsigned long long ev = 0;
    CK(cudaMemcpyAsync(&ev, tm->events.ptr, 8, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaMemcpyAsync(rng_state, drng.ptr, 32, cudaMemcpyDeviceToHost, tm->stream));
    CK(cudaStreamSynchronize(tm->stream));
    tm->entries_dirty = true;
    if (events) *events = ev;
  });
}

TMG_API void tmg_rng_state_init(uint64_t seed, uint64_t stream, uint64_t* state) {
  tmg_rng r;
  tmg_rng_seed(&r, seed, stream);
  std::memcpy(state, r.s, 32);
}

TMG_API uint64_t tmg_rng_state_next(uint64_t* state) {
  tmg_rng r;
  std::memcpy(r.s, state, 32);
  const uint64_t v = tmg_rng_next(&r);
  std::memcpy(state, r.s, 32);
  return v;
}

TMG_API int tmg_epoch_order(uint64_t seed, int32_t epoch, int32_t q, int32_t* order) {
  return guarded([&] {
    if (q < 1) fail(TMG_EINVAL, "q must be >= 1");
    tmg_rng r;
    tmg_rng_seed(&r, seed, tmg_mix_stream(TMG_STREAM_PERMUTATION, static_cast<uint64_t>(epoch), 0));
    tmg_shuffled_indices(q, &r, order);
  });
}
