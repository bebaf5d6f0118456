// clause.cuh — one clause of the asynchronous trainer as seen by one warp:
// its automaton planes in registers (NW words per lane), evaluation, Type II,
// the asynchronous Type I feedback with its Philox/alias draws, and the gate
// of a step. Used by the register-resident clause kernel (train.cu); the
// shared-memory clause kernel (train_smem.cu) shares the gate and draws.
#pragma once

#include "kernels.h"
#include "tm_device.cuh"

#ifndef TMG_ASYNC_P2
#define TMG_ASYNC_P2 1  // fused saturation when N = 2^(B-1)
#endif
#ifndef TMG_ASYNC_UNROLL_NW
#define TMG_ASYNC_UNROLL_NW 1  // widest rows (words per lane) that get the 2x unrolled step loop
#endif
#ifndef TMG_STEP_SAT_REG_NW
// Register kernels: clause-output-1 Type I as ONE up/down saturating pass
// (tm_device.cuh type_i_planes FUSED) for rows of at least this many words per
// lane, two passes below (MNIST 1-word rows: 67.6 vs 68.3 ms fused; FMNIST
// 3-word rows: 524 vs 559 ms fused).
#define TMG_STEP_SAT_REG_NW 2
#endif
#ifndef TMG_ROW_X_ONLY
#define TMG_ROW_X_ONLY 1  // async kernels read the x half of a literal row only (!x = ~x)
#endif
#ifndef TMG_ROW_X_MIN_NW
#define TMG_ROW_X_MIN_NW 2  // register kernel: from this row width (words per lane)
#endif
#ifndef TMG_ALIAS
#define TMG_ALIAS 1  // alias-table sampler for clause-output-0 Type I draws
#endif



namespace tmg {
namespace {

template <int NW, int B, bool P2 = false>  // P2: N = 2^(B-1) (lo = 0, hi = all ones)
struct Clause {
  Planes<B> s[2][NW];  // [part][pass]
  uint32_t valid[NW];  // literal bits that exist (f < o)

  __device__ __forceinline__ void load(const uint32_t* base, int Wp, int lane, int o) {
#pragma unroll
    for (int p = 0; p < NW; ++p) {
      const int wi = p * 32 + lane;
      const int first = wi * 32;
      valid[p] = first >= o ? 0u : (o - first >= 32 ? kFull : ((1u << (o - first)) - 1u));
#pragma unroll
      for (int part = 0; part < 2; ++part)
#pragma unroll
        for (int b = 0; b < B; ++b) s[part][p].p[b] = base[(b * 2 + part) * Wp + wi];
    }
  }

  __device__ __forceinline__ void store(uint32_t* base, int Wp, int lane) const {
#pragma unroll
    for (int p = 0; p < NW; ++p)
#pragma unroll
      for (int part = 0; part < 2; ++part)
#pragma unroll
        for (int b = 0; b < B; ++b) base[(b * 2 + part) * Wp + p * 32 + lane] = s[part][p].p[b];
  }

  bool nonempty = false;  // include count > 0, refreshed by every eval_train

  // Row word of slot p held by this lane (x plane; !x is the same word of
  // the second half).
  __device__ __forceinline__ int word_of(int p, int lane) const { return p * 32 + lane; }

  // Train-mode evaluation (core.hpp:208-219): empty clause -> 1.
  __device__ __forceinline__ int eval_train(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) {
    uint32_t viol = 0, any = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p) {
      const uint32_t ix = s[0][p].p[B - 1], in = s[1][p].p[B - 1];
      viol |= (ix & ~x[p]) | (in & ~n[p]);
      any |= ix | in;
    }
    const unsigned vb = __ballot_sync(kFull, viol != 0);
    nonempty = __any_sync(kFull, any != 0);
    return !nonempty ? 1 : (vb == 0 ? 1 : 0);
  }

  // Same, reusing the include-set emptiness of the last eval_train (valid
  // while the automata have not moved since).
  __device__ __forceinline__ int eval_cached(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) const {
    uint32_t viol = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p) viol |= (s[0][p].p[B - 1] & ~x[p]) | (s[1][p].p[B - 1] & ~n[p]);
    const unsigned vb = __ballot_sync(kFull, viol != 0);
    return !nonempty ? 1 : (vb == 0 ? 1 : 0);
  }

  __device__ __forceinline__ void refresh_nonempty() {
    uint32_t any = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p) any |= s[0][p].p[B - 1] | s[1][p].p[B - 1];
    nonempty = __any_sync(kFull, any != 0);
  }

  __device__ __forceinline__ int include_count() const {
    int cnt = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p) cnt += __popc(s[0][p].p[B - 1]) + __popc(s[1][p].p[B - 1]);
#pragma unroll
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
    return cnt;
  }

  // Type II (feedback.cpp:72-83): with output 1, every excluded automaton of
  // a false literal takes a Penalty (+1). Excluded states sit below the top
  // plane, so no saturation is possible. Returns whether anything moved.
  __device__ __forceinline__ bool type_ii(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) {
    uint32_t moved = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p) {
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const uint32_t lit = part ? n[p] : x[p];
        const uint32_t inc = ~lit & ~s[part][p].p[B - 1] & valid[p];
        add_one<B>(s[part][p], inc);
        moved |= inc;
      }
    }
    return __any_sync(kFull, moved != 0);
  }

  // Type I on word slot p of part `part` (tm_device.cuh type_i_planes).
  __device__ __forceinline__ void type_i_word(int part, int p, uint32_t lit, int out, int boost,
                                              uint32_t bern, uint32_t lo, uint32_t hi) {
    type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(s[part][p], lit, out, boost, bern, valid[p], lo, hi);
  }
};

// The same clause with the last word slot PACKED (rows whose last slot has
// R <= 16 valid words, e.g. FMNIST's 74 words = 2 full slots + 10): lanes
// 0..R-1 hold that slot's x-part words, lanes R..2R-1 its !x-part words, the
// rest a padding word of the x part (never valid). Type I then draws 2NW - 1
// word slots per lane instead of 2NW, with the same Philox counters (keyed by
// word and part, not by lane), so the automata move exactly as in Clause.
// Rows are read x-only: n[p] = ~x[p] (TMG_ROW_X_ONLY).
template <int NW, int B, bool P2 = false>
struct ClausePk {
  static_assert(NW >= 2, "packing needs a full slot before the last");
  Planes<B> s[2][NW - 1];  // full slots [part][pass]
  Planes<B> pk;            // the packed slot
  uint32_t valid[NW - 1];
  uint32_t vpk;
  int pk_part, pk_w;  // part and row word of this lane's packed-slot word
  bool nonempty = false;

  __device__ __forceinline__ int word_of(int p, int lane) const { return p < NW - 1 ? p * 32 + lane : pk_w; }
  __device__ __forceinline__ static uint32_t valid_bits_of(int wi, int o) {
    const int first = wi * 32;
    return first >= o ? 0u : (o - first >= 32 ? kFull : ((1u << (o - first)) - 1u));
  }
  // The literal value word of the packed slot: x for part 0, !x for part 1.
  __device__ __forceinline__ uint32_t pk_lit(const uint32_t (&x)[NW]) const {
    return pk_part ? ~x[NW - 1] : x[NW - 1];
  }

  __device__ __forceinline__ void load(const uint32_t* base, int Wp, int lane, int o) {
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) {
      const int wi = p * 32 + lane;
      valid[p] = valid_bits_of(wi, o);
#pragma unroll
      for (int part = 0; part < 2; ++part)
#pragma unroll
        for (int b = 0; b < B; ++b) s[part][p].p[b] = base[(b * 2 + part) * Wp + wi];
    }
    const int R = (o + 31) / 32 - 32 * (NW - 1);  // valid words of the last slot (<= 16)
    const int last = 32 * (NW - 1);
    pk_part = lane >= R && lane < 2 * R ? 1 : 0;
    pk_w = last + (lane < R ? lane : (lane < 2 * R ? lane - R : lane - R));  // idle: padding words of part 0
    vpk = lane < 2 * R ? valid_bits_of(pk_w, o) : 0u;
#pragma unroll
    for (int b = 0; b < B; ++b) pk.p[b] = base[(b * 2 + pk_part) * Wp + pk_w];
  }

  __device__ __forceinline__ void store(uint32_t* base, int Wp, int lane) const {
#pragma unroll
    for (int p = 0; p < NW - 1; ++p)
#pragma unroll
      for (int part = 0; part < 2; ++part)
#pragma unroll
        for (int b = 0; b < B; ++b) base[(b * 2 + part) * Wp + p * 32 + lane] = s[part][p].p[b];
#pragma unroll
    for (int b = 0; b < B; ++b) base[(b * 2 + pk_part) * Wp + pk_w] = pk.p[b];
  }

  __device__ __forceinline__ uint32_t violations(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) const {
    uint32_t viol = pk.p[B - 1] & ~pk_lit(x);
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) viol |= (s[0][p].p[B - 1] & ~x[p]) | (s[1][p].p[B - 1] & ~n[p]);
    return viol;
  }
  __device__ __forceinline__ int eval_train(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) {
    const uint32_t viol = violations(x, n);
    uint32_t any = pk.p[B - 1];
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) any |= s[0][p].p[B - 1] | s[1][p].p[B - 1];
    const unsigned vb = __ballot_sync(kFull, viol != 0);
    nonempty = __any_sync(kFull, any != 0);
    return !nonempty ? 1 : (vb == 0 ? 1 : 0);
  }
  __device__ __forceinline__ int eval_cached(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) const {
    const unsigned vb = __ballot_sync(kFull, violations(x, n) != 0);
    return !nonempty ? 1 : (vb == 0 ? 1 : 0);
  }
  __device__ __forceinline__ void refresh_nonempty() {
    uint32_t any = pk.p[B - 1];
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) any |= s[0][p].p[B - 1] | s[1][p].p[B - 1];
    nonempty = __any_sync(kFull, any != 0);
  }
  __device__ __forceinline__ int include_count() const {
    int cnt = __popc(pk.p[B - 1]);
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) cnt += __popc(s[0][p].p[B - 1]) + __popc(s[1][p].p[B - 1]);
#pragma unroll
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
    return cnt;
  }
  // Type II (feedback.cpp:72-83), as Clause::type_ii.
  __device__ __forceinline__ bool type_ii(const uint32_t (&x)[NW], const uint32_t (&n)[NW]) {
    uint32_t moved = 0;
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) {
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const uint32_t lit = part ? n[p] : x[p];
        const uint32_t inc = ~lit & ~s[part][p].p[B - 1] & valid[p];
        add_one<B>(s[part][p], inc);
        moved |= inc;
      }
    }
    const uint32_t inc = ~pk_lit(x) & ~pk.p[B - 1] & vpk;
    add_one<B>(pk, inc);
    moved |= inc;
    return __any_sync(kFull, moved != 0);
  }
};

__device__ __forceinline__ uint64_t splitmix_dev(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Fire-and-forget reductions (RED, no return value to wait for).
__device__ __forceinline__ void red_add_gpu(int32_t* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_xor_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.xor.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_sys(int32_t* p, int v) {
  asm volatile("red.relaxed.sys.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One tally change (pool.cpp:93-106 add_to_tally): the local replica, the
// window delta buffer when windows are in use, and — with peer replicas —
// every other rank's replica over NVLink. With peers, the local add is also
// system-scoped: remote GPUs reduce into the same words.
__device__ __forceinline__ void publish_tally(const TrainParams& P, size_t ti, int delta) {
  if (P.npeers == 0) {
    red_add_gpu(P.tallies + ti, delta);
  } else {
    red_add_sys(P.tallies + ti, delta);
    for (int k = 0; k < P.npeers; ++k) red_add_sys(P.peer_tallies[k] + ti, delta);
  }
  if (P.tally_delta) red_add_gpu(P.tally_delta + ti, delta);
}

// Publishes the post-feedback output (pool.cpp:93-106); one lane.
__device__ __forceinline__ void record(const TrainParams& P, uint32_t* prev_row, int64_t i, int c,
                                       bool positive, uint32_t pword, int after) {
  const uint32_t bit = 1u << (i & 31);
  const int before = (pword & bit) ? 1 : 0;
  if (before == after) return;
  prev_row[i >> 5] = pword ^ bit;
  int delta = after ? 1 : -1;
  if (!positive) delta = -delta;
  publish_tally(P, static_cast<size_t>(i) * P.m + c, delta);
}

// --------------------------------------------------------------- async ---

// Type I (feedback.cpp:32-70) on every word of the clause with the exact
// warp-cooperative Bernoulli sampler; counters keyed (clause g, example i,
// literal word, block) so the draws do not depend on scheduling.
template <int NW, int B, bool P2>
__device__ __forceinline__ void type_i_async(Clause<NW, B, P2>& cl, const uint32_t (&x)[NW], const uint32_t (&n)[NW],
                                             int before, const TrainParams& P, uint32_t g, uint32_t i,
                                             int lane, AliasRef atab) {
  constexpr int K = 2 * NW;
  uint32_t need[K], sel[K], bern[K];
#pragma unroll
  for (int p = 0; p < NW; ++p) {
    need[2 * p] = need[2 * p + 1] = cl.valid[p];
    sel[2 * p] = x[p];
    sel[2 * p + 1] = n[p];
  }
  auto gen = [&](int slot, int blk) {
    const uint32_t wid = slot < K ? static_cast<uint32_t>(((slot >> 1) * 32 + lane) * 2 + (slot & 1))
                                  : (0xFFFF0000u | static_cast<uint32_t>(lane));
    return philox4x32(U4{g, i, wid, static_cast<uint32_t>(blk)}, P.rkey);
  };
#ifdef TMG_STATS
  if (P.dbg) {
    // Draws whose outcome cannot move the automaton (a step into the
    // saturated end it already sits at): histogram of the warp maximum per
    // lane and the warp total, per clause output (tools/draw_stats.py).
    int cnt = 0;
#pragma unroll
    for (int p = 0; p < NW; ++p)
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const Planes<B>& w = cl.s[part][p];
        const uint32_t lit = part ? n[p] : x[p];
        const uint32_t at_lo = eq_const<B>(w, P.lo), at_hi = eq_const<B>(w, P.hi), incl = w.p[B - 1];
        const uint32_t rel = before ? ((lit & ~at_hi) | (~lit & ~incl & ~at_lo)) : ~at_lo;
        cnt += __popc(rel & cl.valid[p]);
      }
    const int mx = __reduce_max_sync(kFull, cnt), sum = __reduce_add_sync(kFull, cnt);
    if (lane == 0) {
      unsigned long long* d = P.dbg + (before ? 128 : 0);
      atomicAdd(d + min(mx, 63), 1ULL);
      atomicAdd(d + 64, 1ULL);
      atomicAdd(d + 65, static_cast<unsigned long long>(sum));
      atomicAdd(d + 66, static_cast<unsigned long long>(mx));
    }
  }
#endif
#if TMG_ALIAS
  if (before && !P.alias_sel) {
    bernoulli_words<K, true>(need, sel, P.bern, bern, gen);
  } else {
    alias_words<K>(need, atab, bern, gen);
    // Clause output 1: a true literal fires w.p. p_high = 1 - p_low, a false
    // one w.p. p_low, so one Bernoulli(p_low) bit serves either, negated on
    // the true literals (independence across literals is untouched).
    if (before) {
#pragma unroll
      for (int k = 0; k < K; ++k) bern[k] = (bern[k] ^ sel[k]) & need[k];
    }
  }
#else
  if (before) bernoulli_words<K, true>(need, sel, P.bern, bern, gen);
  else bernoulli_words<K, false>(need, sel, P.bern, bern, gen);
#endif
  // The clause output is warp-uniform: branch once on it (constant `out` in
  // each arm) rather than leave the compiler to predicate both updates.
  if (before) {
#pragma unroll
    for (int p = 0; p < NW; ++p) {
      cl.type_i_word(0, p, x[p], 1, P.boost, bern[2 * p], P.lo, P.hi);
      cl.type_i_word(1, p, n[p], 1, P.boost, bern[2 * p + 1], P.lo, P.hi);
    }
  } else {
#pragma unroll
    for (int p = 0; p < NW; ++p) {
      cl.type_i_word(0, p, x[p], 0, P.boost, bern[2 * p], P.lo, P.hi);
      cl.type_i_word(1, p, n[p], 0, P.boost, bern[2 * p + 1], P.lo, P.hi);
    }
  }
}

// Type I on a packed clause: the full slots as in type_i_async, the packed
// slot as one more word slot with its own (word, part) counter. Clause-output-1
// draws take the alias table only (the launcher packs only when alias_sel).
template <int NW, int B, bool P2>
__device__ __forceinline__ void type_i_async(ClausePk<NW, B, P2>& cl, const uint32_t (&x)[NW],
                                             const uint32_t (&n)[NW], int before, const TrainParams& P, uint32_t g,
                                             uint32_t i, int lane, AliasRef atab) {
  constexpr int K = 2 * NW - 1;
  uint32_t need[K], sel[K], bern[K];
#pragma unroll
  for (int p = 0; p < NW - 1; ++p) {
    need[2 * p] = need[2 * p + 1] = cl.valid[p];
    sel[2 * p] = x[p];
    sel[2 * p + 1] = n[p];
  }
  need[K - 1] = cl.vpk;
  sel[K - 1] = cl.pk_lit(x);
  const uint32_t wid_pk = static_cast<uint32_t>(cl.pk_w * 2 + cl.pk_part);
  auto gen = [&](int slot, int blk) {
    const uint32_t wid = slot < K - 1 ? static_cast<uint32_t>(((slot >> 1) * 32 + lane) * 2 + (slot & 1)) : wid_pk;
    return philox4x32(U4{g, i, wid, static_cast<uint32_t>(blk)}, P.rkey);
  };
  alias_words<K>(need, atab, bern, gen);
  if (before) {
#pragma unroll
    for (int k = 0; k < K; ++k) bern[k] = (bern[k] ^ sel[k]) & need[k];
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) {
      type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(cl.s[0][p], x[p], 1, P.boost, bern[2 * p], cl.valid[p], P.lo, P.hi);
      type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(cl.s[1][p], n[p], 1, P.boost, bern[2 * p + 1], cl.valid[p], P.lo,
                                                  P.hi);
    }
    type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(cl.pk, sel[K - 1], 1, P.boost, bern[K - 1], cl.vpk, P.lo, P.hi);
  } else {
#pragma unroll
    for (int p = 0; p < NW - 1; ++p) {
      type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(cl.s[0][p], x[p], 0, P.boost, bern[2 * p], cl.valid[p], P.lo, P.hi);
      type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(cl.s[1][p], n[p], 0, P.boost, bern[2 * p + 1], cl.valid[p], P.lo,
                                                  P.hi);
    }
    type_i_planes<B, P2, (NW >= TMG_STEP_SAT_REG_NW)>(cl.pk, sel[K - 1], 0, P.boost, bern[K - 1], cl.vpk, P.lo, P.hi);
  }
}

// Gate of step t of clause g's pass (update_clause's skip test,
// trainer.cpp:112-122 / regression.cpp:46-67, 204-206): the example i at
// position offset + t of the epoch order, whether the step would take Type I
// (target = 1) or Type II feedback, and whether it is gated in, by the exact
// integer form r * 2T < e * 2^32 of u < e / 2T (feedback.cpp:24-28) with the
// Philox word r of counter (g, i, ~0, 0). The class tally is read relaxed
// through L2 (deliberately stale, the reference's atomic load).
// The example at position offset + t of the epoch order.
__device__ __forceinline__ int64_t order_at(const TrainParams& P, int64_t offset, int64_t t) {
  int64_t pos = offset + t;
  if (pos >= P.q) pos -= P.q;
  return P.order ? __ldg(P.order + pos) : pos;
}

// The gate decision from the step's example, label and (stale) tally.
__device__ __forceinline__ bool gate_decide(const TrainParams& P, int c, bool positive, uint32_t g, int64_t i,
                                            int label, int v, int& target) {
  const int T = P.margin;
  int64_t e;
  if (P.regress) {
    v = v < 0 ? 0 : (v > T ? T : v);
    e = label > v ? static_cast<int64_t>(label) - v : static_cast<int64_t>(v) - label;
    target = v < label ? 1 : 0;
  } else {
    const int y = label == c ? 1 : 0;
    v = v < -T ? -T : (v > T ? T : v);
    e = y ? static_cast<int64_t>(T) - v : static_cast<int64_t>(T) + v;
    target = (y == 1) == positive ? 1 : 0;
  }
  const U4 r = philox4x32(U4{g, static_cast<uint32_t>(i), 0xFFFFFFFFu, 0u}, P.rkey);
  return static_cast<uint64_t>(r.x) * (2 * static_cast<uint64_t>(T)) < (static_cast<uint64_t>(e) << 32);
}

__device__ __forceinline__ bool gate_step(const TrainParams& P, int c, bool positive, uint32_t g, int64_t offset,
                                          int64_t t, int64_t& i, int& target) {
  i = order_at(P, offset, t);
  return gate_decide(P, c, positive, g, i, __ldg(P.labels + i), __ldcg(P.tallies + i * P.m + c), target);
}

// The clause a warp trains (TrainParams::interleave): class-major (0), or
// classes interleaved per warp (1) or per group of G warps (2, the CTA's
// warps stay one class's consecutive clauses), so that each resident wave of
// the grid holds a slice of every class.
__device__ __forceinline__ int clause_of_warp(const TrainParams& P, int w, int G) {
  if (P.interleave == 0) return w;
  if (P.interleave == 2 && P.n_loc % G == 0) {
    const int b = w / G;
    return (b % P.m) * P.n_loc + (b / P.m) * G + w % G;
  }
  return (w % P.m) * P.n_loc + w / P.m;
}

// Per-clause starting position in the epoch order (trainer.cpp:41-44, 222-223).
__device__ __forceinline__ int64_t clause_offset_dev(uint32_t g, int64_t q) {
  return static_cast<int64_t>(splitmix_dev(static_cast<uint64_t>(g) + 1) % static_cast<uint64_t>(q));
}

// Copies the machine's alias table (P.alias8, 256 entries) into kAliasCopies
// interleaved shared-memory copies; every thread of the CTA takes part.
// This lane's view of the alias image. TMG_ALIAS_HOIST: computed once in the
// kernel prologue and kept in two registers (an opaque copy stops the
// compiler from re-deriving it from %laneid at every Type I event).
#ifndef TMG_ALIAS_HOIST
#define TMG_ALIAS_HOIST 1
#endif
template <int C = kAliasCopies>
__device__ __forceinline__ AliasRef lane_alias(const uint32_t* tab, int lane) {
  AliasRef r = alias_ref(tab, static_cast<uint32_t>(lane) & (C - 1));
#if TMG_ALIAS_HOIST
  asm volatile("mov.u32 %0, %0;" : "+r"(r.base));
  asm volatile("mov.u32 %0, %0;" : "+r"(r.pbase));
#endif
  return r;
}

__device__ __forceinline__ void load_alias(const TrainParams& P, uint32_t* tab) {
#if TMG_ALIAS
  fill_alias(tab, P.alias8, threadIdx.x, blockDim.x);
  __syncthreads();
#endif
}

}  // namespace
}  // namespace tmg
