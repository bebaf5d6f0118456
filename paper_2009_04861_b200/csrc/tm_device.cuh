// tm_device.cuh — device building blocks of the B200 Tsetlin engine.
//
// Data layout:
//   * literal rows: two bit planes per example, u32 words, row stride Wp
//       xplane[i][w] bit b  = literal k = 32w+b      (feature x_f,   k <  o)
//       nplane[i][w] bit b  = literal k = o+32w+b    (negation !x_f, k >= o)
//     i.e. the reference's 2o-bit row (core.cpp:34-46) split at k = o so that
//     feature f and its negation sit at the same (word, bit) position.
//   * automaton states: bit-sliced, B planes x 2 parts (x / !x) x Wp words per
//     clause. Plane value v = counter + (2^(B-1) - N - 1), so counter in [1,2N]
//     maps to v in [lo, hi] = [2^(B-1)-N, 2^(B-1)+N-1] and Include
//     (counter > N, core.hpp:42-44) is exactly the top plane.
//   * one warp owns one clause; lane l holds words l, l+32, ... (NW passes).
#pragma once

#include <cstdint>

#include "kernels.h"

namespace tmg {

constexpr unsigned kFull = 0xffffffffu;

// Rounds of the counter-based generator of the asynchronous trainer.
// Philox4x32 with 7 rounds is the smallest round count that passes TestU01
// BigCrush (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2,
// 3", Table 2); 10 is the library default safety margin. Build with
// -DTMG_PHILOX_ROUNDS=10 for the conservative variant. The synchronous
// mirror replays the reference's xoshiro256++ instead and is unaffected.
#ifndef TMG_PHILOX_ROUNDS
#define TMG_PHILOX_ROUNDS 7
#endif

// Phase-1 "less" accumulation as IMAD (FMA pipe) instead of LOP3 (ALU pipe).
#ifndef TMG_SAMPLER_IMAD
#define TMG_SAMPLER_IMAD 1
#endif

// ---------------------------------------------------------------- Philox ---
// Keyed per (seed, epoch); counters carry (clause, example, literal word,
// draw block).
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < TMG_PHILOX_ROUNDS; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// The same block with the key schedule read from `rk` (TrainParams::rkey,
// kernel-parameter space): the per-round XOR takes its key straight from the
// constant bank instead of holding 2 x rounds key registers live.
__device__ __forceinline__ U4 philox4x32(U4 c, const uint32_t (&rk)[2][kMaxPhiloxRounds]) {
  static_assert(TMG_PHILOX_ROUNDS <= kMaxPhiloxRounds, "round schedule too short");
#pragma unroll
  for (int r = 0; r < TMG_PHILOX_ROUNDS; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x;
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ rk[0][r], lo1, hi0 ^ c.w ^ rk[1][r], lo0};
  }
  return c;
}

// ------------------------------------------------------------ xoshiro256++ ---
// Device copy of the reference stream (rng.hpp:44-54) for the sync mirror.
struct Xoshiro {
  uint64_t s0, s1, s2, s3;
  __device__ __forceinline__ uint64_t next() {
    const uint64_t sum = s0 + s3;
    const uint64_t out = ((sum << 23) | (sum >> 41)) + s0;
    const uint64_t t = s1 << 17;
    s2 ^= s0;
    s3 ^= s1;
    s1 ^= s2;
    s0 ^= s3;
    s2 ^= t;
    s3 = (s3 << 45) | (s3 >> 19);
    return out;
  }
  // rng.hpp:63 — exact: (next >> 11) * 2^-53.
  __device__ __forceinline__ double uniform() {
    return static_cast<double>(next() >> 11) * 0x1.0p-53;
  }
};

// The comparison u < p of a reference draw u = m * 2^-53 (m = next() >> 11 <
// 2^53) as an integer test m < u53_below(p): p * 2^53 is exact in double, so
// m * 2^-53 < p  <=>  m < p * 2^53  <=>  m < ceil(p * 2^53). NaN: never true.
__device__ __forceinline__ uint64_t u53_below(double p) {
  if (!(p > 0.0)) return 0;
  if (p >= 1.0) return uint64_t(1) << 53;
  return static_cast<uint64_t>(ceil(p * 0x1.0p53));
}
__device__ __forceinline__ uint64_t next53(Xoshiro& r) { return r.next() >> 11; }

// ---- xoshiro256 jump-ahead on the GPU: the state update of rng.hpp next()
// is linear over GF(2), so k steps are one 256 x 256 bit matrix M (built on
// the host, engine.cu gf2_pow). It is stored as nibble tables: entry (pos, v)
// = the 8 words of M * (v << 4 pos), i.e. the XOR of the columns of M for the
// set bits of nibble value v at nibble position pos (64 x 16 entries, 32 KB).
// A warp applies it cooperatively: lane L looks up the two nibbles of state
// byte L and the 32 partial products are XOR-reduced (redux.sync) per word.
#ifndef TMG_GF2_REDUX
#define TMG_GF2_REDUX 1  // one redux.sync per word (0: shuffle reduce-scatter, measured slower)
#endif
__device__ __forceinline__ void gf2_apply(const uint32_t* tab, uint32_t (&s)[8], int lane) {
  const int ws = lane >> 2;
  uint32_t v = s[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) v = ws == k ? s[k] : v;
  const uint32_t byte = (v >> (8 * (lane & 3))) & 0xFFu;
  const uint4* e0 = reinterpret_cast<const uint4*>(tab + ((2 * lane) * 16 + (byte & 15u)) * 8);
  const uint4* e1 = reinterpret_cast<const uint4*>(tab + ((2 * lane + 1) * 16 + (byte >> 4)) * 8);
  const uint4 a0 = e0[0], a1 = e0[1], b0 = e1[0], b1 = e1[1];
  const uint32_t x[8] = {a0.x ^ b0.x, a0.y ^ b0.y, a0.z ^ b0.z, a0.w ^ b0.w,
                         a1.x ^ b1.x, a1.y ^ b1.y, a1.z ^ b1.z, a1.w ^ b1.w};
#if TMG_GF2_REDUX
#pragma unroll
  for (int w = 0; w < 8; ++w) s[w] = __reduce_xor_sync(kFull, x[w]);
#else
  // Reduce-scatter by halving (lane bits 4, 3, 2 pick the half kept), then
  // the last two lane bits, so lane L ends with word L >> 2; then gather.
  const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
  uint32_t y[4], z[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) y[k] = (h4 ? x[k + 4] : x[k]) ^ __shfl_xor_sync(kFull, h4 ? x[k] : x[k + 4], 16);
#pragma unroll
  for (int k = 0; k < 2; ++k) z[k] = (h3 ? y[k + 2] : y[k]) ^ __shfl_xor_sync(kFull, h3 ? y[k] : y[k + 2], 8);
  uint32_t v1 = (h2 ? z[1] : z[0]) ^ __shfl_xor_sync(kFull, h2 ? z[0] : z[1], 4);
  v1 ^= __shfl_xor_sync(kFull, v1, 2);
  v1 ^= __shfl_xor_sync(kFull, v1, 1);
#pragma unroll
  for (int w = 0; w < 8; ++w) s[w] = __shfl_sync(kFull, v1, 4 * w);
#endif
}

__device__ __forceinline__ void state_to_words(const Xoshiro& r, uint32_t (&s)[8]) {
  const uint64_t q[4] = {r.s0, r.s1, r.s2, r.s3};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    s[2 * k] = static_cast<uint32_t>(q[k]);
    s[2 * k + 1] = static_cast<uint32_t>(q[k] >> 32);
  }
}

__device__ __forceinline__ Xoshiro words_to_state(const uint32_t (&s)[8]) {
  Xoshiro r;
  r.s0 = s[0] | static_cast<uint64_t>(s[1]) << 32;
  r.s1 = s[2] | static_cast<uint64_t>(s[3]) << 32;
  r.s2 = s[4] | static_cast<uint64_t>(s[5]) << 32;
  r.s3 = s[6] | static_cast<uint64_t>(s[7]) << 32;
  return r;
}


// Draws k .. k + 2o - 1 of a xoshiro stream (the 2o Type I draws of the
// reference, feedback.cpp:45,63) as bit words in literal order: hbits bit k
// = (u_k < p_high), lbits bit k = (u_k < p_low). Warp-cooperative: lane L
// jumps to draw L * chunk (jc = M^chunk applied lane by lane) and draws its
// segment; the stream then continues after the 2o draws (jl = M^(2o)).
// hbits / lbits (at least ceil(2o/32) + 2 words) are zeroed here. rng is
// lane 0's; every lane leaves with the advanced state.
__device__ __forceinline__ void draw_type_i_bits(Xoshiro& rng, int L, int chunk, double p_high, double p_low,
                                                 const uint32_t* jc, const uint32_t* jl, uint32_t* hbits,
                                                 uint32_t* lbits, int refw, int lane) {
  for (int k = lane; k < refw; k += 32) hbits[k] = lbits[k] = 0;
  uint32_t sw[8], mine[8], start[8];
  state_to_words(rng, sw);
#pragma unroll
  for (int w = 0; w < 8; ++w) start[w] = mine[w] = sw[w] = __shfl_sync(kFull, sw[w], 0);
  for (int hop = 1; hop < 32; ++hop) {
    if (hop * chunk >= L) break;  // warp-uniform
    gf2_apply(jc, sw, lane);
    if (lane == hop) {
#pragma unroll
      for (int w = 0; w < 8; ++w) mine[w] = sw[w];
    }
  }
  __syncwarp();
  Xoshiro rl = words_to_state(mine);
  const int k0 = lane * chunk, k1 = min(L, k0 + chunk);
  const uint64_t th = u53_below(p_high), tl = u53_below(p_low);
  uint32_t hw = 0, lw = 0;
  int cw = k0 >> 5;
  for (int k = k0; k < k1; ++k) {
    if ((k >> 5) != cw) {
      if (hw) atomicOr(&hbits[cw], hw);
      if (lw) atomicOr(&lbits[cw], lw);
      hw = lw = 0;
      cw = k >> 5;
    }
    const uint64_t u = next53(rl);
    hw |= (u < th ? 1u : 0u) << (k & 31);
    lw |= (u < tl ? 1u : 0u) << (k & 31);
  }
  if (k1 > k0) {
    if (hw) atomicOr(&hbits[cw], hw);
    if (lw) atomicOr(&lbits[cw], lw);
  }
  gf2_apply(jl, start, lane);  // the state after the 2o draws
  rng = words_to_state(start);
  __syncwarp();
}

// %laneid (one S2R when rematerialised, no mask).
__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// a * b + c on the FMA pipe (IMAD), for ALU-pipe relief.
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// ---------------------------------------------------------- bit-sliced ops ---
// Per-lane view of one clause part (x or !x) word: B planes.
template <int B>
struct Planes {
  uint32_t p[B];
};

// Lanes (literals) whose value equals the constant `val`.
template <int B>
__device__ __forceinline__ uint32_t eq_const(const Planes<B>& s, uint32_t val) {
  uint32_t acc = kFull;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint32_t cb = ((val >> b) & 1u) ? kFull : 0u;
    acc &= ~(s.p[b] ^ cb);
  }
  return acc;
}

// +1 on lanes in `mask` (caller guarantees no lane is at hi).
template <int B>
__device__ __forceinline__ void add_one(Planes<B>& s, uint32_t mask) {
  uint32_t carry = mask;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint32_t t = s.p[b] & carry;
    s.p[b] ^= carry;
    carry = t;
  }
}

// -1 on lanes in `mask` (caller guarantees no lane is at lo).
template <int B>
__device__ __forceinline__ void sub_one(Planes<B>& s, uint32_t mask) {
  uint32_t borrow = mask;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const uint32_t t = ~s.p[b] & borrow;
    s.p[b] ^= borrow;
    borrow = t;
  }
}

// Saturating +-1 (apply_transition's clamp to [1, 2N], core.hpp:62-63).
// Branch-free: the masks are computed for every lane (cheaper than divergence).
template <int B>
__device__ __forceinline__ void step(Planes<B>& s, uint32_t inc, uint32_t dec, uint32_t lo,
                                     uint32_t hi) {
  inc &= ~eq_const<B>(s, hi);
  dec &= ~eq_const<B>(s, lo);
  add_one<B>(s, inc);
  sub_one<B>(s, dec);
}

// Saturating -1 only (Type I with clause output 0).
template <int B>
__device__ __forceinline__ void step_down(Planes<B>& s, uint32_t dec, uint32_t lo) {
  sub_one<B>(s, dec & ~eq_const<B>(s, lo));
}

// The same two steps when N = 2^(B-1), i.e. lo = 0 and hi = 2^B - 1: the
// borrow (carry) chain is formed first; what leaves the top plane is exactly
// the set of lanes already at lo (hi), which are then left untouched. One
// LOP3 per plane for the chain and one for the flip, no separate compare.
// One LOP3 with an explicit truth table (inputs a = 0xF0, b = 0xCC, c = 0xAA).
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

// EXPL: the chains as explicit LOP3s. In the register kernel ptxas rewrites
// the plain form into 3 LOP3 per plane plus moves and is still faster (MNIST
// 69.8 vs 70.3 ms); in the shared-memory kernel the explicit form wins (IMDb
// 231.4 vs 235.3 ms).
template <int B, bool EXPL = false>
__device__ __forceinline__ void sub_one_sat0(Planes<B>& s, uint32_t dec) {
  uint32_t chain[B];
  uint32_t t = dec;
  if constexpr (EXPL) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      chain[b] = t;
      t = lop3<0x30>(t, s.p[b], 0u);  // t & ~p
    }
#pragma unroll
    for (int b = 0; b < B; ++b) s.p[b] = lop3<0xB4>(s.p[b], chain[b], t);  // p ^ (chain & ~t)
  } else {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      chain[b] = t;
      t &= ~s.p[b];
    }
#pragma unroll
    for (int b = 0; b < B; ++b) s.p[b] ^= chain[b] & ~t;
  }
}

// Both at once (P2 layout): lanes in `move` take one step, down (-1) where
// `down` is set, up (+1) elsewhere. The chain continues through plane b while
// that bit equals the direction's ripple value (1 for +1, 0 for -1), i.e.
// t &= p[b] ^ down: one LOP3 per plane, one more for the flip. What leaves the
// top plane is the set of lanes already saturated in their direction, which
// are left untouched -- the same result as a saturating +1 pass then a
// saturating -1 pass on disjoint masks, at half the cost.
template <int B, bool EXPL = false>
__device__ __forceinline__ void step_sat(Planes<B>& s, uint32_t move, uint32_t down) {
  uint32_t chain[B];
  uint32_t t = move;
  if constexpr (EXPL) {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      chain[b] = t;
      t = lop3<0x60>(t, s.p[b], down);  // t & (p ^ down)
    }
#pragma unroll
    for (int b = 0; b < B; ++b) s.p[b] = lop3<0xB4>(s.p[b], chain[b], t);  // p ^ (chain & ~t)
  } else {
#pragma unroll
    for (int b = 0; b < B; ++b) {
      chain[b] = t;
      t &= s.p[b] ^ down;
    }
#pragma unroll
    for (int b = 0; b < B; ++b) s.p[b] ^= chain[b] & ~t;
  }
}


// Type I (feedback.cpp:32-70) on one word of automata given its Bernoulli mask:
//   out=1, lit=1 : +1 w.p. (s-1)/s  (always if boost and included)
//   out=1, lit=0 : Reward w.p. 1/s  (-1 if excluded; +1 if included, which
//                  only a caller-forced output can reach, feedback.cpp:55-57)
//   out=0        : -1 w.p. 1/s       (Penalty on Include, Reward on Exclude)
// P2: N = 2^(B-1) (lo = 0, hi = all ones), saturation fused into the chains.
// FUSED: clause output 1 as one up/down pass (step_sat) instead of a +1 pass
// then a -1 pass. Fewer instructions, but measured slower in the register
// kernel (MNIST 72.8 vs 71.4 ms, FMNIST 656 vs 650 ms) and faster in the
// shared-memory one (IMDb 235.3 vs 236.2 ms), so each kernel picks its own.
template <int B, bool P2, bool FUSED = true, bool EXPL = false>
__device__ __forceinline__ void type_i_planes(Planes<B>& w, uint32_t lit, int out, int boost, uint32_t bern,
                                              uint32_t valid, uint32_t lo, uint32_t hi) {
  if (out) {
    const uint32_t incl = w.p[B - 1];
    if (P2 && FUSED) {  // one up/down pass: false literals of excluded automata step down
      const uint32_t move = ((lit & (bern | (boost ? incl : 0u))) | (~lit & bern)) & valid;
      step_sat<B, EXPL>(w, move, ~(lit | incl));
    } else if (P2) {  // the same as two saturating passes on disjoint masks
      const uint32_t inc = ((lit & (bern | (boost ? incl : 0u))) | (~lit & bern & incl)) & valid;
      const uint32_t dec = ~lit & bern & ~incl & valid;
      step_sat<B, EXPL>(w, inc, 0u);
      sub_one_sat0<B, EXPL>(w, dec);
    } else {
      const uint32_t inc = ((lit & (bern | (boost ? incl : 0u))) | (~lit & bern & incl)) & valid;
      const uint32_t dec = ~lit & bern & ~incl & valid;
      step<B>(w, inc, dec, lo, hi);
    }
  } else if (P2) {
    sub_one_sat0<B, EXPL>(w, bern & valid);
  } else {
    step_down<B>(w, bern & valid, lo);
  }
}

// Alias-table sampler for the Type I draws of a clause with output 0, where
// every literal independently takes its step with the same p = P_low / 2^32
// (feedback.cpp:66-68). Each aligned group of 8 literals draws its whole
// 8-bit pattern from the product law Bernoulli(p)^8 with one 32-bit uniform
// u and Walker's alias method: column = u & 0xFF, and the column's own
// pattern wins iff (u >> 8) < its 24-bit threshold, else its alias
// (entry = threshold << 8 | alias; (u | 0xFF) < entry is that test).
// Pattern probabilities are within 2^-32 of the product law (masses rounded
// to 2^-32 units, engine.cu build_alias8), each literal's within 2^-25 of p. One Philox block = the 32 literals of a word slot;
// `tab` holds kAliasCopies interleaved copies of the 256 entries so the 32
// lanes' random lookups hit at most two shared-memory wavefronts.
#ifndef TMG_ALIAS_COPIES
#define TMG_ALIAS_COPIES 16
#endif
constexpr int kAliasCopies = TMG_ALIAS_COPIES;
// Shared-memory image of the table: thresholds (threshold << 8, low byte 0)
// as 256 x kAliasCopies u32, then the alias patterns as 256 x kAliasCopies
// bytes (20 KB). The threshold test is then a plain u < E (no masking), and
// the second lookup goes to the lightly used LSU pipe instead of the ALU.
constexpr int kAliasWords = 256 * kAliasCopies + 256 * kAliasCopies / 4;

// The packed image (entries threshold << 8 | alias as they are, C copies:
// 4 KB at C = 4), for kernels whose occupancy is bound by shared memory
// (train_smem.cu: fewer copies, one more resident clause per SM at IMDb shape).
#ifndef TMG_SMEM_ALIAS_COPIES
#define TMG_SMEM_ALIAS_COPIES 4
#endif
constexpr int kSmemAliasCopies = TMG_SMEM_ALIAS_COPIES;
constexpr int kAliasWordsPacked = 256 * kSmemAliasCopies;
template <int C = kSmemAliasCopies>
__device__ __forceinline__ void fill_alias_packed(uint32_t* tab, const uint32_t* entries, int tid, int n) {
  for (int k = tid; k < 256 * C; k += n) tab[k] = __ldg(entries + k / C);
}

// Fills the split image from the machine's 256 packed entries
// (threshold << 8 | alias), with the n threads of index tid.
__device__ __forceinline__ void fill_alias(uint32_t* tab, const uint32_t* entries, int tid, int n) {
  uint8_t* pat = reinterpret_cast<uint8_t*>(tab + 256 * kAliasCopies);
  for (int k = tid; k < 256 * kAliasCopies; k += n) {
    const uint32_t e = __ldg(entries + k / kAliasCopies);
    tab[k] = e & ~0xFFu;
    pat[k] = static_cast<uint8_t>(e & 0xFFu);
  }
}

// Shared-space byte addresses of a lane's copies of column 0 of the alias
// image (threshold and pattern); column c is 4 * kAliasCopies * c
// (kAliasCopies * c) further (one IMAD per lookup, on the FMA pipe).
struct AliasRef {
  uint32_t base, pbase;
};
__device__ __forceinline__ AliasRef alias_ref(const uint32_t* tab, uint32_t laneoff) {
  return AliasRef{static_cast<uint32_t>(__cvta_generic_to_shared(tab)) + 4u * laneoff,
                  static_cast<uint32_t>(__cvta_generic_to_shared(tab + 256 * kAliasCopies)) + laneoff};
}

// The 32-literal pattern of one word slot from one Philox block (4 draws).
template <bool SPLIT = true, int C = kAliasCopies>
__device__ __forceinline__ uint32_t alias_word(const U4 r, AliasRef ar, uint32_t need) {
  uint32_t b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t u = j == 0 ? r.x : (j == 1 ? r.y : (j == 2 ? r.z : r.w));
    const uint32_t col = u & 0xFFu;
    uint32_t e;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(mad_u32(col, 4u * C, ar.base)));
    if (SPLIT) {
      uint32_t a;
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(a) : "r"(mad_u32(col, C, ar.pbase)));
      b[j] = u < e ? u : a;  // (u >> 8) < threshold: the column's own pattern; low byte = the draw
    } else {
      b[j] = (u | 0xFFu) < e ? u : e;  // the same test on the packed entry
    }
  }
  const uint32_t lo = __byte_perm(b[0], b[1], 0x0040), hi = __byte_perm(b[2], b[3], 0x0040);
  return __byte_perm(lo, hi, 0x5410) & need;
}

template <int K, bool SPLIT = true, int C = kAliasCopies, typename Gen>
__device__ __forceinline__ void alias_words(const uint32_t (&need)[K], AliasRef ar, uint32_t (&bern)[K], Gen&& gen) {
#pragma unroll
  for (int k = 0; k < K; ++k) bern[k] = alias_word<SPLIT, C>(gen(k, 0), ar, need[k]);
}

// Warp-cooperative exact Bernoulli masks for one Type I event: every lane
// owns K words of literals; bit b of word k is wanted with probability
// P / 2^32 where P = P_high if bit b of sel[k] else P_low (SEL=false: always
// P_low). Every literal compares a fresh 32-bit uniform u with P, most
// significant bit first:
//   phase 1 — 8 bit-serial rounds on whole words (two Philox blocks per word,
//             the K chains interleaved for ILP). A literal is still undecided
//             afterwards only if its 8 bits of u equal P's top 8 bits
//             (probability 2^-8).
//   phase 2 — each still-undecided literal takes one private word from its
//             lane's Philox blocks and compares 24 bits of it with P's low 24
//             bits at once (branch-free, four literals per block).
// Together an exact Bernoulli(P / 2^32) per literal, at ~2.3 random words per
// 32 literals instead of one draw per literal.
// gen(slot, blk) returns Philox block `blk` of word slot `slot` (< K) or of
// the lane's phase-2 pool (slot == K).
template <int K, bool SEL, typename Gen>
__device__ __forceinline__ void bernoulli_words(const uint32_t (&need)[K], const uint32_t (&sel)[K],
                                                const BernThresholds& th, uint32_t (&less)[K],
                                                Gen&& gen) {
  uint32_t und[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    und[k] = need[k];
    less[k] = 0;
  }
#pragma unroll
  for (int blk = 0; blk < 2; ++blk) {
    U4 r[K];
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = gen(k, blk);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t ph = th.hi_mask[4 * blk + i];
      const uint32_t pl = th.lo_mask[4 * blk + i];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t rb = i == 0 ? r[k].x : (i == 1 ? r[k].y : (i == 2 ? r[k].z : r[k].w));
        const uint32_t pk = SEL ? ((sel[k] & ph) | (~sel[k] & pl)) : pl;
#if TMG_SAMPLER_IMAD
        // The literals decided "less" this round are disjoint from `less`, so
        // the OR is an add; as an IMAD with the opaque unit th.one it issues
        // on the FMA pipe and leaves the (binding) ALU pipe two LOP3 a round.
        less[k] = mad_u32(und[k] & ~rb & pk, th.one, less[k]);
#else
        less[k] |= und[k] & ~rb & pk;
#endif
        und[k] &= ~(rb ^ pk);
      }
    }
  }
  // Phase 2: every round resolves the lowest undecided literal of EVERY word
  // slot at once (one private random word per slot, ceil(K/4) Philox blocks
  // per round); rounds repeat while any lane of the warp has one left
  // (~1.3 rounds on average at MNIST shape).
  uint32_t left = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) left |= und[k];
  for (int round = 0; __any_sync(kFull, left != 0); ++round) {
    U4 r[(K + 3) / 4];
#pragma unroll
    for (int b = 0; b < (K + 3) / 4; ++b) r[b] = gen(K, 2 + round * ((K + 3) / 4) + b);
    left = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const U4& rb = r[k / 4];
      const uint32_t word = (k & 3) == 0 ? rb.x : ((k & 3) == 1 ? rb.y : ((k & 3) == 2 ? rb.z : rb.w));
      const uint32_t bit = und[k] & (0u - und[k]);  // lowest undecided literal (0: none)
      const uint32_t rest = (SEL && (sel[k] & bit)) ? th.hi_rest : th.lo_rest;
      less[k] |= ((word >> 8) < rest) ? bit : 0u;
      und[k] ^= bit;
      left |= und[k];
    }
  }
}

}  // namespace tmg
