// eval.cu — clause evaluation / class sums (inference and exact tally
// refresh), literal packing and automaton-state layout conversion.
//
// Class sums replace vote_sum / export_vote_sums / predict_all
// (proj/src/pool.cpp:82-91, proj/src/trainer.cpp:244-279); the train-mode
// variant with previous-output bitmaps replaces refresh_tallies
// (proj/src/pool.cpp:108-124).
//
// Example-sliced evaluation. A clause is a conjunction of its included
// literals, so for 32 examples at once its output word is the AND of the
// included literals' 32-example bit columns. The examples are therefore
// transposed once per call into feature-major bit columns (lit_t: row f =
// bit e of word g is x_f of example 32g+e, plus an all-ones and an all-zeros
// row), and each clause is compacted to the feature indices of its included
// positive literals and of its included negated literals. A warp takes one
// clause at a time over 1024 examples: output = AND(positive columns) &
// ~OR(negated columns), per included literal ONE address IMAD and ONE
// coalesced 128-byte load (half a LOP3) for 1024 (clause, example) pairs,
// with a warp-wide exit once every example is falsified. Clause outputs are summed per
// example in bit-sliced signed counters (one carry/borrow chain per clause
// word), reduced across the CTA's warps with bit-sliced adders in shared
// memory and turned into integers once per CTA.
#include <algorithm>

#include "kernels.h"
#include "tm_device.cuh"

namespace tmg {

namespace {

constexpr int kEvalWarps = 8;   // warps per eval CTA (same example block, disjoint clause ranges)
// Resident eval CTAs per SM the register budget is cut for (48 registers at 5).
// Measured (tools/build_variants.sh, r2 eval sweep): 4 -> MNIST +6%, FMNIST -5%;
// 6 -> MNIST +5%, FMNIST -4%. A software-pipelined short-list path (descriptor
// two clauses ahead, first 8 entries one ahead) spilled at 5 and at 4 ran
// MNIST 0.094 ms vs 0.078 ms, FMNIST +8%, IMDb +14%: removed.
#ifndef TMG_EVAL_MINB
#define TMG_EVAL_MINB 5
#endif
constexpr int kSumPlanes = 12;  // bit-sliced two's-complement counters: |sum| <= 2040 per CTA

// One warp per clause: count the included literals (top plane) -> inc_count,
// npos = its positive-literal list length padded to 4, lens = npos + its
// negated-literal list length padded to 4.
__global__ void count_literals_kernel(const uint32_t* __restrict__ state, int clauses, int B, int Wp, int Wx,
                                      int32_t* __restrict__ inc_count, int32_t* __restrict__ lens,
                                      int32_t* __restrict__ npos) {
  const int lane = threadIdx.x & 31;
  const int lc = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (lc >= clauses) return;
  const uint32_t* top = state + (static_cast<size_t>(lc) * B + (B - 1)) * 2 * Wp;
  int cp = 0, cn = 0;
  for (int w = lane; w < Wx; w += 32) {
    cp += __popc(top[w]);
    cn += __popc(top[Wp + w]);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    cp += __shfl_xor_sync(kFull, cp, off);
    cn += __shfl_xor_sync(kFull, cn, off);
  }
  if (lane == 0) {
    inc_count[lc] = cp + cn;
    npos[lc] = (cp + 3) & ~3;
    lens[lc] = ((cp + 3) & ~3) + ((cn + 3) & ~3);
  }
}

// Exclusive prefix sum of lens -> offs (one CTA; clause counts are small).
// offs[clauses] = total.
__global__ void __launch_bounds__(1024) scan_lengths_kernel(const int32_t* __restrict__ lens, int clauses,
                                                            int64_t* __restrict__ offs) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int per = (clauses + 1023) / 1024;
  const int a = min(clauses, t * per), b = min(clauses, a + per);
  int64_t s = 0;
  for (int k = a; k < b; ++k) s += lens[k];
  part[t] = s;
  __syncthreads();
  for (int d = 1; d < 1024; d <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t v = t >= d ? part[t - d] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - s;
  for (int k = a; k < b; ++k) {
    offs[k] = run;
    run += lens[k];
  }
  if (t == 1023) offs[clauses] = part[1023];
}

// One warp per clause: its included positive literals' feature indices, padded
// to 4 with o (the all-ones row of lit_t), then its included negated
// literals' feature indices, padded to 4 with o + 1 (the all-zeros row).
__global__ void fill_literals_kernel(const uint32_t* __restrict__ state, int clauses, int B, int Wp, int Wx,
                                     int o, const int64_t* __restrict__ offs, const int32_t* __restrict__ npos,
                                     uint32_t* __restrict__ lists, int4* __restrict__ meta) {
  const int lane = threadIdx.x & 31;
  const int lc = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (lc >= clauses) return;
  const uint32_t* top = state + (static_cast<size_t>(lc) * B + (B - 1)) * 2 * Wp;
  uint32_t* out = lists + offs[lc];
  const int split = npos[lc];
  const int len = static_cast<int>(offs[lc + 1] - offs[lc]);
  if (lane == 0) meta[lc] = make_int4(static_cast<int>(offs[lc] >> 2), len, split, 0);
  for (int part = 0; part < 2; ++part) {
    uint32_t* dst = out + (part ? split : 0);
    const int end = part ? len - split : split;
    int base = 0;
    for (int w0 = 0; w0 < Wx; w0 += 32) {
      const int w = w0 + lane;
      uint32_t bits = w < Wx ? top[part * Wp + w] : 0u;
      const int cnt = __popc(bits);
      int incl = cnt;  // inclusive warp scan of the counts
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += v;
      }
      int pos = base + incl - cnt;
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        dst[pos++] = static_cast<uint32_t>(w * 32 + b);
      }
      base += __shfl_sync(kFull, incl, 31);
    }
    for (int k = base + lane; k < end; k += 32) dst[k] = static_cast<uint32_t>(o + part);
  }
}

// Literal rows [q][2][Wp] (x-plane words first) -> feature-major bit columns
// lit_t[f][Gs]: bit e of word g = x_f of example 32g + e (0 beyond q). One
// CTA: one row word w (32 features) x 32 column words (1024 examples); each
// warp transposes 32 x 32 bit blocks with ballots, rows leave coalesced.
__global__ void __launch_bounds__(256) transpose_literals_kernel(const uint32_t* __restrict__ xplane,
                                                                 int64_t row_stride, int64_t q, int o,
                                                                 int64_t Gs, uint32_t* __restrict__ lit_t) {
  __shared__ uint32_t tile[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = blockIdx.y;
  const int64_t g0 = static_cast<int64_t>(blockIdx.x) * 32;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int gl = warp * 4 + r;
    const int64_t i = (g0 + gl) * 32 + lane;
    const uint32_t v = i < q ? __ldg(xplane + i * row_stride + w) : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const uint32_t col = __ballot_sync(kFull, (v >> b) & 1u);
      if (lane == b) mine = col;
    }
    tile[lane][gl] = mine;  // feature 32w + lane, column word g0 + gl
  }
  __syncthreads();
  for (int fl = warp; fl < 32; fl += kEvalWarps) {
    const int f = w * 32 + fl;
    if (f < o) lit_t[static_cast<int64_t>(f) * Gs + g0 + lane] = tile[fl][lane];
  }
}

// counter += x (ADD) or -= x, bit-sliced two's complement, per bit lane.
template <bool ADD>
__device__ __forceinline__ void count_word(uint32_t (&P)[kSumPlanes], uint32_t x) {
#pragma unroll
  for (int b = 0; b < kSumPlanes; ++b) {
    if (x == 0u) break;
    const uint32_t p = P[b];
    P[b] = p ^ x;
    x = ADD ? (p & x) : (~p & x);
  }
}

// Column word of feature f for this lane: col + f * row_bytes, one
// IMAD.WIDE.U32 with the 64-bit base as addend.
__device__ __forceinline__ uint32_t column(const char* __restrict__ col, uint32_t f, uint32_t row_bytes) {
  return __ldg(reinterpret_cast<const uint32_t*>(col + static_cast<uint64_t>(f) * row_bytes));
}

// AND (positive list) or OR (negated list) of the listed feature columns:
// per literal one IMAD.WIDE (address) + one coalesced load, half a LOP3;
// 16 loads in flight per warp between early-exit votes.
template <bool POS>
__device__ __forceinline__ uint32_t fold_columns(const uint32_t* __restrict__ lst, int len,
                                                 const char* __restrict__ col, uint32_t row_bytes, uint32_t acc,
                                                 uint32_t other) {
  const uint4* p = reinterpret_cast<const uint4*>(lst);
  const uint4* const end = p + (len >> 2);  // lengths are multiples of 4
  for (; p + 4 <= end; p += 4) {
    const uint4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
    const uint32_t v0 = column(col, a.x, row_bytes), v1 = column(col, a.y, row_bytes);
    const uint32_t v2 = column(col, a.z, row_bytes), v3 = column(col, a.w, row_bytes);
    const uint32_t v4 = column(col, b.x, row_bytes), v5 = column(col, b.y, row_bytes);
    const uint32_t v6 = column(col, b.z, row_bytes), v7 = column(col, b.w, row_bytes);
    const uint32_t v8 = column(col, c.x, row_bytes), v9 = column(col, c.y, row_bytes);
    const uint32_t va = column(col, c.z, row_bytes), vb = column(col, c.w, row_bytes);
    const uint32_t vc = column(col, d.x, row_bytes), vd = column(col, d.y, row_bytes);
    const uint32_t ve = column(col, d.z, row_bytes), vf = column(col, d.w, row_bytes);
    if (POS) acc &= v0 & v1 & v2 & v3 & v4 & v5 & v6 & v7 & v8 & v9 & va & vb & vc & vd & ve & vf;
    else acc |= v0 | v1 | v2 | v3 | v4 | v5 | v6 | v7 | v8 | v9 | va | vb | vc | vd | ve | vf;
    const uint32_t live = POS ? (acc & ~other) : (other & ~acc);
    if (!__any_sync(kFull, live != 0u)) return POS ? 0u : kFull;  // every example falsified
  }
  for (; p < end; ++p) {
    const uint4 a = __ldg(p);
    const uint32_t v0 = column(col, a.x, row_bytes), v1 = column(col, a.y, row_bytes);
    const uint32_t v2 = column(col, a.z, row_bytes), v3 = column(col, a.w, row_bytes);
    if (POS) acc &= v0 & v1 & v2 & v3;
    else acc |= v0 | v1 | v2 | v3;
  }
  return acc;
}

// Short lists (a few literals, e.g. MNIST-shaped machines): the positive and
// negated parts in one loop of 8 loads — each aligned group of 4 entries is
// all positive or all negated (np is a multiple of 4), so the group's AND
// feeds `pos` and its OR feeds `neg` under a warp-uniform test.
__device__ __forceinline__ uint32_t fold_short(const uint32_t* __restrict__ lst, int len, int np,
                                               const char* __restrict__ col, uint32_t row_bytes, uint32_t pos) {
  const uint4* p = reinterpret_cast<const uint4*>(lst);
  uint32_t neg = 0u;
  int k = 0;
  for (; k + 8 <= len; k += 8, p += 2) {
    const uint4 a = __ldg(p), b = __ldg(p + 1);
    const uint32_t v0 = column(col, a.x, row_bytes), v1 = column(col, a.y, row_bytes);
    const uint32_t v2 = column(col, a.z, row_bytes), v3 = column(col, a.w, row_bytes);
    const uint32_t v4 = column(col, b.x, row_bytes), v5 = column(col, b.y, row_bytes);
    const uint32_t v6 = column(col, b.z, row_bytes), v7 = column(col, b.w, row_bytes);
    if (k < np) pos &= v0 & v1 & v2 & v3;
    else neg |= v0 | v1 | v2 | v3;
    if (k + 4 < np) pos &= v4 & v5 & v6 & v7;
    else neg |= v4 | v5 | v6 | v7;
    if (!__any_sync(kFull, (pos & ~neg) != 0u)) return 0u;  // every example falsified
  }
  if (k < len) {
    const uint4 a = __ldg(p);
    const uint32_t v0 = column(col, a.x, row_bytes), v1 = column(col, a.y, row_bytes);
    const uint32_t v2 = column(col, a.z, row_bytes), v3 = column(col, a.w, row_bytes);
    if (k < np) pos &= v0 & v1 & v2 & v3;
    else neg |= v0 | v1 | v2 | v3;
  }
  return pos & ~neg;
}

template <bool TRAIN>
__global__ void __launch_bounds__(kEvalWarps * 32, TMG_EVAL_MINB) eval_bits_kernel(BitsEvalParams P) {
  __shared__ uint32_t red[kEvalWarps][kSumPlanes][32];
  __shared__ int next_clause;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * 32 + lane;  // this lane's column word
  const int64_t e0 = gw * 32;
  const uint32_t valid = e0 >= P.q ? 0u : (P.q - e0 >= 32 ? kFull : ((1u << (P.q - e0)) - 1u));
  const int c = blockIdx.y / P.chunks;
  const int jc0 = (blockIdx.y % P.chunks) * P.cta_clauses;
  const int jc1 = min(jc0 + P.cta_clauses, P.n_loc);
  const char* __restrict__ col = reinterpret_cast<const char*>(P.lit_t + gw);
  const uint32_t row_bytes = P.Gs * 4u;
  if (threadIdx.x == 0) next_clause = jc0 + kEvalWarps;
  __syncthreads();
  uint32_t cnt[kSumPlanes];
#pragma unroll
  for (int b = 0; b < kSumPlanes; ++b) cnt[b] = 0u;
  // Clauses are handed out one at a time as warps finish (lists differ in
  // length; claiming ahead measured worse: a busy warp sits on its claim), so
  // the warps reach the CTA reduction below together. One 16-byte load per
  // clause: {list offset / 4, list length, positive-part length}.
  const int4* __restrict__ meta = P.meta + static_cast<size_t>(c) * P.n_loc;
  for (int jl = jc0 + warp; jl < jc1;) {
    const int4 mt = __ldg(meta + jl);
    const int len = mt.y, np = mt.z;
    uint32_t acc = valid;  // empty clause: Train 1
    if (TRAIN || len != 0) {  // empty clause: Predict 0 (core.hpp:211-213)
      const uint32_t* lst = P.lists + (static_cast<size_t>(static_cast<uint32_t>(mt.x)) << 2);
      if (!P.dynamic) {
        acc = fold_short(lst, len, np, col, row_bytes, acc);
      } else {
        acc = fold_columns<true>(lst, np, col, row_bytes, acc, 0u);
        if (__any_sync(kFull, acc != 0u) && len > np)
          acc &= ~fold_columns<false>(lst + np, len - np, col, row_bytes, 0u, acc);
      }
      if (TRAIN && P.prev != nullptr && gw < P.Wq)
        P.prev[(static_cast<size_t>(c) * P.n_loc + jl) * P.Wq + gw] = acc;
      const int j = P.j_begin + jl;
      if (P.all_positive || !(j & 1)) count_word<true>(cnt, acc);
      else count_word<false>(cnt, acc);
    }
    if (P.dynamic) {
      int nj = 0;
      if (lane == 0) nj = atomicAdd(&next_clause, 1);
      jl = __shfl_sync(kFull, nj, 0);
    } else {
      jl += kEvalWarps;  // short lists: a fixed stride, no claim on the critical path
    }
  }
  // CTA reduction of the warps' counters: bit-sliced ripple adds in shared memory.
#pragma unroll
  for (int b = 0; b < kSumPlanes; ++b) red[warp][b][lane] = cnt[b];
  __syncthreads();
  for (int half = kEvalWarps / 2; half >= 1; half >>= 1) {
    if (warp < half) {
      uint32_t carry = 0u;
#pragma unroll
      for (int b = 0; b < kSumPlanes; ++b) {
        const uint32_t x = red[warp][b][lane], y = red[warp + half][b][lane];
        red[warp][b][lane] = x ^ y ^ carry;
        carry = (x & y) | (carry & (x ^ y));
      }
    }
    __syncthreads();
  }
  // Per example: the K-bit two's-complement sum -> atomicAdd into sums[i][c].
  const int64_t ib = static_cast<int64_t>(blockIdx.x) * 1024;
  for (int x = threadIdx.x; x < 1024; x += kEvalWarps * 32) {
    const int64_t i = ib + x;
    if (i >= P.q) break;
    const int wd = x >> 5, bit = x & 31;
    int v = 0;
#pragma unroll
    for (int b = 0; b < kSumPlanes; ++b) v |= static_cast<int>((red[0][b][wd] >> bit) & 1u) << b;
    v = (v ^ (1 << (kSumPlanes - 1))) - (1 << (kSumPlanes - 1));
    if (v != 0) atomicAdd(P.sums + i * P.m + c, v);
  }
}

__global__ void counters_to_planes_kernel(const uint16_t* __restrict__ counters,
                                          uint32_t* __restrict__ state, int clauses, int o, int B,
                                          int Wp, int N) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(clauses) * 2 * Wp;
  if (idx >= total) return;
  const int w = static_cast<int>(idx % Wp);
  const int part = static_cast<int>((idx / Wp) % 2);
  const int64_t lc = idx / (2 * Wp);
  const int off = (1 << (B - 1)) - N - 1;  // plane value = counter + off
  uint32_t planes[15] = {0};
  const uint16_t* row = counters + lc * 2 * o;
  for (int b = 0; b < 32; ++b) {
    const int f = w * 32 + b;
    uint32_t v;
    if (f < o) v = static_cast<uint32_t>(row[part * o + f] + off);
    else v = static_cast<uint32_t>(N + off);  // padding: counter N (exclude, never touched)
    for (int pl = 0; pl < B; ++pl) planes[pl] |= ((v >> pl) & 1u) << b;
  }
  for (int pl = 0; pl < B; ++pl) state[((lc * B + pl) * 2 + part) * Wp + w] = planes[pl];
}

__global__ void planes_to_counters_kernel(const uint32_t* __restrict__ state,
                                          uint16_t* __restrict__ counters, int clauses, int o, int B,
                                          int Wp, int N) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = static_cast<int64_t>(clauses) * 2 * o;
  if (idx >= total) return;
  const int k = static_cast<int>(idx % (2 * o));
  const int64_t lc = idx / (2 * o);
  const int part = k >= o ? 1 : 0;
  const int f = k - part * o;
  const int w = f >> 5, b = f & 31;
  uint32_t v = 0;
  for (int pl = 0; pl < B; ++pl) v |= ((state[((lc * B + pl) * 2 + part) * Wp + w] >> b) & 1u) << pl;
  const int off = (1 << (B - 1)) - N - 1;
  counters[idx] = static_cast<uint16_t>(static_cast<int>(v) - off);
}

// bits: q x o uint8 (0/1) -> x plane (bit f = x_f), n plane (bit f = !x_f).
// Also validates the input (ExamplePool ctor, pool.cpp:42-46): err |= 1 on a
// byte other than 0/1.
__global__ void pack_planes_kernel(const uint8_t* __restrict__ bits, uint32_t* __restrict__ xplane,
                                   uint32_t* __restrict__ nplane, int64_t q, int o, int Wp, int* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t total = q * Wp;
  if (warp >= total) return;
  const int64_t i = warp / Wp;
  const int w = static_cast<int>(warp % Wp);
  const int f = w * 32 + lane;
  const bool valid = f < o;
  const uint8_t b = valid ? bits[i * o + f] : 0;
  if (b > 1) atomicOr(err, 1);
  const unsigned xs = __ballot_sync(kFull, valid && b);
  const unsigned ns = __ballot_sync(kFull, valid && !b);
  if (lane == 0) {
    xplane[i * 2 * Wp + w] = xs;
    nplane[i * 2 * Wp + w] = ns;
  }
}

// Label range check (pool.cpp:47-55): err[0] |= 2, err[1] = an offending label.
__global__ void check_labels_kernel(const int32_t* __restrict__ labels, int64_t q, int m, int* err) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= q) return;
  const int32_t y = labels[i];
  if (y < 0 || y >= m) {
    atomicOr(err, 2);
    atomicExch(err + 1, y);
  }
}

// Reference literal rows (q x ceil(2o/64) u64, core.cpp:34-46) -> planes.
__global__ void unpack_ref_kernel(const uint64_t* __restrict__ lits, uint32_t* __restrict__ xplane,
                                  uint32_t* __restrict__ nplane, int64_t q, int o, int Wp) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= q * Wp) return;
  const int64_t i = idx / Wp;
  const int w = static_cast<int>(idx % Wp);
  const int W64 = (2 * o + 63) / 64;
  const uint32_t* row = reinterpret_cast<const uint32_t*>(lits + i * W64);
  const int W32 = 2 * W64;
  auto bits_at = [&](int k) -> uint32_t {  // 32 bits starting at literal k
    const int wd = k >> 5, sh = k & 31;
    const uint32_t lo = wd < W32 ? row[wd] : 0u;
    const uint32_t hi = wd + 1 < W32 ? row[wd + 1] : 0u;
    return __funnelshift_r(lo, hi, sh);
  };
  const int f0 = w * 32;
  uint32_t vmask = f0 >= o ? 0u : (o - f0 >= 32 ? kFull : ((1u << (o - f0)) - 1u));
  xplane[i * 2 * Wp + w] = f0 < o ? (bits_at(f0) & vmask) : 0u;
  nplane[i * 2 * Wp + w] = f0 < o ? (bits_at(o + f0) & vmask) : 0u;
}

// classify (trainer.cpp:244-260): strict '>' keeps the lowest class on ties;
// a single bank is a binary machine with the unit step sum >= 0.
__global__ void argmax_kernel(const int32_t* __restrict__ sums, int32_t* __restrict__ pred, int64_t q,
                              int m) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= q) return;
  const int32_t* row = sums + i * m;
  if (m == 1) {
    pred[i] = row[0] >= 0 ? 1 : 0;
    return;
  }
  int best = 0;
  int32_t bs = row[0];
  for (int c = 1; c < m; ++c)
    if (row[c] > bs) {
      bs = row[c];
      best = c;
    }
  pred[i] = best;
}

// predict_scaled (regression.cpp:86-93): clause count clipped to [0, T].
__global__ void clamp_kernel(const int32_t* __restrict__ sums, int32_t* __restrict__ out, int64_t q, int T) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= q) return;
  const int32_t v = sums[i];
  out[i] = v < 0 ? 0 : (v > T ? T : v);
}

// After an allreduce of per-rank tally deltas: add the remote part
// (reduced - own) to the local replica and clear the own-delta buffer.
__global__ void apply_remote_delta_kernel(int32_t* __restrict__ tallies, const int32_t* __restrict__ reduced,
                                          int32_t* __restrict__ own, int64_t count) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  tallies[idx] += reduced[idx] - own[idx];
  own[idx] = 0;
}

// evaluate_clause (core.hpp:208-219) for one clause and one literal row.
__global__ void eval_one_kernel(const uint32_t* __restrict__ state, int lc, int B, int Wp,
                                const uint32_t* __restrict__ x, const uint32_t* __restrict__ n,
                                int train_mode, int32_t* out) {
  const uint32_t* top = state + (static_cast<size_t>(lc) * B + (B - 1)) * 2 * Wp;
  uint32_t viol = 0, any = 0;
  for (int w = threadIdx.x; w < Wp; w += 32) {
    const uint32_t ix = top[w], in = top[Wp + w];
    viol |= (ix & ~x[w]) | (in & ~n[w]);
    any |= ix | in;
  }
  const unsigned vb = __ballot_sync(kFull, viol != 0), ab = __ballot_sync(kFull, any != 0);
  if (threadIdx.x == 0) *out = ab == 0 ? train_mode : (vb == 0 ? 1 : 0);
}

// Fresh automata (ClassBank ctor, core.cpp:96-100): counter N is plane value
// 2^(B-1) - 1, i.e. every plane set except the top one.
__global__ void init_state_kernel(uint32_t* __restrict__ state, int64_t words, int B, int Wp) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= words) return;
  const int b = static_cast<int>((idx / (2 * Wp)) % B);
  state[idx] = b < B - 1 ? kFull : 0u;
}

inline unsigned blocks_for(int64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace

int64_t build_lists_launch(const uint32_t* state, int clauses, int B, int Wp, int Wx, int32_t* inc_count,
                           int32_t* lens, int32_t* npos, int64_t* offs, cudaStream_t s) {
  if (clauses <= 0) return 0;
  count_launch();
  count_literals_kernel<<<blocks_for(clauses, 4), 128, 0, s>>>(state, clauses, B, Wp, Wx, inc_count, lens, npos);
  count_launch();
  scan_lengths_kernel<<<1, 1024, 0, s>>>(lens, clauses, offs);
  int64_t total = 0;
  if (cudaMemcpyAsync(&total, offs + clauses, sizeof total, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return -1;
  return total;
}

void fill_lists_launch(const uint32_t* state, int clauses, int B, int Wp, int Wx, int o, const int64_t* offs,
                       const int32_t* npos, uint32_t* lists, int4* meta, cudaStream_t s) {
  if (clauses <= 0) return;
  count_launch();
  fill_literals_kernel<<<blocks_for(clauses, 4), 128, 0, s>>>(state, clauses, B, Wp, Wx, o, offs, npos, lists,
                                                              meta);
}

int64_t lit_t_stride(int64_t q) { return ((q + 31) / 32 + 31) / 32 * 32; }

void transpose_literals_launch(const uint32_t* xplane, int64_t row_stride, int64_t q, int o, uint32_t* lit_t,
                               cudaStream_t s) {
  const int64_t Gs = lit_t_stride(q);
  const int Wx = (o + 31) / 32;
  // rows o (all ones) and o + 1 (all zeros): the padding of the positive and
  // the negated clause lists
  cudaMemsetAsync(lit_t + static_cast<int64_t>(o) * Gs, 0xFF, Gs * sizeof(uint32_t), s);
  cudaMemsetAsync(lit_t + static_cast<int64_t>(o + 1) * Gs, 0, Gs * sizeof(uint32_t), s);
  count_launch();
  transpose_literals_kernel<<<dim3(static_cast<unsigned>(Gs / 32), Wx), 256, 0, s>>>(xplane, row_stride, q, o, Gs,
                                                                                      lit_t);
}

void eval_bits_launch(const BitsEvalParams& p, bool train_mode, cudaStream_t s) {
  if (p.q <= 0 || p.n_loc <= 0) return;
  dim3 grid(static_cast<unsigned>((p.q + 1023) / 1024), static_cast<unsigned>(p.m * p.chunks));
  count_launch();
  if (train_mode) eval_bits_kernel<true><<<grid, kEvalWarps * 32, 0, s>>>(p);
  else eval_bits_kernel<false><<<grid, kEvalWarps * 32, 0, s>>>(p);
}

void counters_to_planes_launch(const uint16_t* counters, uint32_t* state, int clauses, int o, int B,
                               int Wp, int N, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(clauses) * 2 * Wp;
  if (total > 0) {
    count_launch();
    counters_to_planes_kernel<<<blocks_for(total, 256), 256, 0, s>>>(counters, state, clauses, o, B, Wp, N);
  }
}

void planes_to_counters_launch(const uint32_t* state, uint16_t* counters, int clauses, int o, int B,
                               int Wp, int N, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(clauses) * 2 * o;
  if (total > 0) {
    count_launch();
    planes_to_counters_kernel<<<blocks_for(total, 256), 256, 0, s>>>(state, counters, clauses, o, B, Wp, N);
  }
}

void check_labels_launch(const int32_t* labels, int64_t q, int m, int* err, cudaStream_t s) {
  if (q <= 0) return;
  count_launch();
  check_labels_kernel<<<blocks_for(q, 256), 256, 0, s>>>(labels, q, m, err);
}

void pack_planes_launch(const uint8_t* bits, uint32_t* xplane, uint32_t* nplane, int64_t q, int o,
                        int Wp, int* err, cudaStream_t s) {
  const int64_t threads = q * Wp * 32;
  if (threads > 0) {
    count_launch();
    pack_planes_kernel<<<blocks_for(threads, 256), 256, 0, s>>>(bits, xplane, nplane, q, o, Wp, err);
  }
}

void unpack_ref_literals_launch(const uint64_t* lits, uint32_t* xplane, uint32_t* nplane, int64_t q,
                                int o, int Wp, cudaStream_t s) {
  if (q * Wp > 0) {
    count_launch();
    unpack_ref_kernel<<<blocks_for(q * Wp, 256), 256, 0, s>>>(lits, xplane, nplane, q, o, Wp);
  }
}

void argmax_launch(const int32_t* sums, int32_t* pred, int64_t q, int m, cudaStream_t s) {
  if (q > 0) {
    count_launch();
    argmax_kernel<<<blocks_for(q, 256), 256, 0, s>>>(sums, pred, q, m);
  }
}

void clamp_launch(const int32_t* sums, int32_t* out, int64_t q, int T, cudaStream_t s) {
  if (q <= 0) return;
  count_launch();
  clamp_kernel<<<blocks_for(q, 256), 256, 0, s>>>(sums, out, q, T);
}

void eval_one_launch(const uint32_t* state, int lc, int B, int Wp, const uint32_t* x, const uint32_t* n,
                     int train_mode, int32_t* out, cudaStream_t s) {
  count_launch();
  eval_one_kernel<<<1, 32, 0, s>>>(state, lc, B, Wp, x, n, train_mode, out);
}

void init_state_launch(uint32_t* state, int clauses, int B, int Wp, cudaStream_t s) {
  const int64_t words = static_cast<int64_t>(clauses) * B * 2 * Wp;
  if (words > 0) {
    count_launch();
    init_state_kernel<<<blocks_for(words, 256), 256, 0, s>>>(state, words, B, Wp);
  }
}

__global__ void apply_snapshot_kernel(int32_t* __restrict__ tallies, const int32_t* __restrict__ reduced,
                                      const int32_t* __restrict__ snap, int64_t count) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < count) tallies[idx] += reduced[idx] - snap[idx];
}

void apply_snapshot_launch(int32_t* tallies, const int32_t* reduced, const int32_t* snap, int64_t count,
                           cudaStream_t s) {
  if (count > 0) {
    count_launch();
    apply_snapshot_kernel<<<blocks_for(count, 256), 256, 0, s>>>(tallies, reduced, snap, count);
  }
}

void apply_remote_delta_launch(int32_t* tallies, const int32_t* reduced, int32_t* own, int64_t count,
                               cudaStream_t s) {
  if (count > 0) {
    count_launch();
    apply_remote_delta_kernel<<<blocks_for(count, 256), 256, 0, s>>>(tallies, reduced, own, count);
  }
}

}  // namespace tmg

// ------------------------------------------------- integer-pipe peak probe ---
// Roofline denominator for the INT-bound kernels (MEASURED_PEAKS.json has no
// integer figure): 8 independent LOP3 chains per thread (ALU pipe), and the
// same interleaved 1:1 with IMAD (FMA pipe) for the dual-pipe issue peak.
namespace tmg {
namespace {
template <bool MIXED>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t* sink, int iters, uint32_t seed) {
  uint32_t a[8], b[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = seed * (threadIdx.x + 1) + k;
    b[k] = seed ^ (blockIdx.x * 977u + k);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a[k]), "r"(b[k]), "r"(a[(k + 1) & 7]));
      a[k] = r;
      if (MIXED) {
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b[k]), "r"(0x9E3779B9u), "r"(a[k]));
        b[k] = r;
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= a[k] ^ b[k];
  if (acc == 0x12345678u) sink[0] = acc;
}
}  // namespace

bool int_peak_launch(int sms, double* lop3_ops, double* mixed_ops) {
  uint32_t* sink = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return false;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double res[2] = {0, 0};
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {  // first rep is warm-up
      cudaEventRecord(e0);
      count_launch();
      if (mode == 0) int_peak_kernel<false><<<blocks, threads>>>(sink, iters, 12345u);
      else int_peak_kernel<true><<<blocks, threads>>>(sink, iters, 12345u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = static_cast<double>(blocks) * threads * iters * 8 * (mode ? 2 : 1);
      res[mode] = std::max(res[mode], ops / (ms * 1e-3));
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  *lop3_ops = res[0];
  *mixed_ops = res[1];
  return cudaGetLastError() == cudaSuccess;
}
}  // namespace tmg
