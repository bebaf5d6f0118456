// eval.cu — clause evaluation / class sums (inference and exact tally
// refresh), literal packing and automaton-state layout conversion.
//
// Class sums replace vote_sum / export_vote_sums / predict_all
// (proj/src/pool.cpp:82-91, proj/src/trainer.cpp:244-279); the train-mode
// variant with previous-output bitmaps replaces refresh_tallies
// (proj/src/pool.cpp:108-124).
//
// Trained clauses are very sparse (tens of included literals out of 2o), so
// each clause is first compacted to the list of its nonzero include words
// (build_entries). A CTA owns a tile of 128 examples staged in shared memory
// word-major (conflict-free: lane = example) and a chunk of clauses of one
// class; every thread evaluates its example against each clause's word list
// (a warp-uniform loop over broadcast loads) with a warp-wide early exit.
#include <algorithm>

#include "kernels.h"
#include "tm_device.cuh"

#ifndef TMG_EVAL_STAGE
#define TMG_EVAL_STAGE 4  // (r1au: 4 -> 1.22 ms, 32 -> 1.48, unstaged 1.33) clauses whose include lists a CTA stages in shared memory at a time
#endif

namespace tmg {

namespace {

// Examples per CTA in eval_sums: 128 (one thread each), or 32 for very wide
// rows (IMDb) so the staged tile fits in shared memory. Rows are padded to
// TILE+1 words: conflict-free staging and reads.

// One warp per clause: list its nonzero include words and count includes.
__global__ void build_entries_kernel(const uint32_t* __restrict__ state, int clauses, int B, int Wp,
                                     int Wx, EvalEntry* __restrict__ entries,
                                     int32_t* __restrict__ nentries, int32_t* __restrict__ inc_count) {
  const int lane = threadIdx.x & 31;
  const int lc = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (lc >= clauses) return;
  const uint32_t* top = state + (static_cast<size_t>(lc) * B + (B - 1)) * 2 * Wp;
  EvalEntry* out = entries + static_cast<size_t>(lc) * Wx;
  int base = 0, cnt = 0;
  for (int w0 = 0; w0 < Wx; w0 += 32) {
    const int w = w0 + lane;
    uint32_t ix = 0, in = 0;
    if (w < Wx) {
      ix = top[w];
      in = top[Wp + w];
    }
    cnt += __popc(ix) + __popc(in);
    const bool nz = (ix | in) != 0;
    const unsigned bal = __ballot_sync(kFull, nz);
    if (nz) out[base + __popc(bal & ((1u << lane) - 1u))] = EvalEntry{static_cast<uint32_t>(w), ix, in, 0u};
    base += __popc(bal);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  if (lane == 0) {
    nentries[lc] = base;
    inc_count[lc] = cnt;
  }
}

template <bool TRAIN, int kTile>
__global__ void __launch_bounds__(kTile) eval_sums_kernel(EvalParams P) {
  constexpr int kTS = kTile + 1;
  extern __shared__ uint32_t tile[];  // [2][Wx][kTS], then P.stage staged clauses' entries
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t i = i0 + tid;
  const bool live = i < P.q;
  // Stage the literal planes of the example tile, transposed to word-major.
  for (int idx = tid; idx < P.Wx * kTile; idx += kTile) {
    const int e = idx / P.Wx, w = idx % P.Wx;
    const int64_t ie = i0 + e;
    uint32_t xv = 0, nv = 0;
    if (ie < P.q) {
      xv = __ldg(P.xplane + ie * 2 * P.Wp + w);
      nv = __ldg(P.nplane + ie * 2 * P.Wp + w);
    }
    tile[w * kTS + e] = xv;
    tile[(P.Wx + w) * kTS + e] = nv;
  }
  __syncthreads();

  const int chunks = (P.n_loc + P.chunk - 1) / P.chunk;
  const int c = blockIdx.y / chunks;
  const int jl0 = (blockIdx.y % chunks) * P.chunk;
  const int jl1 = min(jl0 + P.chunk, P.n_loc);
  // Clause include-word lists are staged P.stage clauses at a time (every
  // warp copies whole lists, coalesced), so the evaluation loop reads them
  // from shared memory instead of a dependent global load per clause.
  uint4* sent = reinterpret_cast<uint4*>(tile + ((2 * P.Wx * kTS + 3) & ~3));
  int* sne = reinterpret_cast<int*>(sent + static_cast<size_t>(P.stage) * P.Wx);
  const int warp = tid >> 5, nwarps = kTile >> 5;
  int sum = 0;
  for (int jb = jl0; jb < jl1; jb += P.stage) {
    const int nb = min(P.stage, jl1 - jb);
    __syncthreads();  // the previous block's lists are consumed
    for (int cs = warp; cs < nb; cs += nwarps) {
      const int lc = c * P.n_loc + jb + cs;
      const int ne = __ldg(P.nentries + lc);
      const uint4* src = reinterpret_cast<const uint4*>(P.entries + static_cast<size_t>(lc) * P.Wx);
      for (int k = lane; k < ne; k += 32) {
        uint4 en = __ldg(src + k);
        en.w = (P.Wx + en.x) * kTS;  // !x-plane row of word w in the tile
        en.x *= kTS;                 // x-plane row
        sent[cs * P.Wx + k] = en;
      }
      if (lane == 0) sne[cs] = ne;
    }
    __syncthreads();
    for (int cs = 0; cs < nb; ++cs) {
      const int jl = jb + cs;
      const int lc = c * P.n_loc + jl;
      const int ne = sne[cs];
      int out;
      if (ne == 0) {
        out = TRAIN ? 1 : 0;  // empty-clause convention (core.hpp:211-213)
      } else {
        const uint4* en = sent + cs * P.Wx;
        const uint32_t* xt = tile + tid;  // this example's column of the tile
        uint32_t viol = 0;
        for (int k = 0; k < ne; k += 4) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (k + u < ne) {
              const uint4 ent = en[k + u];
              viol |= (ent.y & ~xt[ent.x]) | (ent.z & ~xt[ent.w]);
            }
          }
          if (__all_sync(kFull, viol != 0 || !live)) break;
        }
        out = viol == 0 ? 1 : 0;
      }
      const int j = P.j_begin + jl;
      sum += (!P.all_positive && (j & 1)) ? -out : out;
      if (TRAIN && P.prev != nullptr) {  // refresh_tallies also rewrites previous outputs
        const unsigned bits = __ballot_sync(kFull, live && out);
        if (lane == 0 && i < P.q) P.prev[static_cast<size_t>(lc) * P.Wq + (i >> 5)] = bits;
      }
    }
  }
  if (live) atomicAdd(P.sums + i * P.m + c, sum);
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

// Rows too wide for even a 32-example staged tile (beyond ~26k features):
// each thread reads its example's literal words straight from HBM/L2 at the
// clause's include-list positions, and the lists are read from global memory.
template <bool TRAIN>
__global__ void __launch_bounds__(128) eval_sums_direct_kernel(EvalParams P) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * 128 + tid;
  const bool live = i < P.q;
  const uint32_t* xr = P.xplane + (live ? i : 0) * 2 * P.Wp;
  const int chunks = (P.n_loc + P.chunk - 1) / P.chunk;
  const int c = blockIdx.y / chunks;
  const int jl0 = (blockIdx.y % chunks) * P.chunk;
  const int jl1 = min(jl0 + P.chunk, P.n_loc);
  int sum = 0;
  for (int jl = jl0; jl < jl1; ++jl) {
    const int lc = c * P.n_loc + jl;
    const int ne = __ldg(P.nentries + lc);
    int out;
    if (ne == 0) {
      out = TRAIN ? 1 : 0;  // empty-clause convention (core.hpp:211-213)
    } else {
      const uint4* en = reinterpret_cast<const uint4*>(P.entries + static_cast<size_t>(lc) * P.Wx);
      uint32_t viol = 0;
      for (int k = 0; k < ne; ++k) {
        const uint4 ent = __ldg(en + k);
        viol |= (ent.y & ~__ldg(xr + ent.x)) | (ent.z & ~__ldg(xr + P.Wp + ent.x));
        if (__all_sync(kFull, viol != 0 || !live)) break;
      }
      out = viol == 0 ? 1 : 0;
    }
    const int j = P.j_begin + jl;
    sum += (!P.all_positive && (j & 1)) ? -out : out;
    if (TRAIN && P.prev != nullptr) {
      const unsigned bits = __ballot_sync(kFull, live && out);
      if (lane == 0 && i < P.q) P.prev[static_cast<size_t>(lc) * P.Wq + (i >> 5)] = bits;
    }
  }
  if (live) atomicAdd(P.sums + i * P.m + c, sum);
}

inline unsigned blocks_for(int64_t n, int per) { return static_cast<unsigned>((n + per - 1) / per); }

}  // namespace

void build_entries_launch(const uint32_t* state, int clauses, int B, int Wp, int Wx, EvalEntry* e,
                          int32_t* ne, int32_t* inc_count, cudaStream_t s) {
  if (clauses <= 0) return;
  count_launch();
  build_entries_kernel<<<blocks_for(clauses, 4), 128, 0, s>>>(state, clauses, B, Wp, Wx, e, ne, inc_count);
}

void eval_sums_launch(const EvalParams& p, bool train_mode, cudaStream_t s) {
  if (p.q <= 0 || p.n_loc <= 0) return;
  const int chunks = (p.n_loc + p.chunk - 1) / p.chunk;
  auto go = [&](auto kern, int tile) {
    dim3 grid(blocks_for(p.q, tile), p.m * chunks);
    EvalParams q = p;
    // ~16 KB of staged include lists per CTA (at least one clause).
    q.stage = std::max(1, std::min(TMG_EVAL_STAGE, static_cast<int>((16 * 1024) / (16 * std::max(1, p.Wx)))));
    const size_t shm = sizeof(uint32_t) * ((2 * p.Wx * (tile + 1) + 3) & ~3) +
                       sizeof(uint4) * static_cast<size_t>(q.stage) * p.Wx + sizeof(int) * q.stage;
    if (shm > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shm));
    count_launch();
    kern<<<grid, tile, shm, s>>>(q);
  };
  const bool wide = sizeof(uint32_t) * 2 * p.Wx * 129 > 200 * 1024;
  const bool direct = sizeof(uint32_t) * 2 * p.Wx * 33 + 16 * p.Wx + 16 > 200 * 1024;
  if (direct) {
    dim3 grid(blocks_for(p.q, 128), p.m * chunks);
    count_launch();
    if (train_mode) eval_sums_direct_kernel<true><<<grid, 128, 0, s>>>(p);
    else eval_sums_direct_kernel<false><<<grid, 128, 0, s>>>(p);
    return;
  }
  if (train_mode) {
    if (wide) go(eval_sums_kernel<true, 32>, 32);
    else go(eval_sums_kernel<true, 128>, 128);
  } else {
    if (wide) go(eval_sums_kernel<false, 32>, 32);
    else go(eval_sums_kernel<false, 128>, 128);
  }
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
