// sequential.cu — bit-exact GPU mirror of the classic sequential trainer
// (train_epoch_sequential / feed_bank_sequential, proj/src/trainer.cpp:57-85,
// 138-179).
//
// One CTA per epoch. Per example the two fed banks are evaluated by all warps
// in parallel (clause per warp, literal words per lane, Train mode), the vote
// sum is reduced in shared memory, and warp 0 then replays the reference's
// single xoshiro256++ stream: one gate draw per clause, 2o Type I draws in
// literal order, the negative-class draw below(m-1) — exactly the reference's
// draw order, so automaton states match bit for bit. The automata are read
// and written in place in their bit-plane layout (any NW, any B).
#include <algorithm>

#include <cooperative_groups.h>

#include "kernels.h"
#include "tm_device.cuh"

namespace tmg {

namespace {

constexpr int kSeqThreads = 1024;

// TMG_STATS builds: phase cycle counts of the grid replay's lead warp in
// P.dbg[200..204] (vote+barrier, scan, barrier, apply+barrier, jumps in scan).
#ifdef TMG_STATS
#define TMG_SEQ_CLOCK(var) const long long var = clock64()
#define TMG_SEQ_ADD(k, v) \
  if (P.dbg && lane == 0) P.dbg[k] += static_cast<unsigned long long>(v)
#else
#define TMG_SEQ_CLOCK(var)
#define TMG_SEQ_ADD(k, v)
#endif

__device__ __forceinline__ uint32_t below_dev(Xoshiro& r, uint32_t bound) {  // rng.hpp:68-79
  uint64_t m = static_cast<uint64_t>(static_cast<uint32_t>(r.next())) * bound;
  uint32_t low = static_cast<uint32_t>(m);
  if (low < bound) {
    const uint32_t cutoff = (0u - bound) % bound;
    while (low < cutoff) {
      m = static_cast<uint64_t>(static_cast<uint32_t>(r.next())) * bound;
      low = static_cast<uint32_t>(m);
    }
  }
  return static_cast<uint32_t>(m >> 32);
}

template <int B>
__device__ __forceinline__ void load_word(const uint32_t* base, int Wp, int part, int w, Planes<B>& s) {
#pragma unroll
  for (int b = 0; b < B; ++b) s.p[b] = base[(b * 2 + part) * Wp + w];
}

template <int B>
__device__ __forceinline__ void store_word(uint32_t* base, int Wp, int part, int w, const Planes<B>& s) {
#pragma unroll
  for (int b = 0; b < B; ++b) base[(b * 2 + part) * Wp + w] = s.p[b];
}

__device__ __forceinline__ uint32_t valid_bits(int w, int o) {
  const int first = w * 32;
  return first >= o ? 0u : (o - first >= 32 ? kFull : ((1u << (o - first)) - 1u));
}

// The gate probability of a fed bank (feedback.cpp:24-28; regression:
// regression.cpp:46-48, 145-151) and, for regression, whether the step is Type I.
__device__ __forceinline__ double bank_gate(const TrainParams& P, int v0, int y, int target, bool& regress_type1) {
  const int T = P.margin;
  regress_type1 = false;
  if (P.regress) {
    const int vc = v0 < 0 ? 0 : (v0 > T ? T : v0);
    const int e = y > vc ? y - vc : vc - y;
    regress_type1 = vc < y;
    return fmin(1.0, static_cast<double>(e) / (2.0 * static_cast<double>(T)));
  }
  const int vc = v0 < -T ? -T : (v0 > T ? T : v0);
  const int e = target ? T - vc : T + vc;
  return static_cast<double>(e) / (2.0 * static_cast<double>(T));
}

__device__ __forceinline__ bool is_type2(const TrainParams& P, int j, int target, bool regress_type1) {
  const bool positive = P.all_positive || (j & 1) == 0;
  return P.regress ? !regress_type1 : (target == 1) != positive;
}

// Parallel replay, phase 1 (one warp): gate draws in clause order; a gated
// Type I clause's state is recorded in S.tstate and its 2o draws skipped with
// one jump (jl = M^(2o)). Gated bits go to gbits. Every lane steps its own
// copy of the stream (identical in all lanes after the broadcast below), so
// the loop is warp-uniform without shuffles; the gate is the integer test
// next() < tp << 11 (tm_device.cuh u53_below), the Type I candidates a
// per-feed bit pattern over j mod 32. Returns the number of gated clauses.
__device__ unsigned long long scan_bank(const TrainParams& P, const SeqParams& S, Xoshiro& rng, double p, int target,
                                        bool regress_type1, const uint32_t* jl, uint32_t* gbits, int lane) {
  {
    uint64_t q[4] = {rng.s0, rng.s1, rng.s2, rng.s3};
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = __shfl_sync(kFull, q[k], 0);
    rng = Xoshiro{q[0], q[1], q[2], q[3]};
  }
  const uint64_t tp = u53_below(p);
  const bool every = (tp >> 53) != 0;  // p >= 1
  const uint64_t th = tp << 11;        // (next >> 11) < tp  <=>  next < tp * 2^11
  // is_type2 == false, as bits of j - j0 (j0 even)
  const uint32_t cand = P.regress ? (regress_type1 ? kFull : 0u)
                                  : (P.all_positive ? (target ? kFull : 0u) : (target ? 0x55555555u : 0xAAAAAAAAu));
  unsigned long long gated_n = 0;
  Xoshiro r = rng;
  for (int j0 = 0; j0 < P.n; j0 += 32) {
    const int nb = min(32, P.n - j0);
    uint32_t gw = 0;
    for (int b = 0; b < nb; ++b) {
      if (!every && r.next() >= th) continue;  // skip iff u >= p (trainer.cpp:121)
      if (every) r.next();
      gw |= 1u << b;
      if (!((cand >> b) & 1u)) continue;
      TMG_SEQ_CLOCK(j0c);
      if (lane == 0) {
        uint64_t* ts = S.tstate + static_cast<size_t>(j0 + b) * 4;
        ts[0] = r.s0;
        ts[1] = r.s1;
        ts[2] = r.s2;
        ts[3] = r.s3;
      }
      uint32_t sw[8];
      state_to_words(r, sw);
      gf2_apply(jl, sw, lane);
      r = words_to_state(sw);
      TMG_SEQ_ADD(204, clock64() - j0c);
    }
    gated_n += __popc(gw);
    if (lane == 0) gbits[j0 >> 5] = gw;
  }
  rng = r;
  return gated_n;
}

// Parallel replay, phase 2: one warp applies gated clause j of bank c
// (feedback.cpp:32-99). A Type I clause regenerates its 2o draws from the
// recorded state: lane L jumps to draw L * chunk (jc = M^chunk, applied lane
// by lane) and draws its segment into the warp's hb / lb bit buffers.
template <int B>
__device__ void apply_gated(const TrainParams& P, const SeqParams& S, int c, int j, int out, bool type2,
                            const uint32_t* xr, const uint32_t* nr, const uint32_t* jc, uint32_t* hb, uint32_t* lb,
                            int refw, int lane) {
  const int Wp = P.Wp, L = 2 * P.o;
  uint32_t* base = P.state + (static_cast<size_t>(c) * P.n + j) * (static_cast<size_t>(B) * 2 * Wp);
  if (type2) {  // Type II (feedback.cpp:72-83)
    if (!out) return;
    for (int w = lane; w < Wp; w += 32) {
      const uint32_t vm = valid_bits(w, P.o);
      for (int part = 0; part < 2; ++part) {
        Planes<B> s;
        load_word<B>(base, Wp, part, w, s);
        const uint32_t lit = part ? nr[w] : xr[w];
        const uint32_t inc = ~lit & ~s.p[B - 1] & vm;
        if (inc) {
          add_one<B>(s, inc);
          store_word<B>(base, Wp, part, w, s);
        }
      }
    }
    return;
  }
  for (int k = lane; k < 2 * refw; k += 32) hb[k] = 0;  // hb, then lb
  const uint64_t* ts = S.tstate + static_cast<size_t>(j) * 4;  // written by the scanning warp (L2 reads)
  Xoshiro r0{__ldcg(ts), __ldcg(ts + 1), __ldcg(ts + 2), __ldcg(ts + 3)};
  uint32_t sw[8], mine[8];
  state_to_words(r0, sw);
#pragma unroll
  for (int w = 0; w < 8; ++w) mine[w] = sw[w];
  for (int hop = 1; hop < 32; ++hop) {
    if (hop * S.chunk >= L) break;  // warp-uniform
    gf2_apply(jc, sw, lane);
    if (lane == hop) {
#pragma unroll
      for (int w = 0; w < 8; ++w) mine[w] = sw[w];
    }
  }
  __syncwarp();
  Xoshiro rl = words_to_state(mine);
  const int k0 = lane * S.chunk, k1 = min(L, k0 + S.chunk);
  const uint64_t th = u53_below(S.p_high), tl = u53_below(S.p_low);
  uint32_t hw = 0, lw = 0;
  int cw = k0 >> 5;
  for (int k = k0; k < k1; ++k) {
    if ((k >> 5) != cw) {
      if (hw) atomicOr(&hb[cw], hw);
      if (lw) atomicOr(&lb[cw], lw);
      hw = lw = 0;
      cw = k >> 5;
    }
    const uint64_t u = next53(rl);
    hw |= (u < th ? 1u : 0u) << (k & 31);
    lw |= (u < tl ? 1u : 0u) << (k & 31);
  }
  if (k1 > k0) {
    if (hw) atomicOr(&hb[cw], hw);
    if (lw) atomicOr(&lb[cw], lw);
  }
  __syncwarp();
  for (int w = lane; w < Wp; w += 32) {
    if (w * 32 >= P.o) continue;
    const uint32_t vm = valid_bits(w, P.o);
    const int kk = P.o + w * 32;
    const uint32_t hsel[2] = {hb[w], __funnelshift_r(hb[kk >> 5], hb[(kk >> 5) + 1], kk & 31)};
    const uint32_t lsel[2] = {lb[w], __funnelshift_r(lb[kk >> 5], lb[(kk >> 5) + 1], kk & 31)};
    for (int part = 0; part < 2; ++part) {
      Planes<B> s;
      load_word<B>(base, Wp, part, w, s);
      const uint32_t lit = part ? nr[w] : xr[w];
      uint32_t inc = 0, dec;
      if (out) {
        const uint32_t bern = (lit & hsel[part]) | (~lit & lsel[part]);
        const uint32_t incl = s.p[B - 1];
        inc = ((lit & (bern | (P.boost ? incl : 0u))) | (~lit & bern & incl)) & vm;
        dec = ~lit & bern & ~incl & vm;
      } else {
        dec = lsel[part] & vm;
      }
      step<B>(s, inc, dec, P.lo, P.hi);
      store_word<B>(base, Wp, part, w, s);
    }
  }
  __syncwarp();
}

template <int B>
__global__ void __launch_bounds__(kSeqThreads) train_sequential_kernel(TrainParams P, SeqParams S) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int L = 2 * P.o;
  const int refw = (L + 31) / 32 + 2;
  // parallel replay (S.jump_chunk != null): jump tables first (16-byte
  // aligned), then the serial replay's draw bits and the clause outputs, then
  // the gated bits and per-warp draw buffers (hbits / lbits of the clause a
  // warp is applying)
  const int tabw = S.jump_chunk ? 2 * kGf2TabWords : 0;
  uint32_t* jc = smem;
  uint32_t* jl = jc + kGf2TabWords;
  uint32_t* hbits = smem + tabw;          // u < p_high, reference literal order
  uint32_t* lbits = hbits + refw;         // u < p_low
  uint32_t* outs = lbits + refw;          // clause outputs of the fed bank (bit per clause)
  const int nwords = (P.n + 31) / 32;
  uint32_t* gbits = outs + nwords;
  uint32_t* wbuf = gbits + nwords;
  __shared__ int vote;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int n = P.n, Wp = P.Wp, T = P.margin;
  const size_t cstride = static_cast<size_t>(B) * 2 * Wp;
  Xoshiro rng{S.rng[0], S.rng[1], S.rng[2], S.rng[3]};
  unsigned long long ev_local = 0;
  for (int k = tid; k < 2 * refw; k += blockDim.x) hbits[k] = 0;
  const bool par = S.jump_chunk != nullptr;
  if (par) {
    for (int k = tid; k < kGf2TabWords; k += blockDim.x) {
      jc[k] = S.jump_chunk[k];
      jl[k] = S.jump_lits[k];
    }
  }

  for (int64_t t = 0; t < P.q; ++t) {
    const int64_t i = P.order[t];
    const int y = P.labels[i];
    // negative class (trainer.cpp:159-165), drawn before the two feeds
    __shared__ int neg_s;
    if (tid == 0) {
      int neg;
      if (P.regress) {
        neg = 0;  // regression: one feed of the single bank per example
      } else if (P.m == 2) {
        neg = 1 - y;
      } else {
        neg = static_cast<int>(below_dev(rng, static_cast<uint32_t>(P.m - 1)));
        if (neg >= y) ++neg;
      }
      neg_s = neg;
    }
    __syncthreads();
    const int neg = neg_s;
    const uint32_t* xr = P.xplane + i * 2 * Wp;
    const uint32_t* nr = P.nplane + i * 2 * Wp;
    for (int feed = 0; feed < (P.regress ? 1 : 2); ++feed) {
      const int c = P.regress ? 0 : (feed == 0 ? y : neg);
      const int target = feed == 0 ? 1 : 0;
      // ---- vote pass: every clause of bank c, Train mode (trainer.cpp:62-68)
      if (tid == 0) vote = 0;
      for (int k = tid; k < (n + 31) / 32; k += blockDim.x) outs[k] = 0;
      __syncthreads();
      for (int j = warp; j < n; j += nwarps) {
        const uint32_t* top = P.state + (static_cast<size_t>(c) * n + j) * cstride + static_cast<size_t>(B - 1) * 2 * Wp;
        uint32_t viol = 0, any = 0;
        for (int w = lane; w < Wp; w += 32) {
          const uint32_t ix = top[w], in = top[Wp + w];
          viol |= (ix & ~xr[w]) | (in & ~nr[w]);
          any |= ix | in;
        }
        const unsigned vb = __ballot_sync(kFull, viol != 0), ab = __ballot_sync(kFull, any != 0);
        const int out = ab == 0 ? 1 : (vb == 0 ? 1 : 0);
        if (lane == 0 && out) {
          atomicOr(&outs[j >> 5], 1u << (j & 31));
          atomicAdd(&vote, (!P.all_positive && (j & 1)) ? -1 : 1);
        }
      }
      __syncthreads();
      if (par) {
        // ---- parallel replay: the gate scan by warp 0 (scan_bank), then the
        // gated clauses applied one warp each (apply_gated).
        bool regress_type1;
        const double p = bank_gate(P, vote, y, target, regress_type1);
        if (warp == 0) {
          const unsigned long long g = scan_bank(P, S, rng, p, target, regress_type1, jl, gbits, lane);
          if (lane == 0) S.events[c] += g;
        }
        __syncthreads();
        if (warp < S.par_warps) {
          uint32_t* hb = wbuf + static_cast<size_t>(warp) * 2 * refw;
          for (int j = warp; j < n; j += S.par_warps) {
            if (!((gbits[j >> 5] >> (j & 31)) & 1u)) continue;
            apply_gated<B>(P, S, c, j, (outs[j >> 5] >> (j & 31)) & 1, is_type2(P, j, target, regress_type1), xr, nr,
                           jc, hb, hb + refw, refw, lane);
          }
        }
        __syncthreads();
        continue;
      }
      // ---- serial gate + feedback replay by warp 0 (trainer.cpp:69-83)
      if (warp == 0) {
        const int v0 = vote;
        double p;
        bool regress_type1 = false;
        if (P.regress) {  // regression.cpp:46-48, 145-151 (t = scaled target)
          const int vc = v0 < 0 ? 0 : (v0 > T ? T : v0);
          const int e = y > vc ? y - vc : vc - y;
          p = fmin(1.0, static_cast<double>(e) / (2.0 * static_cast<double>(T)));
          regress_type1 = vc < y;
        } else {
          const int vc = v0 < -T ? -T : (v0 > T ? T : v0);
          const int e = target ? T - vc : T + vc;
          p = static_cast<double>(e) / (2.0 * static_cast<double>(T));
        }
        const uint64_t tp = u53_below(p);
        for (int j = 0; j < n; ++j) {
          int gated = 0;
          if (lane == 0) gated = next53(rng) < tp ? 1 : 0;
          gated = __shfl_sync(kFull, gated, 0);
          if (!gated) continue;
          ++ev_local;
          const int out = (outs[j >> 5] >> (j & 31)) & 1;
          uint32_t* base = P.state + (static_cast<size_t>(c) * n + j) * cstride;
          const bool positive = P.all_positive || (j & 1) == 0;
          const bool type2 = P.regress ? !regress_type1 : (target == 1) != positive;
          if (type2) {  // Type II (feedback.cpp:72-83)
            if (out) {
              for (int w = lane; w < Wp; w += 32) {
                const uint32_t vm = valid_bits(w, P.o);
                for (int part = 0; part < 2; ++part) {
                  Planes<B> s;
                  load_word<B>(base, Wp, part, w, s);
                  const uint32_t lit = part ? nr[w] : xr[w];
                  const uint32_t inc = ~lit & ~s.p[B - 1] & vm;
                  if (inc) {
                    add_one<B>(s, inc);
                    store_word<B>(base, Wp, part, w, s);
                  }
                }
              }
            }
          } else {  // Type I: 2o draws in literal order (feedback.cpp:45,63)
            if (lane == 0) {
              const uint64_t th = u53_below(S.p_high), tl = u53_below(S.p_low);
              uint32_t hw = 0, lw = 0;
              for (int k = 0; k < L; ++k) {
                const uint64_t u = next53(rng);
                hw |= (u < th ? 1u : 0u) << (k & 31);
                lw |= (u < tl ? 1u : 0u) << (k & 31);
                if ((k & 31) == 31 || k == L - 1) {
                  hbits[k >> 5] = hw;
                  lbits[k >> 5] = lw;
                  hw = lw = 0;
                }
              }
            }
            __syncwarp();
            for (int w = lane; w < Wp; w += 32) {
              if (w * 32 >= P.o) continue;
              const uint32_t vm = valid_bits(w, P.o);
              const int k1 = P.o + w * 32;
              const uint32_t hsel[2] = {hbits[w], __funnelshift_r(hbits[k1 >> 5], hbits[(k1 >> 5) + 1], k1 & 31)};
              const uint32_t lsel[2] = {lbits[w], __funnelshift_r(lbits[k1 >> 5], lbits[(k1 >> 5) + 1], k1 & 31)};
              for (int part = 0; part < 2; ++part) {
                Planes<B> s;
                load_word<B>(base, Wp, part, w, s);
                const uint32_t lit = part ? nr[w] : xr[w];
                uint32_t inc = 0, dec;
                if (out) {
                  const uint32_t bern = (lit & hsel[part]) | (~lit & lsel[part]);
                  const uint32_t incl = s.p[B - 1];
                  inc = ((lit & (bern | (P.boost ? incl : 0u))) | (~lit & bern & incl)) & vm;
                  dec = ~lit & bern & ~incl & vm;
                } else {
                  dec = lsel[part] & vm;
                }
                step<B>(s, inc, dec, P.lo, P.hi);
                store_word<B>(base, Wp, part, w, s);
              }
            }
            __syncwarp();
          }
          if (lane == 0) S.events[c] += 1;
        }
      }
      __syncthreads();
    }
  }
  (void)ev_local;
  if (tid == 0) {
    S.rng[0] = rng.s0;
    S.rng[1] = rng.s1;
    S.rng[2] = rng.s2;
    S.rng[3] = rng.s3;
  }
}

// The same parallel replay over the whole GPU (cooperative launch, one CTA
// per SM): per fed bank, (a) every warp of the grid evaluates clauses for the
// vote, (b) one warp scans the gates (the only owner of the stream, which
// also draws the negative class first, trainer.cpp:159-165), (c) every warp
// of the grid applies gated clauses — three grid barriers per feed. Buffers
// alternate between two slots (feed, or example for regression); the scan
// zeroes the slot not in use.
template <int B>
__global__ void __launch_bounds__(kSeqThreads) train_sequential_grid_kernel(TrainParams P, SeqParams S) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint32_t smem[];
  const int L = 2 * P.o;
  const int refw = (L + 31) / 32 + 2;
  uint32_t* jc = smem;
  uint32_t* jl = jc + kGf2TabWords;
  uint32_t* wbuf = jl + kGf2TabWords;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int n = P.n, Wp = P.Wp, nwords = (n + 31) / 32;
  const int gwarp = blockIdx.x * nwarps + warp, gwarps = gridDim.x * nwarps;
  const bool lead = blockIdx.x == 0 && warp == 0;  // owns the reference stream
  const size_t cstride = static_cast<size_t>(B) * 2 * Wp;
  Xoshiro rng{S.rng[0], S.rng[1], S.rng[2], S.rng[3]};
  for (int k = tid; k < kGf2TabWords; k += blockDim.x) {
    jc[k] = S.jump_chunk[k];
    jl[k] = S.jump_lits[k];
  }
  __syncthreads();
  const int feeds = P.regress ? 1 : 2;
  int slot = 0;
  for (int64_t t = 0; t < P.q; ++t) {
    const int64_t i = P.order[t];
    const int y = P.labels[i];
    const uint32_t* xr = P.xplane + i * 2 * Wp;
    const uint32_t* nr = P.nplane + i * 2 * Wp;
    for (int feed = 0; feed < feeds; ++feed, slot ^= 1) {
      const int c = P.regress ? 0 : (feed == 0 ? y : __ldcg(S.g_misc + 2));
      const int target = feed == 0 ? 1 : 0;
      uint32_t* outs = S.g_outs + static_cast<size_t>(slot) * nwords;
      int32_t* vote = S.g_misc + slot;
      TMG_SEQ_CLOCK(c0);
      // (a) vote pass (trainer.cpp:62-68)
      for (int j = gwarp; j < n; j += gwarps) {
        const uint32_t* top = P.state + (static_cast<size_t>(c) * n + j) * cstride + static_cast<size_t>(B - 1) * 2 * Wp;
        uint32_t viol = 0, any = 0;
        for (int w = lane; w < Wp; w += 32) {
          // planes another SM may have updated: read through L2
          const uint32_t ix = __ldcg(top + w), in = __ldcg(top + Wp + w);
          viol |= (ix & ~xr[w]) | (in & ~nr[w]);
          any |= ix | in;
        }
        const unsigned vb = __ballot_sync(kFull, viol != 0), ab = __ballot_sync(kFull, any != 0);
        const int out = ab == 0 ? 1 : (vb == 0 ? 1 : 0);
        if (lane == 0 && out) {
          atomicOr(&outs[j >> 5], 1u << (j & 31));
          atomicAdd(vote, (!P.all_positive && (j & 1)) ? -1 : 1);
        }
      }
      grid.sync();
      TMG_SEQ_CLOCK(c1);
      // (b) gate scan
      if (lead) {
        if (feed == 0 && !P.regress && lane == 0) {
          int neg;
          if (P.m == 2) {
            neg = 1 - y;
          } else {
            neg = static_cast<int>(below_dev(rng, static_cast<uint32_t>(P.m - 1)));
            if (neg >= y) ++neg;
          }
          S.g_misc[2] = neg;
        }
        bool rt1;
        const double p = bank_gate(P, __ldcg(vote), y, target, rt1);
        const unsigned long long g = scan_bank(P, S, rng, p, target, rt1, jl, S.g_gbits, lane);
        if (lane == 0) S.events[c] += g;
        uint32_t* other = S.g_outs + static_cast<size_t>(slot ^ 1) * nwords;
        for (int k = lane; k < nwords; k += 32) other[k] = 0;
        if (lane == 0) S.g_misc[slot ^ 1] = 0;
      }
      TMG_SEQ_CLOCK(c2);
      grid.sync();
      TMG_SEQ_CLOCK(c3);
      // (c) apply the gated clauses
      if (warp < S.par_warps) {
        bool rt1;
        (void)bank_gate(P, __ldcg(vote), y, target, rt1);
        uint32_t* hb = wbuf + static_cast<size_t>(warp) * 2 * refw;
        for (int j = blockIdx.x * S.par_warps + warp; j < n; j += gridDim.x * S.par_warps) {
          if (!((__ldcg(S.g_gbits + (j >> 5)) >> (j & 31)) & 1u)) continue;
          apply_gated<B>(P, S, c, j, (__ldcg(outs + (j >> 5)) >> (j & 31)) & 1, is_type2(P, j, target, rt1), xr, nr,
                         jc, hb, hb + refw, refw, lane);
        }
      }
      grid.sync();
#ifdef TMG_STATS
      if (lead) {
        TMG_SEQ_ADD(200, c1 - c0);
        TMG_SEQ_ADD(201, c2 - c1);
        TMG_SEQ_ADD(202, c3 - c2);
        TMG_SEQ_ADD(203, clock64() - c3);
      }
#endif
    }
  }
  if (lead && lane == 0) {
    S.rng[0] = rng.s0;
    S.rng[1] = rng.s1;
    S.rng[2] = rng.s2;
    S.rng[3] = rng.s3;
  }
}

}  // namespace

bool train_sequential_launch(const TrainParams& p, const SeqParams& sp_in, int B, cudaStream_t s) {
  const int refw = (2 * p.o + 31) / 32 + 2;
  const size_t nwords = (p.n + 31) / 32;
  SeqParams sp = sp_in;
  size_t words = 2 * refw + nwords;
  if (sp.jump_chunk) {  // parallel replay: as many applying warps as shared memory holds draw buffers for
    const size_t fixed = words + 2 * kGf2TabWords + nwords;
    const size_t budget = 220 * 1024 / sizeof(uint32_t);  // of the 227 KB a CTA may opt into
    const long pw = fixed < budget ? static_cast<long>((budget - fixed) / (2 * refw)) : 0;
    sp.par_warps = static_cast<int32_t>(std::min<long>(kSeqThreads / 32, pw));
    if (sp.par_warps < 1) {
      sp.jump_chunk = sp.jump_lits = nullptr;  // rows too wide for even one buffer: serial replay
    } else {
      words = fixed + static_cast<size_t>(sp.par_warps) * 2 * refw;
    }
  }
  const size_t shm = sizeof(uint32_t) * words;
  if (sp.jump_chunk && sp.g_outs) {  // grid-wide replay: one CTA per SM, as many as there are clauses for
    const size_t gshm = sizeof(uint32_t) * (2 * kGf2TabWords + static_cast<size_t>(sp.par_warps) * 2 * refw);
    auto grid_go = [&](auto kern) {
      if (gshm > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gshm));
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSeqThreads, gshm);
      const int want = std::max(1, (p.n + sp.par_warps - 1) / sp.par_warps);
      const int grid = std::max(1, std::min(sms * std::max(per_sm, 1), want));
      TrainParams pp = p;
      SeqParams ss = sp;
      void* args[] = {&pp, &ss};
      count_launch();
      return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), grid, kSeqThreads, args, gshm, s) ==
             cudaSuccess;
    };
    bool ok = false;
    switch (B) {
      case 4: ok = grid_go(train_sequential_grid_kernel<4>); break;
      case 8: ok = grid_go(train_sequential_grid_kernel<8>); break;
      case 15: ok = grid_go(train_sequential_grid_kernel<15>); break;
      default: return false;
    }
    if (ok) return true;
    cudaGetLastError();  // cooperative launch refused (e.g. the GPU is shared): one CTA instead
  }
  auto go = [&](auto kern) {
    if (shm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shm));
    count_launch();
    kern<<<1, kSeqThreads, shm, s>>>(p, sp);
  };
  switch (B) {
    case 4: go(train_sequential_kernel<4>); return true;
    case 8: go(train_sequential_kernel<8>); return true;
    case 15: go(train_sequential_kernel<15>); return true;
    default: return false;
  }
}

}  // namespace tmg
