// train_smem.cu — Algorithm 1 for wide literal rows (IMDb-shaped, 2o above
// 8192 literals): the same per-warp clause pass as train_async_kernel
// (train.cu), but the clause's automaton planes live in shared memory
// (B x 2 x Wp words per warp, 20 KB at IMDb) instead of registers, and the
// feedback walks the clause one 32-literal word pair per lane at a time, so
// register use does not grow with the feature count.
//
// NW > 0: the step's literal row is held in registers (6..16 words per lane,
// up to 16 384 features). NW == 0: any width — the row stays in global
// memory (L1-cached) and is read where it is used, and a CTA holds one or two
// clauses depending on what fits in shared memory.
#include <algorithm>
#include <cstdlib>

#include "clause.cuh"
#include "kernels.h"
#include "tm_device.cuh"

#ifndef TMG_SMEM_UNROLL
#define TMG_SMEM_UNROLL 5  // word pairs of a Type I feedback processed together (ILP at low occupancy; IMDb: 1 / 2 / 4 / 5 / 10 -> 214 / 203 / 200 / 198.5 / 284 ms)
#endif

namespace tmg {

namespace {

#ifndef TMG_STEP_SAT_SMEM
#define TMG_STEP_SAT_SMEM 1  // clause-output-1 Type I as one up/down pass (tm_device.cuh type_i_planes)
#endif

#ifndef TMG_SMEM_MAXCPB
#define TMG_SMEM_MAXCPB 2  // most clauses (warps) per CTA; the launcher picks the count with the most warps per SM
#endif

constexpr int kSmemUnroll = TMG_SMEM_UNROLL;
constexpr int kSmemMaxCpb = TMG_SMEM_MAXCPB;
#ifndef TMG_SMEM_PERSIST_MAX
#define TMG_SMEM_PERSIST_MAX 12  // most clause slots of the persistent CTA
#endif
constexpr int kSmemPersistMax = TMG_SMEM_PERSIST_MAX;
constexpr size_t kSmemMax = 227 * 1024;  // opt-in shared memory per CTA on sm_100

// One clause's automaton planes in shared memory (or, INPLACE, in HBM with
// the global [plane][part][Wp] layout). The shared-memory copy (QUAD) keeps,
// per part, the planes below the top one in 16-byte quads
// ([quad][Wp] of uint4: one LDS.128 / STS.128 reads or writes 4 planes of a
// word; lanes hold consecutive words, so a warp's access is 512 contiguous
// bytes, conflict-free), the 1-3 planes left over as single-plane arrays, and
// the top plane (the include mask, read by every evaluation) as its own
// conflict-free array: B = 8 takes 5 accesses per word instead of 8, B = 15
// takes 6 instead of 15, with no padding.
template <int B, bool QUAD = false>
struct SmemPlanes {
  static constexpr int KQ = QUAD ? (B - 1) / 4 : 0;  // full quads below the top plane
  uint32_t* s;  // this warp's planes
  int Wp;
  __host__ __device__ static size_t index(int b, int part, int w, int Wp) {
    if (!QUAD) return (static_cast<size_t>(b) * 2 + part) * Wp + w;
    const size_t base = static_cast<size_t>(part) * B * Wp;
    if (b < 4 * KQ) return base + (static_cast<size_t>(b / 4) * Wp + w) * 4 + b % 4;
    return base + static_cast<size_t>(b) * Wp + w;  // leftover planes, then the top plane at b = B - 1
  }
  __device__ __forceinline__ void get(int part, int w, Planes<B>& out) const {
    if constexpr (QUAD) {
      const uint32_t* base = s + static_cast<size_t>(part) * B * Wp;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const uint4 v = reinterpret_cast<const uint4*>(base)[static_cast<size_t>(q) * Wp + w];
        out.p[4 * q] = v.x;
        out.p[4 * q + 1] = v.y;
        out.p[4 * q + 2] = v.z;
        out.p[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int b = 4 * KQ; b < B; ++b) out.p[b] = base[static_cast<size_t>(b) * Wp + w];
    } else {
#pragma unroll
      for (int b = 0; b < B; ++b) out.p[b] = s[(b * 2 + part) * Wp + w];
    }
  }
  __device__ __forceinline__ void put(int part, int w, const Planes<B>& in) {
    if constexpr (QUAD) {
      uint32_t* base = s + static_cast<size_t>(part) * B * Wp;
#pragma unroll
      for (int q = 0; q < KQ; ++q)
        reinterpret_cast<uint4*>(base)[static_cast<size_t>(q) * Wp + w] =
            make_uint4(in.p[4 * q], in.p[4 * q + 1], in.p[4 * q + 2], in.p[4 * q + 3]);
#pragma unroll
      for (int b = 4 * KQ; b < B; ++b) base[static_cast<size_t>(b) * Wp + w] = in.p[b];
    } else {
#pragma unroll
      for (int b = 0; b < B; ++b) s[(b * 2 + part) * Wp + w] = in.p[b];
    }
  }
  __device__ __forceinline__ uint32_t top(int part, int w) const { return s[index(B - 1, part, w, Wp)]; }
};

// A step's literal row as seen by one lane: words p*32 + lane of the x- and
// !x-planes, p < words(). Held in registers for a compile-time width.
// With TMG_ROW_X_ONLY the !x words are taken as ~x (train.cu fetch: bits
// past o differ from the stored plane, and every use masks them out).
template <int NW>
struct LitRow {
#if TMG_ROW_X_ONLY
  uint32_t xw[NW];
  __device__ __forceinline__ void load(const uint32_t* rp, int) {
#pragma unroll
    for (int p = 0; p < NW; ++p) xw[p] = __ldg(rp + p * 32);
  }
  __device__ __forceinline__ uint32_t n(int p) const { return ~xw[p]; }
#else
  uint32_t xw[NW], nw_[NW];
  __device__ __forceinline__ void load(const uint32_t* rp, int Wp) {
#pragma unroll
    for (int p = 0; p < NW; ++p) {
      xw[p] = __ldg(rp + p * 32);
      nw_[p] = __ldg(rp + Wp + p * 32);
    }
  }
  __device__ __forceinline__ uint32_t n(int p) const { return nw_[p]; }
#endif
  __device__ __forceinline__ uint32_t x(int p) const { return xw[p]; }
  __device__ __forceinline__ int words() const { return NW; }
};

// Runtime width: the row stays in global memory and is read on use.
template <>
struct LitRow<0> {
  const uint32_t* rp;
  int Wp;
  __device__ __forceinline__ void load(const uint32_t* r, int w) {
    rp = r;
    Wp = w;
  }
  __device__ __forceinline__ uint32_t x(int p) const { return __ldg(rp + p * 32); }
#if TMG_ROW_X_ONLY
  __device__ __forceinline__ uint32_t n(int p) const { return ~__ldg(rp + p * 32); }
#else
  __device__ __forceinline__ uint32_t n(int p) const { return __ldg(rp + Wp + p * 32); }
#endif
  __device__ __forceinline__ int words() const { return Wp >> 5; }
};

template <int NW, typename SP>
__device__ __forceinline__ int eval_train_smem(const SP& S, const LitRow<NW>& r, int lane) {
  uint32_t viol = 0, any = 0;
#pragma unroll
  for (int p = 0; p < r.words(); ++p) {
    const int w = p * 32 + lane;
    const uint32_t ix = S.top(0, w), in = S.top(1, w);
    viol |= (ix & ~r.x(p)) | (in & ~r.n(p));
    any |= ix | in;
  }
  const unsigned vb = __ballot_sync(kFull, viol != 0), ab = __ballot_sync(kFull, any != 0);
  return ab == 0 ? 1 : (vb == 0 ? 1 : 0);
}

__device__ __forceinline__ uint32_t valid_of(int w, int o) {
  const int first = w * 32;
  return first >= o ? 0u : (o - first >= 32 ? kFull : ((1u << (o - first)) - 1u));
}

// Type I (feedback.cpp:32-70) on a shared-memory clause, one word pair per
// lane at a time, with the register kernel's draws (clause.cuh type_i_async):
// alias patterns from Philox counters (clause, example, 2*word + part, 0),
// or the bit-serial sampler when p_high != 1 - p_low.
template <int NW, int B, bool P2, int OUT, typename SP>
__device__ __forceinline__ void type_i_smem_out(SP& S, const LitRow<NW>& r, const TrainParams& P,
                                                uint32_t g, uint32_t i32, int lane, AliasRef aref) {
  constexpr int before = OUT;
#pragma unroll kSmemUnroll
  for (int p = 0; p < r.words(); ++p) {
    const int w = p * 32 + lane;
    const uint32_t vm = valid_of(w, P.o);
    const uint32_t need[2] = {vm, vm};
    const uint32_t sel[2] = {r.x(p), r.n(p)};
    uint32_t bern[2];
    auto gen = [&](int slot, int blk) {
      const uint32_t wid = slot < 2 ? static_cast<uint32_t>(w * 2 + slot)
                                    : (0xFFFF0000u | static_cast<uint32_t>(p * 32 + lane));
      return philox4x32(U4{g, i32, wid, static_cast<uint32_t>(blk)}, P.rkey);
    };
    if (before && !P.alias_sel) {
      bernoulli_words<2, true>(need, sel, P.bern, bern, gen);
    } else {
      alias_words<2, false, kSmemAliasCopies>(need, aref, bern, gen);
      if (before) {
        bern[0] = (bern[0] ^ sel[0]) & need[0];
        bern[1] = (bern[1] ^ sel[1]) & need[1];
      }
    }
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      Planes<B> pl;
      S.get(part, w, pl);
      type_i_planes<B, P2, TMG_STEP_SAT_SMEM != 0, true>(pl, sel[part], before, P.boost, bern[part], vm, P.lo, P.hi);
      S.put(part, w, pl);
    }
  }
  __syncwarp();
}

// The clause output is warp-uniform: one branch, each arm with a constant one.
template <int NW, int B, bool P2, typename SP>
__device__ __forceinline__ void type_i_smem(SP& S, const LitRow<NW>& r, int before, const TrainParams& P,
                                            uint32_t g, uint32_t i32, int lane, AliasRef aref) {
  if (before)
    type_i_smem_out<NW, B, P2, 1>(S, r, P, g, i32, lane, aref);
  else
    type_i_smem_out<NW, B, P2, 0>(S, r, P, g, i32, lane, aref);
}

// One clause of the shared-memory path, run by one warp: clause-order index
// w (G: clause_of_warp's block size), its planes copied into `slot` (or
// updated in place at `st` when INPLACE), every window of its pass, the
// planes written back, its include count and events published.
template <int NW, int B, bool P2, bool INPLACE>
__device__ __forceinline__ void smem_clause(const TrainParams& P, uint32_t* slot, int w, int G, AliasRef aref,
                                            int lane) {
  using SP = SmemPlanes<B, !INPLACE>;  // shared-memory copies use the quad layout
  const int Wp = P.Wp;
  const size_t words = static_cast<size_t>(B) * 2 * Wp;  // per clause, either layout
  const int lc = clause_of_warp(P, w, G);
  const int c = lc / P.n_loc;
  const int j = P.j_begin + lc % P.n_loc;
  const uint32_t g = static_cast<uint32_t>(c) * P.n + j;
  const bool positive = P.all_positive || (j & 1) == 0;
  uint32_t* st = P.state + static_cast<size_t>(lc) * words;
  SP S{INPLACE ? st : slot, Wp};
  if (!INPLACE)
    for (size_t k = lane; k < words; k += 32) {
      const int b = static_cast<int>(k / (2 * Wp)), part = static_cast<int>((k / Wp) & 1), w = static_cast<int>(k % Wp);
      S.s[SP::index(b, part, w, Wp)] = st[k];
    }
  __syncwarp();
  uint32_t* prev_row = P.prev + static_cast<size_t>(lc) * P.Wq;
  const int64_t offset = clause_offset_dev(g, P.q);
  unsigned long long events = 0, events_type1 = 0;

  for (int64_t t0 = P.t_begin; t0 < P.t_end; t0 += 32) {
    const int64_t t = t0 + lane;
    int64_t i = 0;
    int target = 0;
    const bool gated = t < P.t_end && gate_step(P, c, positive, g, offset, t, i, target);
    unsigned gm = __ballot_sync(kFull, gated);
    if (!gm) continue;
    events += __popc(gm);
    events_type1 += __popc(__ballot_sync(kFull, gated && target));
    // Lane-owned bookkeeping, published after the window (see train.cu).
    uint32_t prevbit = 0;
    if (gated) prevbit = (__ldcg(prev_row + (i >> 5)) >> (i & 31)) & 1u;
    const int code = target ? ~static_cast<int>(i) : static_cast<int>(i);
    unsigned outs = 0;
    while (gm) {
      const int sl = __ffs(gm) - 1;
      gm &= gm - 1;
      const int cd = __shfl_sync(kFull, code, sl);
      const int64_t is = cd < 0 ? ~cd : cd;
      LitRow<NW> r;
      r.load(P.xplane + is * 2 * Wp + lane, Wp);
      const int before = eval_train_smem<NW>(S, r, lane);
      int after = before;
      if (cd >= 0) {  // Type II (feedback.cpp:72-83)
        if (before) {
          uint32_t moved = 0;
#pragma unroll
          for (int p = 0; p < r.words(); ++p) {
            const int w = p * 32 + lane;
            const uint32_t vm = valid_of(w, P.o);
#pragma unroll
            for (int part = 0; part < 2; ++part) {
              const uint32_t inc = ~(part ? r.n(p) : r.x(p)) & ~S.top(part, w) & vm;
              if (inc) {
                Planes<B> pl;
                S.get(part, w, pl);
                add_one<B>(pl, inc);
                S.put(part, w, pl);
              }
              moved |= inc;
            }
          }
          __syncwarp();
          if (__any_sync(kFull, moved != 0)) after = eval_train_smem<NW>(S, r, lane);
        }
      } else {  // Type I (feedback.cpp:32-70), one word pair at a time
        type_i_smem<NW, B, P2>(S, r, before, P, g, static_cast<uint32_t>(is), lane, aref);
        after = eval_train_smem<NW>(S, r, lane);
      }
      outs |= static_cast<unsigned>(after) << sl;
    }
    if (gated && ((outs >> lane) & 1u) != prevbit) {  // pool.cpp:93-106
      red_xor_gpu(prev_row + (i >> 5), 1u << (i & 31));
      int delta = prevbit ? -1 : 1;
      if (!positive) delta = -delta;
      const size_t ti = static_cast<size_t>(i) * P.m + c;
      publish_tally(P, ti, delta);  // local replica (+ window deltas, + peers over NVLink)
    }
  }
  __syncwarp();
  int cnt = 0;
  for (size_t k = lane; k < words; k += 32) {
    const int b = static_cast<int>(k / (2 * Wp)), part = static_cast<int>((k / Wp) & 1), w = static_cast<int>(k % Wp);
    const uint32_t v = S.s[SP::index(b, part, w, Wp)];
    if (!INPLACE) st[k] = v;
    if (b == B - 1) cnt += __popc(v);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  if (P.npeers) __threadfence_system();  // remote tally adds performed before the kernel retires
  if (lane == 0) {
    P.inc_count[lc] = cnt;
    atomicAdd(P.events + c, events);
    atomicAdd(P.events + P.m + c, events_type1);
  }
}


// One warp per clause, blockDim.x / 32 clauses per CTA; dynamic shared memory
// = the clauses' planes, then kSmemAliasCopies copies of the alias table.
// INPLACE (rows whose planes exceed shared memory, beyond ~107k features at
// 8 planes): one clause per CTA, the planes stay in HBM/L2 and are updated in
// place (every word is lane-owned), shared memory holds the alias table only.
template <int NW, int B, bool P2, bool INPLACE = false>
__global__ void __launch_bounds__(32 * kSmemMaxCpb) train_async_smem_kernel(TrainParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int cpb = blockDim.x >> 5;
  const size_t words = static_cast<size_t>(B) * 2 * P.Wp;
  uint32_t* atab = INPLACE ? smem : smem + cpb * words;
  fill_alias_packed(atab, P.alias8, threadIdx.x, blockDim.x);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const AliasRef aref = lane_alias<kSmemAliasCopies>(atab, lane);
  const int wib = threadIdx.x >> 5;
  const int w = P.w_begin + blockIdx.x * cpb + wib;
  if (w >= P.w_end) return;
  smem_clause<NW, B, P2, INPLACE>(P, smem + wib * words, w, cpb, aref, lane);
}

// Persistent form: one CTA per SM with as many clause slots (warps) as shared
// memory holds next to ONE alias table; each warp pulls the next clause-order
// index from P.work until the range is done, so a slow clause never holds a
// whole CTA's shared memory idle (the launched form frees a CTA's slots only
// when its last clause ends). Same clause order (G = kSmemOrderG).
constexpr int kSmemOrderG = 2;
template <int NW, int B, bool P2>
__global__ void __launch_bounds__(32 * kSmemPersistMax, 1) train_async_smem_persistent_kernel(TrainParams P) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int slots = blockDim.x >> 5;
  const size_t words = static_cast<size_t>(B) * 2 * P.Wp;
  uint32_t* atab = smem + slots * words;
  fill_alias_packed(atab, P.alias8, threadIdx.x, blockDim.x);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const AliasRef aref = lane_alias<kSmemAliasCopies>(atab, lane);
  uint32_t* slot = smem + (threadIdx.x >> 5) * words;
  const int total = P.w_end - P.w_begin;
  while (true) {
    int k = 0;
    if (lane == 0) k = atomicAdd(P.work, 1);
    k = __shfl_sync(kFull, k, 0);
    if (k >= total) break;
    smem_clause<NW, B, P2, false>(P, slot, P.w_begin + k, kSmemOrderG, aref, lane);
    __syncwarp();
  }
}

// The persistent kernel's plan: clause slots per CTA (as many as shared
// memory holds beside one alias table, <= kSmemPersistMax) and resident CTAs
// per SM; returns the resident clause warps per SM (0: not applicable).
// TMG_SMEM_PERSIST=0 disables it (A/B checks).
template <int NW, int B, bool P2>
int persistent_plan(const TrainParams& p, int* slots_out, int* ctas_out) {
  const char* e = std::getenv("TMG_SMEM_PERSIST");
  if ((e && e[0] == '0') || p.work == nullptr) return 0;
  const size_t per = sizeof(uint32_t) * static_cast<size_t>(B) * 2 * p.Wp;
  const size_t atab = sizeof(uint32_t) * kAliasWordsPacked;
  if (per + atab > kSmemMax) return 0;
  const int slots = static_cast<int>(std::min<size_t>(kSmemPersistMax, (kSmemMax - atab) / per));
  const size_t shm = slots * per + atab;
  auto kern = train_async_smem_persistent_kernel<NW, B, P2>;
  if (shm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shm));
  int ctas = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, kern, 32 * slots, shm);
  *slots_out = slots;
  *ctas_out = ctas;
  return ctas * slots;
}

size_t smem_bytes(int B, int Wp, int cpb) {
  return sizeof(uint32_t) * (static_cast<size_t>(cpb) * B * 2 * Wp + kAliasWordsPacked);
}

// Clauses per CTA: the count (<= kSmemMaxCpb) with the most resident warps
// per SM (every CTA carries its own alias table); returns those warps per SM
// (0: no count fits in shared memory — planes in place).
template <int NW, int B, bool P2>
int smem_plan(const TrainParams& p, int* cpb_out) {
  int cpb = 1, best = 0;
  for (int c = 1; c <= kSmemMaxCpb; ++c) {
    const size_t b = smem_bytes(B, p.Wp, c);
    if (b > kSmemMax) break;
    if (b > 48 * 1024)
      cudaFuncSetAttribute(train_async_smem_kernel<NW, B, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(b));
    int ctas = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, train_async_smem_kernel<NW, B, P2>, 32 * c, b);
    if (ctas * c > best) {
      best = ctas * c;
      cpb = c;
    }
  }
  int slots = 0, pctas = 0;
  const int pw = persistent_plan<NW, B, P2>(p, &slots, &pctas);
  if (pw > best && pctas > 0) {
    *cpb_out = slots;
    return pw;
  }
  *cpb_out = cpb;
  return best;
}

template <int NW, int B, bool P2>
bool launch_smem_p2(const TrainParams& p, cudaStream_t s, int* blocks) {
  // Clauses per CTA: the count (<= kSmemMaxCpb) with the most resident warps
  // per SM (every CTA carries its own alias table); none fits: planes in place.
  int cpb = 1, best = 0;
  for (int c = 1; c <= kSmemMaxCpb; ++c) {
    const size_t b = smem_bytes(B, p.Wp, c);
    if (b > kSmemMax) break;
    if (b > 48 * 1024)
      cudaFuncSetAttribute(train_async_smem_kernel<NW, B, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(b));
    int ctas = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, train_async_smem_kernel<NW, B, P2>, 32 * c, b);
    if (ctas * c > best) {
      best = ctas * c;
      cpb = c;
    }
  }
  const size_t shm = smem_bytes(B, p.Wp, cpb);
  const int clauses = p.w_end - p.w_begin;
  if (shm > kSmemMax) {
    if constexpr (NW != 0) {
      return false;
    } else {
      if (blocks) *blocks = clauses;
      const size_t ashm = sizeof(uint32_t) * kAliasWordsPacked;
      count_launch();
      train_async_smem_kernel<0, B, P2, true><<<clauses, 32, ashm, s>>>(p);
      return true;
    }
  }
  int slots = 0, pctas = 0;
  if (persistent_plan<NW, B, P2>(p, &slots, &pctas) > best && pctas > 0) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pgrid = std::max(1, std::min(sms * pctas, (clauses + slots - 1) / slots));
    if (blocks) *blocks = pgrid;
    if (cudaMemsetAsync(p.work, 0, sizeof(int32_t), s) != cudaSuccess) return false;
    const size_t pshm = sizeof(uint32_t) * (static_cast<size_t>(slots) * B * 2 * p.Wp + kAliasWordsPacked);
    count_launch();
    train_async_smem_persistent_kernel<NW, B, P2><<<pgrid, 32 * slots, pshm, s>>>(p);
    return true;
  }
  const int grid = (clauses + cpb - 1) / cpb;
  if (blocks) *blocks = grid;
  if (shm > 48 * 1024)
    cudaFuncSetAttribute(train_async_smem_kernel<NW, B, P2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(shm));
  count_launch();
  train_async_smem_kernel<NW, B, P2><<<grid, 32 * cpb, shm, s>>>(p);
  return true;
}

template <int NW, int B>
bool launch_smem(const TrainParams& p, cudaStream_t s, int* blocks) {
  if (p.lo == 0 && p.hi == (1u << B) - 1u) return launch_smem_p2<NW, B, true>(p, s, blocks);
  return launch_smem_p2<NW, B, false>(p, s, blocks);
}

// One Type I feedback of the shared-memory path on the clause planes at
// `state` (global), literal row 0 of P: the wide-row counterpart of
// train.cu type_i_async_once_kernel for the async sampler's parity test.
template <int NW, int B, bool P2>
__global__ void __launch_bounds__(32) type_i_smem_once_kernel(TrainParams P, uint32_t* state, uint32_t g,
                                                              uint32_t i, int out) {
  extern __shared__ __align__(16) uint32_t smem[];
  using SP = SmemPlanes<B, true>;
  const int lane = threadIdx.x;
  const int Wp = P.Wp;
  const size_t words = static_cast<size_t>(B) * 2 * Wp;
  uint32_t* atab = smem + words;
  fill_alias_packed(atab, P.alias8, lane, 32);
  auto at = [&](size_t k) {
    return SP::index(static_cast<int>(k / (2 * Wp)), static_cast<int>((k / Wp) & 1), static_cast<int>(k % Wp), Wp);
  };
  for (size_t k = lane; k < words; k += 32) smem[at(k)] = state[k];
  __syncwarp();
  SP S{smem, Wp};
  LitRow<NW> r;
  r.load(P.xplane + lane, Wp);
  type_i_smem<NW, B, P2>(S, r, out, P, g, i, lane, lane_alias<kSmemAliasCopies>(atab, lane));
  __syncwarp();
  for (size_t k = lane; k < words; k += 32) state[k] = smem[at(k)];
}

// Row widths (words per lane) with a register-held literal row.
bool compiled_width(int NW) { return NW == 6 || NW == 8 || NW == 10 || NW == 12 || NW == 16; }

}  // namespace

bool type_i_smem_once_launch(const TrainParams& p, uint32_t* state, uint32_t g, uint32_t i, int out, int B, int NW,
                             cudaStream_t s) {
  const bool p2 = p.lo == 0 && p.hi == (1u << B) - 1u;
  const size_t shm = smem_bytes(B, p.Wp, 1);
  if (shm > kSmemMax) return false;
  auto go = [&](auto kern) {
    if (shm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(shm));
    count_launch();
    kern<<<1, 32, shm, s>>>(p, state, g, i, out);
    return true;
  };
#define TMG_SONCE(nw, b)                                                           \
  if (NW == nw && B == b)                                                          \
    return p2 ? go(type_i_smem_once_kernel<nw, b, true>) : go(type_i_smem_once_kernel<nw, b, false>);
  TMG_SONCE(6, 4) TMG_SONCE(6, 8) TMG_SONCE(6, 15) TMG_SONCE(8, 4) TMG_SONCE(8, 8) TMG_SONCE(8, 15)
  TMG_SONCE(10, 4) TMG_SONCE(10, 8) TMG_SONCE(10, 15) TMG_SONCE(12, 4) TMG_SONCE(12, 8) TMG_SONCE(12, 15)
  TMG_SONCE(16, 4) TMG_SONCE(16, 8) TMG_SONCE(16, 15)
#undef TMG_SONCE
  if (!compiled_width(NW)) {
    if (B == 4) return p2 ? go(type_i_smem_once_kernel<0, 4, true>) : go(type_i_smem_once_kernel<0, 4, false>);
    if (B == 8) return p2 ? go(type_i_smem_once_kernel<0, 8, true>) : go(type_i_smem_once_kernel<0, 8, false>);
    if (B == 15) return p2 ? go(type_i_smem_once_kernel<0, 15, true>) : go(type_i_smem_once_kernel<0, 15, false>);
  }
  return false;
}

int train_async_smem_resident_warps(const TrainParams& p, int B, int NW, int* warps_per_cta) {
  const int nw = compiled_width(NW) ? NW : 0;
  const bool p2 = p.lo == 0 && p.hi == (1u << B) - 1u;
  int cpb = 1, per_sm = 0, dev = 0, sms = 0;
#define TMG_PLAN(nw_, b_)                                                                          \
  if (nw == nw_ && B == b_) per_sm = p2 ? smem_plan<nw_, b_, true>(p, &cpb) : smem_plan<nw_, b_, false>(p, &cpb);
#define TMG_PLAN_B(nw_) TMG_PLAN(nw_, 4) TMG_PLAN(nw_, 8) TMG_PLAN(nw_, 15)
  TMG_PLAN_B(6) TMG_PLAN_B(8) TMG_PLAN_B(10) TMG_PLAN_B(12) TMG_PLAN_B(16) TMG_PLAN_B(0)
#undef TMG_PLAN_B
#undef TMG_PLAN
  if (per_sm == 0) per_sm = 8, cpb = 1;  // in place: one clause per CTA
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  *warps_per_cta = cpb;
  return per_sm * sms;
}

bool train_async_smem_launch(const TrainParams& p, int B, int NW, cudaStream_t s, int* blocks) {
  const int nw = compiled_width(NW) ? NW : 0;
#define TMG_SMEM(nw_)                                        \
  if (nw == nw_) {                                           \
    if (B == 4) return launch_smem<nw_, 4>(p, s, blocks);    \
    if (B == 8) return launch_smem<nw_, 8>(p, s, blocks);    \
    if (B == 15) return launch_smem<nw_, 15>(p, s, blocks);  \
  }
  TMG_SMEM(6) TMG_SMEM(8) TMG_SMEM(10) TMG_SMEM(12) TMG_SMEM(16) TMG_SMEM(0)
#undef TMG_SMEM
  return false;
}

}  // namespace tmg
