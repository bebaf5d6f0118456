// train.cu — Algorithm 1 (decentralized clause updating) on sm_100a.
//
// One warp owns one clause for a whole pass over the example order and keeps
// its automaton states in registers as bit planes. Per step it reads the
// (deliberately stale) class tally, gates, applies Type I / Type II feedback,
// re-evaluates and publishes the output change to the tally with an atomic
// add — the reference's update_clause (proj/src/trainer.cpp:102-136) with
// record_output_and_tally (proj/src/pool.cpp:93-106).
//
//   train_async  : all clauses concurrently (the paper's GPU architecture),
//                  counter-based Philox keyed by (seed^epoch, clause, example,
//                  literal word). Gates of 32 consecutive steps are drawn in
//                  parallel, one per lane, then only the gated steps run.
//   train_mirror : one warp replays the reference's W-worker schedule with the
//                  reference xoshiro streams, bit-exact (sync mirror mode).
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "clause.cuh"
#include "kernels.h"
#include "tm_device.cuh"

namespace tmg {

namespace {

// Resident CTAs (4 warps each) per SM for one instantiation: as many as the
// register file allows for the clause planes (2*NW*B registers), the literal
// double buffer and the sampler's working set without spilling. NW=1, B=8
// (MNIST) gets 8 CTAs = 32 warps at 64 registers, the fastest in the r1m sweep.
#ifndef TMG_ASYNC_MINB
constexpr int async_regs(int NW, int B) { return 2 * NW * B + 40 + 8 * NW + (B == 8 ? 0 : (B == 4 ? 16 : 24)); }
constexpr int async_min_blocks(int NW, int B) {
  return 65536 / (128 * async_regs(NW, B)) < 1 ? 1 : 65536 / (128 * async_regs(NW, B));
}
// A packed last slot (ClausePk) frees one slot's planes: at 3 words per lane
// and 8 planes the kernel fits 102 registers without spilling (96 used), so
// 5 CTAs per SM instead of 4 (FMNIST 558 vs 577 ms; 6 CTAs spill: 597 ms).
// Other packed shapes keep the unpacked bound (not measured).
constexpr int async_min_blocks_pk(int NW, int B, bool PACK) {
  return PACK && NW == 3 && B == 8 ? 5 : async_min_blocks(NW, B);
}
#define TMG_ASYNC_BOUNDS __launch_bounds__(128, async_min_blocks_pk(NW, B, PACK))
#else
#define TMG_ASYNC_BOUNDS __launch_bounds__(128, TMG_ASYNC_MINB)
#endif
template <int NW, int B, bool P2, bool PACK = false>
__global__ void TMG_ASYNC_BOUNDS train_async_kernel(TrainParams P) {
  __shared__ uint32_t atab[TMG_ALIAS ? kAliasWords : 1];
  load_alias(P, atab);
  const int lane = static_cast<int>(lane_id());
  const AliasRef aref = lane_alias(atab, lane);
  const int w = P.w_begin + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w >= P.w_end) return;
  const int lc = clause_of_warp(P, w, blockDim.x >> 5);
  const int c = lc / P.n_loc;
  const int j = P.j_begin + lc % P.n_loc;
  const uint32_t g = static_cast<uint32_t>(c) * P.n + j;
  const bool positive = P.all_positive || (j & 1) == 0;

  std::conditional_t<PACK, ClausePk<NW, B, P2>, Clause<NW, B, P2>> cl;
  uint32_t* st = P.state + static_cast<size_t>(lc) * B * 2 * P.Wp;
  cl.load(st, P.Wp, lane, P.o);
  cl.refresh_nonempty();
  uint32_t* prev_row = P.prev + static_cast<size_t>(lc) * P.Wq;
  const int64_t offset = clause_offset_dev(g, P.q);
  unsigned long long events = 0, events_type1 = 0;

  for (int64_t t0 = P.t_begin; t0 < P.t_end; t0 += 32) {
    // ---- gates of 32 consecutive steps, one per lane (a legal interleaving
    // of the reference: other workers' tally adds in this window land later).
    const int64_t t = t0 + lane;
    int64_t i = 0;
    int target = 0;  // 1: the step would take Type I feedback, 0: Type II
    const bool gated = t < P.t_end && gate_step(P, c, positive, g, offset, t, i, target);
    unsigned gm = __ballot_sync(kFull, gated);
    if (!gm) continue;
    events += __popc(gm);

    // ---- gated steps in order. Each lane owns the bookkeeping of its own
    // step: it fetched the previous-output bit of its example above and
    // publishes the new output after the window (record_output_and_tally,
    // pool.cpp:93-106). Deferring the publish to the end of the 32 steps is a
    // legal interleaving: a clause visits each example once per pass, so no
    // step of this window reads a tally this window writes; other clauses'
    // reads were never ordered with respect to it. The step loop is unrolled
    // twice so the next step's literal words load into the idle buffer.
    uint32_t prevbit = 0;
    if (gated) prevbit = (__ldcg(prev_row + (i >> 5)) >> (i & 31)) & 1u;
    const int code = target ? ~static_cast<int>(i) : static_cast<int>(i);  // q < 2^31: sign = Type I
    unsigned outs = 0;  // bit l: output after the step lane l drew
    uint32_t xa[NW], na[NW], xb[NW], nb[NW];
    events_type1 += __popc(__ballot_sync(kFull, gated && target));
    auto fetch = [&](uint32_t (&xs)[NW], uint32_t (&ns)[NW], int& cd, uint32_t& sl) {
      const int l = __ffs(gm) - 1;
      sl = gm & (0u - gm);  // this step's lane bit
      gm ^= sl;
      cd = __shfl_sync(kFull, code, l);
      // Literal rows are [x words | !x words] (2 * Wp words, nplane = xplane
      // + Wp): one address, both planes at compile-time offsets.
      const uint32_t* rp = P.xplane + static_cast<size_t>(cd < 0 ? ~cd : cd) * (64 * NW);
#pragma unroll
      for (int p = 0; p < NW; ++p) {
        xs[p] = __ldg(rp + cl.word_of(p, lane));
        // !x words as ~x (TMG_ROW_X_ONLY, rows of >= TMG_ROW_X_MIN_NW words
        // per lane): the bits past o differ from the stored !x plane (0
        // there) but every use is masked by the valid bits or meets an
        // include bit, which is never set past o.
        if constexpr (PACK || (TMG_ROW_X_ONLY && NW >= TMG_ROW_X_MIN_NW)) ns[p] = ~xs[p];
        else ns[p] = __ldg(rp + 32 * NW + p * 32 + lane);
      }
    };
    auto run = [&](const uint32_t (&xs)[NW], const uint32_t (&ns)[NW], int cd, uint32_t sl) {
      const int before = cl.eval_cached(xs, ns);
      int after = before;
      if (cd >= 0) {
        if (before && cl.type_ii(xs, ns)) after = cl.eval_train(xs, ns);
      } else {
        type_i_async<NW, B, P2>(cl, xs, ns, before, P, g, static_cast<uint32_t>(~cd), lane, aref);
        after = cl.eval_train(xs, ns);
      }
      outs = mad_u32(sl, static_cast<uint32_t>(after), outs);  // disjoint bits: OR as an FMA-pipe add
    };
    int cda, cdb;
    uint32_t sla, slb;
    if (NW <= TMG_ASYNC_UNROLL_NW) {
      // Two copies of the step body, no register moves between buffers.
      fetch(xa, na, cda, sla);
      while (true) {
        const bool more_b = gm != 0;
        if (more_b) fetch(xb, nb, cdb, slb);
        run(xa, na, cda, sla);
        if (!more_b) break;
        const bool more_a = gm != 0;
        if (more_a) fetch(xa, na, cda, sla);
        run(xb, nb, cdb, slb);
        if (!more_a) break;
      }
    } else {
      // Wide rows: one copy of the (large) step body keeps the kernel inside
      // the instruction cache; the row of the step is loaded at its start.
      while (gm) {
        fetch(xa, na, cda, sla);
        run(xa, na, cda, sla);
      }
    }
    if (gated && ((outs >> lane) & 1u) != prevbit) {
      red_xor_gpu(prev_row + (i >> 5), 1u << (i & 31));
      int delta = prevbit ? -1 : 1;
      if (!positive) delta = -delta;
      const size_t ti = static_cast<size_t>(i) * P.m + c;
      publish_tally(P, ti, delta);  // local replica (+ window deltas, + peers over NVLink)
    }
  }
  cl.store(st, P.Wp, lane);
  const int cnt = cl.include_count();
  if (P.npeers) __threadfence_system();  // remote tally adds performed before the kernel retires
  if (lane == 0) {
    P.inc_count[lc] = cnt;
    atomicAdd(P.events + c, events);
    atomicAdd(P.events + P.m + c, events_type1);
  }
}

// -------------------------------------------------------------- mirror ---

// Single warp. Replays, job by job, update_clause (trainer.cpp:102-136) with
// the reference xoshiro streams: exactly one gate draw per step and 2o Type I
// draws in literal order k = 0..2o-1 (feedback.cpp:45,63).
template <int NW, int B>
__global__ void __launch_bounds__(32) train_mirror_kernel(TrainParams P, MirrorParams M) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x;
  const int L = 2 * P.o;
  const int refw = (L + 31) / 32 + 2;  // + padding for funnel shifts
  const int tabw = M.jump_chunk ? 2 * kGf2TabWords : 0;
  uint32_t* jc = smem;                 // jump tables (M.jump_chunk != null)
  uint32_t* jl = jc + kGf2TabWords;
  uint32_t* hbits = smem + tabw;       // u < p_high, reference literal order
  uint32_t* lbits = hbits + refw;      // u < p_low
  const int64_t q = P.q;
  const int T = P.margin;
  for (int k = lane; k < 2 * refw; k += 32) hbits[k] = 0;
  if (M.jump_chunk)
    for (int k = lane; k < kGf2TabWords; k += 32) {
      jc[k] = M.jump_chunk[k];
      jl[k] = M.jump_lits[k];
    }
  __syncwarp();

  for (int jb = 0; jb < M.njobs; ++jb) {
    const MirrorJob job = M.jobs[jb];
    const int c = job.c;
    const int lc = c * P.n_loc + (job.j - P.j_begin);
    const bool positive = P.all_positive || (job.j & 1) == 0;
    Xoshiro rng;
    uint64_t* rs = M.rng + 4 * job.worker;
    rng.s0 = rs[0];
    rng.s1 = rs[1];
    rng.s2 = rs[2];
    rng.s3 = rs[3];
    Clause<NW, B> cl;
    uint32_t* st = P.state + static_cast<size_t>(lc) * B * 2 * P.Wp;
    cl.load(st, P.Wp, lane, P.o);
    uint32_t* prev_row = P.prev + static_cast<size_t>(lc) * P.Wq;
    unsigned long long events = 0;

    const bool forced = job.forced != 0;
    // Type I feedback of one step (feedback.cpp:32-70) with the 2o draws of
    // the stream in literal order.
    auto type_i = [&](const uint32_t (&x)[NW], const uint32_t (&n)[NW], int before) {
      if (M.jump_chunk) {
        draw_type_i_bits(rng, L, M.chunk, M.p_high, M.p_low, jc, jl, hbits, lbits, refw, lane);
      } else {
        if (lane == 0) {
          const uint64_t th = u53_below(M.p_high), tl = u53_below(M.p_low);
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
      }
#pragma unroll
      for (int p = 0; p < NW; ++p) {
        const int wi = p * 32 + lane;
        if (wi * 32 >= P.o) continue;
        // part 0: literal k = 32*wi + b; part 1: literal k = o + 32*wi + b.
        const int k1 = P.o + wi * 32;
        const uint32_t h0 = hbits[wi], l0 = lbits[wi];
        const uint32_t h1 = __funnelshift_r(hbits[k1 >> 5], hbits[(k1 >> 5) + 1], k1 & 31);
        const uint32_t l1 = __funnelshift_r(lbits[k1 >> 5], lbits[(k1 >> 5) + 1], k1 & 31);
        if (before) {
          // c=1: lit=1 uses the p_high draw, lit=0 the p_low draw.
          cl.type_i_word(0, p, x[p], 1, P.boost, (x[p] & h0) | (~x[p] & l0), P.lo, P.hi);
          cl.type_i_word(1, p, n[p], 1, P.boost, (n[p] & h1) | (~n[p] & l1), P.lo, P.hi);
        } else {
          cl.type_i_word(0, p, x[p], 0, P.boost, l0, P.lo, P.hi);
          cl.type_i_word(1, p, n[p], 0, P.boost, l1, P.lo, P.hi);
        }
      }
      __syncwarp();
    };
    if (!forced) {
      // Windows of 32 steps: the gate inputs (order, label, tally ->
      // probability and feedback type) and the previous-output bit of each
      // step's example are loaded by its own lane up front, and the new
      // outputs are published at the window end. Exact for the replay: a
      // pass visits each example once, so no step reads a tally or an output
      // bit an earlier step of the same pass writes. Only the stream is
      // serial: lane 0 draws each gate (trainer.cpp:121) and, on Type I, the
      // 2o draws.
      // A window never spans more than q steps: with batch > q (the
      // reference's (offset + t) % q wraps) an example would otherwise meet
      // two lanes of one window and both would see its stale tally and bit.
      const int64_t win = q < 32 ? q : 32;
      for (int64_t t0 = 0; t0 < job.batch; t0 += win) {
        const int64_t t = t0 + lane;
        const int steps = static_cast<int>(job.batch - t0 < win ? job.batch - t0 : win);
        int64_t i = 0;
        int target = 0;
        double p = 0.0;
        uint32_t prevbit = 0;
        if (lane < steps) {
          const int64_t pos = (job.offset + t) % q;
          i = P.order ? P.order[pos] : pos;
          const int v0 = __ldcg(P.tallies + i * P.m + c);
          const int label = P.labels[i];
          if (P.regress) {  // gate_probability, regression.cpp:46-48
            const int v = v0 < 0 ? 0 : (v0 > T ? T : v0);
            const int e = label > v ? label - v : v - label;
            p = fmin(1.0, static_cast<double>(e) / (2.0 * static_cast<double>(T)));
            target = v < label ? 1 : 0;
          } else {  // clause_update_probability, feedback.cpp:24-28
            const int y = label == c ? 1 : 0;
            const int v = v0 < -T ? -T : (v0 > T ? T : v0);
            const int e = y ? T - v : T + v;
            p = static_cast<double>(e) / (2.0 * static_cast<double>(T));
            target = (y == 1) == positive ? 1 : 0;
          }
          prevbit = (__ldcg(prev_row + (i >> 5)) >> (i & 31)) & 1u;
        }
        unsigned gm = 0, outs = 0;
        for (int sidx = 0; sidx < steps; ++sidx) {
          const double ps = __shfl_sync(kFull, p, sidx);
          int gated = 0;
          if (lane == 0) gated = next53(rng) < u53_below(ps) ? 1 : 0;  // skip iff u >= p (trainer.cpp:121)
          gated = __shfl_sync(kFull, gated, 0);
          if (!gated) continue;
          ++events;
          gm |= 1u << sidx;
          const int64_t is = __shfl_sync(kFull, i, sidx);
          const int ts = __shfl_sync(kFull, target, sidx);
          uint32_t x[NW], n[NW];
#pragma unroll
          for (int pw = 0; pw < NW; ++pw) {
            x[pw] = P.xplane[is * 2 * P.Wp + pw * 32 + lane];
            n[pw] = P.nplane[is * 2 * P.Wp + pw * 32 + lane];
          }
          const int before = cl.eval_train(x, n);
          int after = before;
          if (ts == 0) {
            if (before && cl.type_ii(x, n)) after = cl.eval_train(x, n);
          } else {
            type_i(x, n, before);
            after = cl.eval_train(x, n);
          }
          outs |= static_cast<unsigned>(after) << sidx;
        }
        if ((gm >> lane) & 1u) {  // record_output_and_tally (pool.cpp:93-106)
          const uint32_t now = (outs >> lane) & 1u;
          if (now != prevbit) {
            red_xor_gpu(prev_row + (i >> 5), 1u << (i & 31));
            int delta = now ? 1 : -1;
            if (!positive) delta = -delta;
            publish_tally(P, static_cast<size_t>(i) * P.m + c, delta);
          }
        }
        __syncwarp();
      }
    }
    for (int64_t t = 0; forced && t < job.batch; ++t) {
      int64_t i = 0;
      int target = 0, gated = 1;  // target: 1 = Type I step, 0 = Type II
      if (lane == 0 && !forced) {
        const int64_t pos = (job.offset + t) % q;
        i = P.order ? P.order[pos] : pos;
        const int v0 = P.tallies[i * P.m + c];
        const int label = P.labels[i];
        double p;
        if (P.regress) {  // gate_probability, regression.cpp:46-48
          const int v = v0 < 0 ? 0 : (v0 > T ? T : v0);
          const int e = label > v ? label - v : v - label;
          p = fmin(1.0, static_cast<double>(e) / (2.0 * static_cast<double>(T)));
          target = v < label ? 1 : 0;
        } else {  // clause_update_probability, feedback.cpp:24-28
          const int y = label == c ? 1 : 0;
          const int v = v0 < -T ? -T : (v0 > T ? T : v0);
          const int e = y ? T - v : T + v;
          p = static_cast<double>(e) / (2.0 * static_cast<double>(T));
          target = (y == 1) == positive ? 1 : 0;
        }
        gated = next53(rng) < u53_below(p) ? 1 : 0;  // skip iff u >= p (trainer.cpp:121)
      }
      gated = __shfl_sync(kFull, gated, 0);
      if (!gated) continue;
      ++events;
      i = __shfl_sync(kFull, i, 0);
      target = __shfl_sync(kFull, target, 0);
      uint32_t x[NW], n[NW];
#pragma unroll
      for (int p = 0; p < NW; ++p) {
        x[p] = P.xplane[i * 2 * P.Wp + p * 32 + lane];
        n[p] = P.nplane[i * 2 * P.Wp + p * 32 + lane];
      }
      const bool type2 = forced ? job.forced == 2 : target == 0;
      const int evald = cl.eval_train(x, n);
      const int before = (forced && job.out_override >= 0) ? job.out_override : evald;
      int after = evald;
      if (type2) {
        if (before && cl.type_ii(x, n)) after = cl.eval_train(x, n);
      } else {
        type_i(x, n, before);
        after = cl.eval_train(x, n);
      }
      if (lane == 0 && !forced) {
        const uint32_t pword = prev_row[i >> 5];
        record(P, prev_row, i, c, positive, pword, after);
      }
      __syncwarp();
    }
    cl.store(st, P.Wp, lane);
    const int cnt = cl.include_count();
    if (lane == 0) {
      P.inc_count[lc] = cnt;
      P.events[c] += events;
      rs[0] = rng.s0;
      rs[1] = rng.s1;
      rs[2] = rng.s2;
      rs[3] = rng.s3;
    }
    __syncwarp();
  }
}

// The same replay for rows wider than the register-held widths (NW > 16,
// more than 16 384 features): the clause's planes are read and written in
// place in HBM (lane-owned words, as in sequential.cu), the row is read on use.
template <int B>
__global__ void __launch_bounds__(32) train_mirror_wide_kernel(TrainParams P, MirrorParams M) {
  extern __shared__ __align__(16) uint32_t smem[];
  const int lane = threadIdx.x;
  const int L = 2 * P.o;
  const int refw = (L + 31) / 32 + 2;
  const int tabw = M.jump_chunk ? 2 * kGf2TabWords : 0;
  uint32_t* jc = smem;  // jump tables (M.jump_chunk != null)
  uint32_t* jl = jc + kGf2TabWords;
  uint32_t* hbits = smem + tabw;
  uint32_t* lbits = hbits + refw;
  const int64_t q = P.q;
  const int T = P.margin;
  const int Wp = P.Wp, words = P.Wp >> 5;
  for (int k = lane; k < 2 * refw; k += 32) hbits[k] = 0;
  if (M.jump_chunk)
    for (int k = lane; k < kGf2TabWords; k += 32) {
      jc[k] = M.jump_chunk[k];
      jl[k] = M.jump_lits[k];
    }
  __syncwarp();

  for (int jb = 0; jb < M.njobs; ++jb) {
    const MirrorJob job = M.jobs[jb];
    const int c = job.c;
    const int lc = c * P.n_loc + (job.j - P.j_begin);
    const bool positive = P.all_positive || (job.j & 1) == 0;
    Xoshiro rng;
    uint64_t* rs = M.rng + 4 * job.worker;
    rng.s0 = rs[0];
    rng.s1 = rs[1];
    rng.s2 = rs[2];
    rng.s3 = rs[3];
    uint32_t* st = P.state + static_cast<size_t>(lc) * B * 2 * Wp;
    uint32_t* prev_row = P.prev + static_cast<size_t>(lc) * P.Wq;
    unsigned long long events = 0;
    auto get = [&](int part, int w, Planes<B>& pl) {
#pragma unroll
      for (int b = 0; b < B; ++b) pl.p[b] = st[(b * 2 + part) * Wp + w];
    };
    auto put = [&](int part, int w, const Planes<B>& pl) {
#pragma unroll
      for (int b = 0; b < B; ++b) st[(b * 2 + part) * Wp + w] = pl.p[b];
    };
    auto valid = [&](int w) {
      const int first = w * 32;
      return first >= P.o ? 0u : (P.o - first >= 32 ? kFull : ((1u << (P.o - first)) - 1u));
    };

    const bool forced = job.forced != 0;
    for (int64_t t = 0; t < job.batch; ++t) {
      int64_t i = 0;
      int target = 0, gated = 1;
      if (lane == 0 && !forced) {  // identical to train_mirror_kernel
        const int64_t pos = (job.offset + t) % q;
        i = P.order ? P.order[pos] : pos;
        const int v0 = P.tallies[i * P.m + c];
        const int label = P.labels[i];
        double p;
        if (P.regress) {
          const int v = v0 < 0 ? 0 : (v0 > T ? T : v0);
          const int e = label > v ? label - v : v - label;
          p = fmin(1.0, static_cast<double>(e) / (2.0 * static_cast<double>(T)));
          target = v < label ? 1 : 0;
        } else {
          const int y = label == c ? 1 : 0;
          const int v = v0 < -T ? -T : (v0 > T ? T : v0);
          const int e = y ? T - v : T + v;
          p = static_cast<double>(e) / (2.0 * static_cast<double>(T));
          target = (y == 1) == positive ? 1 : 0;
        }
        gated = next53(rng) < u53_below(p) ? 1 : 0;
      }
      gated = __shfl_sync(kFull, gated, 0);
      if (!gated) continue;
      ++events;
      i = __shfl_sync(kFull, i, 0);
      target = __shfl_sync(kFull, target, 0);
      const uint32_t* xr = P.xplane + i * 2 * Wp;
      const uint32_t* nr = P.nplane + i * 2 * Wp;
      auto eval = [&]() {  // Train mode (core.hpp:208-219): empty clause -> 1
        uint32_t viol = 0, any = 0;
        for (int p = 0; p < words; ++p) {
          const int w = p * 32 + lane;
          const uint32_t ix = st[((B - 1) * 2) * Wp + w], in = st[((B - 1) * 2 + 1) * Wp + w];
          viol |= (ix & ~xr[w]) | (in & ~nr[w]);
          any |= ix | in;
        }
        const unsigned vb = __ballot_sync(kFull, viol != 0), ab = __ballot_sync(kFull, any != 0);
        return ab == 0 ? 1 : (vb == 0 ? 1 : 0);
      };
      const bool type2 = forced ? job.forced == 2 : target == 0;
      const int evald = eval();
      const int before = (forced && job.out_override >= 0) ? job.out_override : evald;
      int after = evald;
      if (type2) {
        if (before) {  // Type II (feedback.cpp:72-83)
          uint32_t moved = 0;
          for (int p = 0; p < words; ++p) {
            const int w = p * 32 + lane;
#pragma unroll
            for (int part = 0; part < 2; ++part) {
              const uint32_t lit = part ? nr[w] : xr[w];
              const uint32_t inc = ~lit & ~st[((B - 1) * 2 + part) * Wp + w] & valid(w);
              if (inc) {
                Planes<B> pl;
                get(part, w, pl);
                add_one<B>(pl, inc);
                put(part, w, pl);
              }
              moved |= inc;
            }
          }
          __syncwarp();
          if (__any_sync(kFull, moved != 0)) after = eval();
        }
      } else {
        if (M.jump_chunk) {
          draw_type_i_bits(rng, L, M.chunk, M.p_high, M.p_low, jc, jl, hbits, lbits, refw, lane);
        } else {
          if (lane == 0) {
            const uint64_t th = u53_below(M.p_high), tl = u53_below(M.p_low);
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
        }
        for (int p = 0; p < words; ++p) {
          const int wi = p * 32 + lane;
          if (wi * 32 >= P.o) continue;
          const int k1 = P.o + wi * 32;
          const uint32_t h[2] = {hbits[wi], __funnelshift_r(hbits[k1 >> 5], hbits[(k1 >> 5) + 1], k1 & 31)};
          const uint32_t l[2] = {lbits[wi], __funnelshift_r(lbits[k1 >> 5], lbits[(k1 >> 5) + 1], k1 & 31)};
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint32_t lit = part ? nr[wi] : xr[wi];
            const uint32_t bern = before ? (lit & h[part]) | (~lit & l[part]) : l[part];
            Planes<B> pl;
            get(part, wi, pl);
            type_i_planes<B, false>(pl, lit, before, P.boost, bern, valid(wi), P.lo, P.hi);
            put(part, wi, pl);
          }
        }
        __syncwarp();
        after = eval();
      }
      if (lane == 0 && !forced) record(P, prev_row, i, c, positive, prev_row[i >> 5], after);
      __syncwarp();
    }
    int cnt = 0;
    for (int w = lane; w < 2 * Wp; w += 32) cnt += __popc(st[(B - 1) * 2 * Wp + w]);
#pragma unroll
    for (int off = 16; off; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
    if (lane == 0) {
      P.inc_count[lc] = cnt;
      P.events[c] += events;
      rs[0] = rng.s0;
      rs[1] = rng.s1;
      rs[2] = rng.s2;
      rs[3] = rng.s3;
    }
    __syncwarp();
  }
}

// --------------------------------------------------- feedback-rate probe ---
// Statistical conformance of the async Type I path (acceptance criterion 1,
// SPEC.md:530): every trial applies type_i_async to a fresh copy of one
// clause (planes at `state0`) with its own Philox counter (example = trial)
// and counts, per reference literal k, the +1 / -1 transitions.
template <int NW, int B>
__global__ void __launch_bounds__(128) feedback_rates_kernel(TrainParams P, const uint32_t* __restrict__ state0,
                                                             int out, uint32_t trials,
                                                             unsigned long long* inc_cnt,
                                                             unsigned long long* dec_cnt) {
  __shared__ uint32_t atab[TMG_ALIAS ? kAliasWords : 1];
  load_alias(P, atab);
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t x[NW], n[NW];
#pragma unroll
  for (int p = 0; p < NW; ++p) {
    x[p] = P.xplane[p * 32 + lane];
    n[p] = P.nplane[p * 32 + lane];
  }
  for (uint32_t trial = warp; trial < trials; trial += nwarps) {
    Clause<NW, B> cl, c0;
    cl.load(state0, P.Wp, lane, P.o);
    c0 = cl;
    type_i_async<NW, B, false>(cl, x, n, out, P, 0u, trial, lane, lane_alias(atab, lane));
#pragma unroll
    for (int p = 0; p < NW; ++p)
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        uint32_t up = 0, down = 0;
#pragma unroll
        for (int b = 0; b < B; ++b) {  // the highest changed plane tells the direction
          const uint32_t ch = c0.s[part][p].p[b] ^ cl.s[part][p].p[b];
          up = (up & ~ch) | (ch & cl.s[part][p].p[b]);
          down = (down & ~ch) | (ch & ~cl.s[part][p].p[b]);
        }
        const int base = part * P.o + (p * 32 + lane) * 32;
        while (up) {
          const int b = __ffs(up) - 1;
          up &= up - 1;
          atomicAdd(inc_cnt + base + b, 1ULL);
        }
        while (down) {
          const int b = __ffs(down) - 1;
          down &= down - 1;
          atomicAdd(dec_cnt + base + b, 1ULL);
        }
      }
  }
}

// One asynchronous Type I feedback (type_i_async, exactly as the epoch kernel
// applies it) on the clause planes at `state`, literal row 0 of P, Philox
// counters (clause g, example i): the deterministic unit the async sampler's
// bit-exact parity test checks against oracle/tm_oracle.c:tm_async_type_i.
template <int NW, int B, bool P2, bool PACK = false>
__global__ void __launch_bounds__(32) type_i_async_once_kernel(TrainParams P, uint32_t* state, uint32_t g,
                                                               uint32_t i, int out) {
  __shared__ uint32_t atab[TMG_ALIAS ? kAliasWords : 1];
  load_alias(P, atab);
  const int lane = threadIdx.x;
  std::conditional_t<PACK, ClausePk<NW, B, P2>, Clause<NW, B, P2>> cl;
  cl.load(state, P.Wp, lane, P.o);
  uint32_t x[NW], n[NW];
#pragma unroll
  for (int p = 0; p < NW; ++p) {
    x[p] = P.xplane[cl.word_of(p, lane)];
    n[p] = PACK ? ~x[p] : P.nplane[p * 32 + lane];
  }
  type_i_async<NW, B, P2>(cl, x, n, out, P, g, i, lane, lane_alias(atab, lane));
  cl.store(state, P.Wp, lane);
}

// Pack the last word slot (ClausePk) when it holds at most 16 valid words and
// the clause-output-1 draws use the alias table; TMG_ASYNC_PACK=0 disables it
// (A/B checks).
bool pack_last_slot(const TrainParams& p, int NW) {
  const char* e = std::getenv("TMG_ASYNC_PACK");
  if ((e && e[0] == '0') || NW < 2 || !TMG_ALIAS || !TMG_ROW_X_ONLY || !p.alias_sel) return false;
  return (p.o + 31) / 32 - 32 * (NW - 1) <= 16;
}

template <int NW, int B>
void launch_async(const TrainParams& p, cudaStream_t s, int* blocks) {
  const int clauses = p.w_end - p.w_begin;
  const int warps_per_block = 4;
  const int grid = (clauses + warps_per_block - 1) / warps_per_block;
  if (blocks) *blocks = grid;
  count_launch();
  const bool p2 = TMG_ASYNC_P2 && p.lo == 0 && p.hi == (1u << B) - 1u;
  if constexpr (NW >= 2) {
    if (pack_last_slot(p, NW)) {
      if (p2) train_async_kernel<NW, B, true, true><<<grid, 32 * warps_per_block, 0, s>>>(p);
      else train_async_kernel<NW, B, false, true><<<grid, 32 * warps_per_block, 0, s>>>(p);
      return;
    }
  }
  if (p2)
    train_async_kernel<NW, B, true><<<grid, 32 * warps_per_block, 0, s>>>(p);
  else
    train_async_kernel<NW, B, false><<<grid, 32 * warps_per_block, 0, s>>>(p);
}

template <int NW, int B>
void launch_mirror(const TrainParams& p, const MirrorParams& mp, cudaStream_t s) {
  const int refw = (2 * p.o + 31) / 32 + 2;
  const size_t shm = sizeof(uint32_t) * (2 * refw + (mp.jump_chunk ? 2 * kGf2TabWords : 0));
  if (shm > 48 * 1024)
    cudaFuncSetAttribute(train_mirror_kernel<NW, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(shm));
  count_launch();
  train_mirror_kernel<NW, B><<<1, 32, shm, s>>>(p, mp);
}

template <int NW, int B>
int resident_async(bool pack) {
  int per_sm = 0, dev = 0, sms = 0;
  if constexpr (NW >= 2) {
    if (pack) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, train_async_kernel<NW, B, true, true>, 128, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, train_async_kernel<NW, B, true>, 128, 0);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, train_async_kernel<NW, B, true>, 128, 0);
  }
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms * 4;
}

template <int B>
int resident_async_nw(int NW, bool pack) {
  switch (NW) {
    case 1: return resident_async<1, B>(false);
    case 2: return resident_async<2, B>(pack);
    case 3: return resident_async<3, B>(pack);
    case 4: return resident_async<4, B>(pack);
    default: return 0;
  }
}

template <int B>
bool dispatch_async(const TrainParams& p, int NW, cudaStream_t s, int* blocks) {
  switch (NW) {
    case 1: launch_async<1, B>(p, s, blocks); return true;
    case 2: launch_async<2, B>(p, s, blocks); return true;
    case 3: launch_async<3, B>(p, s, blocks); return true;
    case 4: launch_async<4, B>(p, s, blocks); return true;
    default: return false;  // wider rows: train_smem.cu
  }
}

template <int B>
bool dispatch_mirror(const TrainParams& p, const MirrorParams& mp, int NW, cudaStream_t s) {
  switch (NW) {
    case 1: launch_mirror<1, B>(p, mp, s); return true;
    case 2: launch_mirror<2, B>(p, mp, s); return true;
    case 3: launch_mirror<3, B>(p, mp, s); return true;
    case 4: launch_mirror<4, B>(p, mp, s); return true;
    case 6: launch_mirror<6, B>(p, mp, s); return true;
    case 8: launch_mirror<8, B>(p, mp, s); return true;
    case 10: launch_mirror<10, B>(p, mp, s); return true;
    case 12: launch_mirror<12, B>(p, mp, s); return true;
    case 16: launch_mirror<16, B>(p, mp, s); return true;
    default: {  // rows wider than 16 words per lane: planes in place
      const int refw = (2 * p.o + 31) / 32 + 2;
      const size_t shm = sizeof(uint32_t) * (2 * refw + (mp.jump_chunk ? 2 * kGf2TabWords : 0));
      if (shm > 227 * 1024) return false;
      if (shm > 48 * 1024)
        cudaFuncSetAttribute(train_mirror_wide_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(shm));
      count_launch();
      train_mirror_wide_kernel<B><<<1, 32, shm, s>>>(p, mp);
      return true;
    }
  }
}

}  // namespace

bool feedback_rates_launch(const TrainParams& p, const uint32_t* state0, int out, uint32_t trials, int B, int NW,
                           unsigned long long* inc, unsigned long long* dec, cudaStream_t s) {
  const int grid = 148 * 4;
  auto go = [&](auto kern) {
    count_launch();
    kern<<<grid, 128, 0, s>>>(p, state0, out, trials, inc, dec);
    return true;
  };
  if (NW == 1 && B == 4) return go(feedback_rates_kernel<1, 4>);
  if (NW == 1 && B == 8) return go(feedback_rates_kernel<1, 8>);
  if (NW == 1 && B == 15) return go(feedback_rates_kernel<1, 15>);
  if (NW == 3 && B == 8) return go(feedback_rates_kernel<3, 8>);
  return false;
}

template <int NW, int B, typename Go>
bool once_dispatch(const TrainParams& p, bool p2, Go&& go) {
  if constexpr (NW >= 2) {
    if (pack_last_slot(p, NW))
      return p2 ? go(type_i_async_once_kernel<NW, B, true, true>) : go(type_i_async_once_kernel<NW, B, false, true>);
  }
  return p2 ? go(type_i_async_once_kernel<NW, B, true>) : go(type_i_async_once_kernel<NW, B, false>);
}

bool type_i_async_once_launch(const TrainParams& p, uint32_t* state, uint32_t g, uint32_t i, int out, int B, int NW,
                              cudaStream_t s) {
  const bool p2 = TMG_ASYNC_P2 && p.lo == 0 && p.hi == (1u << B) - 1u;
  auto go = [&](auto kern) {
    count_launch();
    kern<<<1, 32, 0, s>>>(p, state, g, i, out);
    return true;
  };
#define TMG_ONCE(nw, b) \
  if (NW == nw && B == b) return once_dispatch<nw, b>(p, p2, go);
  TMG_ONCE(1, 4) TMG_ONCE(1, 8) TMG_ONCE(1, 15) TMG_ONCE(2, 4) TMG_ONCE(2, 8) TMG_ONCE(2, 15)
  TMG_ONCE(3, 4) TMG_ONCE(3, 8) TMG_ONCE(3, 15) TMG_ONCE(4, 4) TMG_ONCE(4, 8) TMG_ONCE(4, 15)
#undef TMG_ONCE
  return false;
}

int train_async_resident_warps(const TrainParams& p, int B, int NW, int* warps_per_cta) {
  if (NW > 4) return train_async_smem_resident_warps(p, B, NW, warps_per_cta);
  *warps_per_cta = 4;
  switch (B) {
    case 4: return resident_async_nw<4>(NW, pack_last_slot(p, NW));
    case 8: return resident_async_nw<8>(NW, pack_last_slot(p, NW));
    case 15: return resident_async_nw<15>(NW, pack_last_slot(p, NW));
    default: return 0;
  }
}

bool train_async_launch(const TrainParams& p, int B, int NW, cudaStream_t s, int* blocks) {
  switch (B) {
    case 4: return dispatch_async<4>(p, NW, s, blocks);
    case 8: return dispatch_async<8>(p, NW, s, blocks);
    case 15: return dispatch_async<15>(p, NW, s, blocks);
    default: return false;
  }
}

bool train_mirror_launch(const TrainParams& p, const MirrorParams& mp, int B, int NW, cudaStream_t s) {
  switch (B) {
    case 4: return dispatch_mirror<4>(p, mp, NW, s);
    case 8: return dispatch_mirror<8>(p, mp, NW, s);
    case 15: return dispatch_mirror<15>(p, mp, NW, s);
    default: return false;
  }
}

}  // namespace tmg
