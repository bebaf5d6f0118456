/*
 * tm_oracle_async.c — CPU restatement of the B200 engine's ASYNCHRONOUS
 * Type I feedback draw (paper_2009_04861_b200/csrc/tm_device.cuh
 * bernoulli_words + train.cu type_i_async), for the deterministic parity test
 * of the async sampler. TEST INFRASTRUCTURE ONLY (see tm_oracle.h).
 *
 * The reference draws one xoshiro uniform per literal and feeds back w.p.
 * p_high = (s-1)/s or p_low = 1/s (src/feedback.cpp:24-70). The async engine
 * keeps that rule but replaces the stream by counter-based Philox4x32-R
 * (Salmon et al., SC'11) keyed per (seed, epoch) and draws each literal's
 * 32-bit uniform u bit-serially; the literal is fed back iff u < P with
 * P = round(p * 2^32). This file states that draw literal by literal:
 *
 *   literal k < o is feature f = k (part 0), k >= o is f = k - o (part 1);
 *   word wi = f / 32, bit b = f % 32, lane = wi % 32, pass = wi / 32,
 *   slot = 2 * pass + part, word id = 2 * wi + part, K = 2 * NW slots.
 *   u bits 31..24: bit b of word (r % 4) of Philox(g, i, word id, r / 4),
 *                  r = 0..7 (MSB first);
 *   u bits 23..0 (only when bits 31..24 equal P's): bits 31..8 of word
 *                  (slot % 4) of Philox(g, i, 0xFFFF0000 | lane,
 *                  2 + t * ceil(K/4) + slot / 4), where t is the number of
 *                  lower still-undecided literals of the same slot.
 *
 * The transition applied with the drawn bit is the reference's
 * (feedback.cpp:32-70, saturating counters in [1, 2N], core.hpp:55-65):
 *   out=1, lit=1: +1 w.p. p_high (always if boost and included)
 *   out=1, lit=0: +1 if included / -1 if excluded, w.p. p_low
 *   out=0       : -1 w.p. p_low
 * With out=0 and an alias table the engine draws whole 8-literal patterns
 * instead (see orc_async_type_i below and tm_device.cuh alias_words).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "tm_oracle.h"

void orc_philox4x32(const uint32_t ctr[4], uint32_t k0, uint32_t k1, int rounds, uint32_t out[4]) {
  uint32_t x = ctr[0], y = ctr[1], z = ctr[2], w = ctr[3];
  for (int r = 0; r < rounds; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * x, p1 = (uint64_t)0xCD9E8D57u * z;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t nx = hi1 ^ y ^ k0, ny = lo1, nz = hi0 ^ w ^ k1, nw = lo0;
    x = nx;
    y = ny;
    z = nz;
    w = nw;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = x;
  out[1] = y;
  out[2] = z;
  out[3] = w;
}

/* Philox key of an epoch: mix_stream(4, epoch, seed), low word first. */
void orc_async_key(uint64_t seed, int32_t epoch, uint32_t* key0, uint32_t* key1) {
  uint64_t k = orc_mix_stream(4, (uint64_t)epoch, seed);
  *key0 = (uint32_t)k;
  *key1 = (uint32_t)(k >> 32);
}

/* P(u < p) as 32-bit fixed point (engine.cu prob_threshold). */
uint32_t orc_prob_threshold(double p) {
  if (!(p > 0.0)) return 0u;
  double v = ldexp(p, 32);
  if (v >= 4294967295.0) return 0xFFFFFFFFu;
  return (uint32_t)llround(v);
}

static int lit_bit(const uint64_t* w, int k) { return (int)((w[k >> 6] >> (k & 63)) & 1u); }

void orc_async_type_i(uint16_t* counters, const uint64_t* lits, int32_t o, int32_t N, int32_t out, double s,
                      int32_t boost, uint32_t g, uint32_t i, uint32_t key0, uint32_t key1, int32_t nw,
                      int32_t rounds, const uint32_t* alias8) {
  const int L = 2 * o;
  const uint32_t p_high0 = orc_prob_threshold((s - 1.0) / s), p_low0 = orc_prob_threshold(1.0 / s);
  const int alias_sel = (uint64_t)p_high0 + p_low0 == ((uint64_t)1 << 32);
  if (out && alias8 && alias_sel) {
    /* Clause output 1 with p_high = 1 - p_low exactly: the same alias
     * patterns, negated on the true literals (tm_device.cuh / train.cu). */
    for (int part = 0; part < 2; ++part)
      for (int wi = 0; wi * 32 < o; ++wi) {
        const uint32_t ctr[4] = {g, i, (uint32_t)(2 * wi + part), 0u};
        uint32_t blk[4];
        orc_philox4x32(ctr, key0, key1, rounds, blk);
        for (int j = 0; j < 4; ++j) {
          const uint32_t u = blk[j], e = alias8[u & 0xFFu];
          const uint32_t pattern = ((u | 0xFFu) < e ? u : e) & 0xFFu;
          for (int b = 0; b < 8; ++b) {
            const int f = wi * 32 + j * 8 + b;
            if (f >= o) continue;
            const int k = part * o + f, lit = lit_bit(lits, k);
            const int fire = (int)((pattern >> b) & 1u) ^ lit;
            const int included = counters[k] > N;
            int v = counters[k];
            if (lit) {
              if (fire || (boost && included)) v += 1;
            } else if (fire) {
              v += included ? 1 : -1;
            }
            if (v < 1) v = 1;
            if (v > 2 * N) v = 2 * N;
            counters[k] = (uint16_t)v;
          }
        }
      }
    return;
  }
  if (!out && alias8) {
    /* Clause output 0: each aligned 8-literal group of word slot (wi, part)
     * draws its pattern with byte j's uniform u = word j of Philox(g, i,
     * 2*wi + part, 0) from the alias table (tm_device.cuh alias_words). */
    for (int part = 0; part < 2; ++part)
      for (int wi = 0; wi * 32 < o; ++wi) {
        const uint32_t ctr[4] = {g, i, (uint32_t)(2 * wi + part), 0u};
        uint32_t blk[4];
        orc_philox4x32(ctr, key0, key1, rounds, blk);
        for (int j = 0; j < 4; ++j) {
          const uint32_t u = blk[j], e = alias8[u & 0xFFu];
          const uint32_t pattern = ((u | 0xFFu) < e ? u : e) & 0xFFu;
          for (int b = 0; b < 8; ++b) {
            const int f = wi * 32 + j * 8 + b;
            if (f >= o || !((pattern >> b) & 1u)) continue;
            const int k = part * o + f;
            if (counters[k] > 1) counters[k] -= 1; /* -1 w.p. p_low, saturating at 1 */
          }
        }
      }
    return;
  }
  const uint32_t p_high = orc_prob_threshold((s - 1.0) / s), p_low = orc_prob_threshold(1.0 / s);
  const int K = 2 * nw, nb = (K + 3) / 4;
  uint8_t* bern = (uint8_t*)malloc((size_t)L);
  uint8_t* und = (uint8_t*)malloc((size_t)L);
  uint32_t* thr = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)L);
  /* Per literal: the threshold, then phase 1 on the top 8 bits. */
  for (int k = 0; k < L; ++k) {
    const int part = k >= o, f = part ? k - o : k, wi = f >> 5, b = f & 31;
    const uint32_t P = (out && lit_bit(lits, k)) ? p_high : p_low;
    thr[k] = P;
    uint32_t top = 0;
    for (int r = 0; r < 8; ++r) {
      const uint32_t ctr[4] = {g, i, (uint32_t)(2 * wi + part), (uint32_t)(r / 4)};
      uint32_t blk[4];
      orc_philox4x32(ctr, key0, key1, rounds, blk);
      top = (top << 1) | ((blk[r % 4] >> b) & 1u);
    }
    const uint32_t ptop = P >> 24;
    bern[k] = top < ptop;
    und[k] = top == ptop;
  }
  /* Phase 2: per (lane, slot), undecided literals in increasing bit order. */
  for (int part = 0; part < 2; ++part) {
    for (int wi = 0; wi * 32 < o; ++wi) {
      const int lane = wi & 31, pass = wi >> 5, slot = 2 * pass + part;
      int t = 0;
      for (int b = 0; b < 32 && wi * 32 + b < o; ++b) {
        const int k = part * o + wi * 32 + b;
        if (!und[k]) continue;
        const uint32_t ctr[4] = {g, i, 0xFFFF0000u | (uint32_t)lane, (uint32_t)(2 + t * nb + slot / 4)};
        uint32_t blk[4];
        orc_philox4x32(ctr, key0, key1, rounds, blk);
        bern[k] = (blk[slot % 4] >> 8) < (thr[k] & 0x00FFFFFFu);
        ++t;
      }
    }
  }
  for (int k = 0; k < L; ++k) {
    if (!bern[k] && !(out && boost && lit_bit(lits, k) && counters[k] > N)) continue;
    const int included = counters[k] > N;
    int v = counters[k];
    if (out) {
      if (lit_bit(lits, k)) v += 1;
      else v += included ? 1 : -1;
    } else {
      v -= 1;
    }
    if (v < 1) v = 1;
    if (v > 2 * N) v = 2 * N;
    counters[k] = (uint16_t)v;
  }
  free(bern);
  free(und);
  free(thr);
}
