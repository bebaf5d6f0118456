/*
 * Synthetic example generators for the configs in BASELINE.json.
 *
 * No dataset ships with the reference and the box has no network, so every
 * config is generated from one seeded xoshiro256++ stream (include/tmgpu_rng.h)
 * in a fixed draw order. The same C file is linked into the reference driver
 * (oracle/ref_driver.cpp), so the CPU reference and the GPU engine train on
 * byte-identical inputs.
 *
 *   XOR12 : SURVEY.md §8(d) — y = x0 ^ x1 over `features` uniform bits,
 *           label noise on the train split only (like synth_xor,
 *           proj/src/data_io.cpp:322-346, widened to distractor bits).
 *   MNIST : the oracle-calibrated prototype recipe, SURVEY.md §8(d).
 *   FMNIST: grey prototypes + noise, thermometer-coded at 3 thresholds.
 *   IMDB  : Zipf bag-of-words with class-conditional sentiment words.
 *
 * Input bits are row-major q x o uint8 in {0,1}; labels int32.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "tmgpu_rng.h"

#if defined(__GNUC__)
#define TMG_EXPORT __attribute__((visibility("default")))
#else
#define TMG_EXPORT
#endif

TMG_EXPORT int tmg_synth_xor(uint64_t seed, int64_t rows, int features, double noise,
                             int with_noise, uint8_t* bits, int32_t* labels) {
  tmg_rng g;
  int64_t r;
  int f;
  if (features < 2 || rows < 0 || noise < 0.0 || noise >= 0.5) return -1;
  tmg_rng_seed(&g, seed, 0xD47A);
  for (r = 0; r < rows; ++r) {
    uint8_t* x = bits + r * features;
    int32_t y;
    for (f = 0; f < features; ++f) x[f] = (uint8_t)tmg_rng_below(&g, 2);
    y = x[0] ^ x[1];
    if (with_noise && noise > 0.0 && tmg_rng_uniform(&g) < noise) y = 1 - y;
    labels[r] = y;
  }
  return 0;
}

/* Prototype recipe: stream Rng(seed, 0x4D4E); base pattern,
 * per-class resample at r_class, 8 sub-prototypes per class at r_sub, rows =
 * sub-prototype xor Bernoulli(flip). Train rows first, then test rows. */
TMG_EXPORT int tmg_synth_mnist(uint64_t seed, int features, int classes, double r_class,
                               double r_sub, double flip, int64_t train_rows,
                               int64_t test_rows, uint8_t* train_bits,
                               int32_t* train_labels, uint8_t* test_bits,
                               int32_t* test_labels) {
  enum { SUBS = 8 };
  tmg_rng g;
  uint8_t *base, *pc, *sub;
  int i, c, k;
  int64_t r;
  if (features < 1 || classes < 2 || train_rows < 0 || test_rows < 0) return -1;
  base = (uint8_t*)malloc((size_t)features);
  pc = (uint8_t*)malloc((size_t)features);
  sub = (uint8_t*)malloc((size_t)features * classes * SUBS);
  if (!base || !pc || !sub) {
    free(base); free(pc); free(sub);
    return -2;
  }
  tmg_rng_seed(&g, seed, 0x4D4E);
  for (i = 0; i < features; ++i) base[i] = (uint8_t)tmg_rng_bernoulli(&g, 0.2);
  for (c = 0; c < classes; ++c) {
    memcpy(pc, base, (size_t)features);
    for (i = 0; i < features; ++i)
      if (tmg_rng_bernoulli(&g, r_class)) pc[i] = (uint8_t)tmg_rng_bernoulli(&g, 0.2);
    for (k = 0; k < SUBS; ++k) {
      uint8_t* dst = sub + ((size_t)c * SUBS + k) * features;
      for (i = 0; i < features; ++i) {
        uint8_t b = pc[i];
        if (tmg_rng_bernoulli(&g, r_sub)) b = (uint8_t)tmg_rng_bernoulli(&g, 0.2);
        dst[i] = b;
      }
    }
  }
  for (r = 0; r < train_rows + test_rows; ++r) {
    const int in_train = r < train_rows;
    uint8_t* x = in_train ? train_bits + r * features : test_bits + (r - train_rows) * features;
    const int cls = (int)tmg_rng_below(&g, (uint32_t)classes);
    const int kk = (int)tmg_rng_below(&g, SUBS);
    const uint8_t* proto = sub + ((size_t)cls * SUBS + kk) * features;
    for (i = 0; i < features; ++i) x[i] = proto[i] ^ (uint8_t)tmg_rng_bernoulli(&g, flip);
    if (in_train) train_labels[r] = cls; else test_labels[r - train_rows] = cls;
  }
  free(base); free(pc); free(sub);
  return 0;
}

/* Fashion-MNIST-shaped: `pixels` grey levels from per-class grey prototypes
 * (resampled at r_class from a shared base, 8 sub-prototypes at r_sub),
 * blended with a random other class's prototype at weight w ~ U[0, mix)
 * (ambiguous, non-saturating examples), plus uniform additive noise of +-amp,
 * thermometer-coded at 64/128/192 into 3*pixels bits (bit 3*i+t =
 * grey_i > threshold_t). */
TMG_EXPORT int tmg_synth_fmnist(uint64_t seed, int pixels, int classes, double r_class,
                                double r_sub, int amp, double mix, int64_t train_rows,
                                int64_t test_rows, uint8_t* train_bits, int32_t* train_labels,
                                uint8_t* test_bits, int32_t* test_labels) {
  enum { SUBS = 8 };
  static const int thresholds[3] = {64, 128, 192};
  tmg_rng g;
  uint8_t *base, *pc, *sub;
  int i, c, k, t;
  int64_t r;
  const int o = 3 * pixels;
  if (pixels < 1 || classes < 2 || amp < 0) return -1;
  base = (uint8_t*)malloc((size_t)pixels);
  pc = (uint8_t*)malloc((size_t)pixels);
  sub = (uint8_t*)malloc((size_t)pixels * classes * SUBS);
  if (!base || !pc || !sub) {
    free(base); free(pc); free(sub);
    return -2;
  }
  tmg_rng_seed(&g, seed, 0x464D);
  for (i = 0; i < pixels; ++i) base[i] = (uint8_t)tmg_rng_below(&g, 256);
  for (c = 0; c < classes; ++c) {
    for (i = 0; i < pixels; ++i)
      pc[i] = tmg_rng_bernoulli(&g, r_class) ? (uint8_t)tmg_rng_below(&g, 256) : base[i];
    for (k = 0; k < SUBS; ++k) {
      uint8_t* dst = sub + ((size_t)c * SUBS + k) * pixels;
      for (i = 0; i < pixels; ++i)
        dst[i] = tmg_rng_bernoulli(&g, r_sub) ? (uint8_t)tmg_rng_below(&g, 256) : pc[i];
    }
  }
  for (r = 0; r < train_rows + test_rows; ++r) {
    const int in_train = r < train_rows;
    uint8_t* x = in_train ? train_bits + r * o : test_bits + (r - train_rows) * o;
    const int cls = (int)tmg_rng_below(&g, (uint32_t)classes);
    const int kk = (int)tmg_rng_below(&g, SUBS);
    const uint8_t* proto = sub + ((size_t)cls * SUBS + kk) * pixels;
    int other = (int)tmg_rng_below(&g, (uint32_t)(classes - 1));
    const double w = tmg_rng_uniform(&g) * mix;
    const uint8_t* oproto;
    if (other >= cls) ++other;
    oproto = sub + ((size_t)other * SUBS + kk) * pixels;
    for (i = 0; i < pixels; ++i) {
      const double blend = (1.0 - w) * (double)proto[i] + w * (double)oproto[i];
      int v = (int)(blend + 0.5) + (int)tmg_rng_below(&g, (uint32_t)(2 * amp + 1)) - amp;
      if (v < 0) v = 0;
      if (v > 255) v = 255;
      for (t = 0; t < 3; ++t) x[3 * i + t] = (uint8_t)(v > thresholds[t]);
    }
    if (in_train) train_labels[r] = cls; else test_labels[r - train_rows] = cls;
  }
  free(base); free(pc); free(sub);
  return 0;
}

/* The canonical datasets of BASELINE.json configs (single source of truth for
 * the GPU bench/tests and oracle/ref_driver): kind 0 XOR12 (label noise
 * `noise`), 1 MNIST-shaped, 2 FMNIST-shaped, 3 IMDb-shaped. Returns the
 * feature count via *features (bits must hold rows x features). */
int tmg_synth_imdb(uint64_t seed, int vocab, int sentiment, double p_sent, double cross,
                   int64_t train_rows, int64_t test_rows, uint8_t* train_bits,
                   int32_t* train_labels, uint8_t* test_bits, int32_t* test_labels);

TMG_EXPORT int tmg_synth_preset(int kind, uint64_t seed, double noise, int64_t train_rows, int64_t test_rows,
                                uint8_t* train_bits, int32_t* train_labels, uint8_t* test_bits,
                                int32_t* test_labels) {
  switch (kind) {
    case 0: {
      const int rc = tmg_synth_xor(seed, train_rows, 12, noise, 1, train_bits, train_labels);
      return rc ? rc : tmg_synth_xor(seed + 1000003, test_rows, 12, noise, 0, test_bits, test_labels);
    }
    case 1:  /* SURVEY.md §8(d) calibrated recipe */
      return tmg_synth_mnist(seed, 784, 10, 0.10, 0.10, 0.30, train_rows, test_rows, train_bits,
                             train_labels, test_bits, test_labels);
    case 2:
      /* blend weight ~ U[0, 0.55): ~9 % of rows lean to another class
         (calibrated on the GPU, tools/calib_synth.py: mix 0.8 -> 62 %). */
      return tmg_synth_fmnist(seed, 784, 10, 0.10, 0.15, 60, 0.55, train_rows, test_rows, train_bits,
                              train_labels, test_bits, test_labels);
    case 3:
      return tmg_synth_imdb(seed, 10000, 250, 0.10, 0.3, train_rows, test_rows, train_bits, train_labels,
                            test_bits, test_labels);
    default:
      return -1;
  }
}

/* IMDb-shaped bag of words: vocabulary `vocab`, Zipf(1) frequencies with rank
 * shift 10, `sentiment` words per class drawn from ranks [100, 100+4*sentiment*2),
 * documents of 120..279 tokens, each token a sentiment word of the document's
 * class w.p. p_sent (of the other class w.p. p_sent*cross), else a Zipf word. */
TMG_EXPORT int tmg_synth_imdb(uint64_t seed, int vocab, int sentiment, double p_sent,
                              double cross, int64_t train_rows, int64_t test_rows,
                              uint8_t* train_bits, int32_t* train_labels,
                              uint8_t* test_bits, int32_t* test_labels) {
  tmg_rng g;
  double* cdf;
  int32_t* sent;
  uint8_t* used;
  int i, s;
  int64_t r;
  double total = 0.0;
  const int span = 8 * sentiment;
  if (vocab < 100 + span || sentiment < 1) return -1;
  cdf = (double*)malloc(sizeof(double) * (size_t)vocab);
  sent = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)sentiment);
  used = (uint8_t*)calloc((size_t)vocab, 1);
  if (!cdf || !sent || !used) {
    free(cdf); free(sent); free(used);
    return -2;
  }
  for (i = 0; i < vocab; ++i) {
    total += 1.0 / (double)(i + 10);
    cdf[i] = total;
  }
  for (i = 0; i < vocab; ++i) cdf[i] /= total;
  tmg_rng_seed(&g, seed, 0x494D);
  for (s = 0; s < 2 * sentiment; ++s) {
    int w;
    do {
      w = 100 + (int)tmg_rng_below(&g, (uint32_t)span);
    } while (used[w]);
    used[w] = 1;
    sent[s] = w;
  }
  for (r = 0; r < train_rows + test_rows; ++r) {
    const int in_train = r < train_rows;
    uint8_t* x = in_train ? train_bits + r * vocab : test_bits + (r - train_rows) * vocab;
    const int y = (int)tmg_rng_below(&g, 2);
    const int len = 120 + (int)tmg_rng_below(&g, 160);
    int tok;
    memset(x, 0, (size_t)vocab);
    for (tok = 0; tok < len; ++tok) {
      const double u = tmg_rng_uniform(&g);
      int w;
      if (u < p_sent) {
        w = sent[y * sentiment + (int)tmg_rng_below(&g, (uint32_t)sentiment)];
      } else if (u < p_sent * (1.0 + cross)) {
        w = sent[(1 - y) * sentiment + (int)tmg_rng_below(&g, (uint32_t)sentiment)];
      } else {
        const double v = tmg_rng_uniform(&g);
        int lo = 0, hi = vocab - 1;
        while (lo < hi) {
          const int mid = (lo + hi) / 2;
          if (cdf[mid] > v) hi = mid; else lo = mid + 1;
        }
        w = lo;
      }
      x[w] = 1;
    }
    if (in_train) train_labels[r] = y; else test_labels[r - train_rows] = y;
  }
  free(cdf); free(sent); free(used);
  return 0;
}
