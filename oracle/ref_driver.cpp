// ref_driver — test-infrastructure driver for the CPU reference.
//
// Written ONLY against the reference's public C++ API (tsetlin/core.hpp,
// rng.hpp, feedback.hpp, pool.hpp, trainer.hpp); oracle/Makefile compiles it
// with the reference sources under /root/reference/proj into oracle/_ref/.
// It is the checker, never the product:
//   golden <dir>   dump known-answer vectors (tests/golden/gen_golden.sh)
//   train  ...     time train_epoch_parallel / _sequential on synthetic data
//                  (bench.py's cpu_baseline and --impl reference arm, and the
//                  async-accuracy reference numbers in tests/golden/)
//   predict <model> ...  time predict_all on a saved model (tools/eval_time.py)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <sstream>

#include "npy.hpp"
#include "tsetlin/feedback.hpp"
#include "tsetlin/model_io.hpp"
#include "tsetlin/regression.hpp"
#include "tsetlin/pool.hpp"
#include "tsetlin/rng.hpp"
#include "tsetlin/trainer.hpp"

extern "C" {
// csrc/synth.c: the canonical BASELINE.json datasets (shared with the GPU side)
int tmg_synth_preset(int kind, std::uint64_t seed, double noise, std::int64_t train_rows,
                     std::int64_t test_rows, std::uint8_t* train_bits, std::int32_t* train_labels,
                     std::uint8_t* test_bits, std::int32_t* test_labels);
}

namespace fs = std::filesystem;
using namespace tsetlin;

namespace {

struct Split {
  int features = 0;
  int classes = 0;
  std::vector<std::uint8_t> train_x, test_x;
  std::vector<std::int32_t> train_y, test_y;
};

Split make_data(const std::string& kind, std::int64_t q, std::int64_t qt, std::uint64_t seed,
                double noise) {
  Split s;
  if (kind == "xor") {
    s.features = 12;
    s.classes = 2;
  } else if (kind == "mnist") {
    s.features = 784;
    s.classes = 10;
  } else if (kind == "fmnist") {
    s.features = 2352;
    s.classes = 10;
  } else if (kind == "imdb") {
    s.features = 10000;
    s.classes = 2;
  } else {
    throw std::invalid_argument("unknown data kind " + kind);
  }
  s.train_x.resize(static_cast<std::size_t>(q) * s.features);
  s.test_x.resize(static_cast<std::size_t>(qt) * s.features);
  s.train_y.resize(static_cast<std::size_t>(q));
  s.test_y.resize(static_cast<std::size_t>(qt));
  const int k = kind == "xor" ? 0 : kind == "mnist" ? 1 : kind == "fmnist" ? 2 : 3;
  if (tmg_synth_preset(k, seed, noise, q, qt, s.train_x.data(), s.train_y.data(), s.test_x.data(),
                       s.test_y.data()))
    throw std::runtime_error("synthetic generator failed");
  return s;
}

std::vector<std::uint64_t> prev_bitmap(const ClassBank& bank) {
  const int q = bank.bound_examples();
  const int words = (q + 63) / 64;
  std::vector<std::uint64_t> out(static_cast<std::size_t>(bank.clause_count()) * words, 0);
  for (int j = 0; j < bank.clause_count(); ++j)
    for (int i = 0; i < q; ++i)
      if (bank.prev_output(j, i)) out[static_cast<std::size_t>(j) * words + (i >> 6)] |= 1ULL << (i & 63);
  return out;
}

void dump_state(const std::string& dir, const std::string& tag, const MultiClassTM& tm,
                const ExamplePool& pool) {
  const int m = tm.num_banks();
  const int n = tm.config.clauses;
  const int L = tm.banks[0].literal_count();
  const int W = tm.banks[0].words_per_clause();
  std::vector<std::uint16_t> counters;
  std::vector<std::uint64_t> masks, prev;
  std::vector<std::int32_t> counts, tallies;
  for (const auto& bank : tm.banks) {
    counters.insert(counters.end(), bank.counters().begin(), bank.counters().end());
    for (int j = 0; j < n; ++j) {
      auto mk = bank.include_mask(j);
      masks.insert(masks.end(), mk.begin(), mk.end());
      counts.push_back(bank.include_count(j));
    }
    auto pb = prev_bitmap(bank);
    prev.insert(prev.end(), pb.begin(), pb.end());
  }
  for (int i = 0; i < pool.size(); ++i)
    for (int c = 0; c < pool.num_classes(); ++c) tallies.push_back(pool.tally(i, c));
  const std::size_t ms = static_cast<std::size_t>(m), ns = static_cast<std::size_t>(n);
  npyio::save(dir + "/" + tag + "_counters.npy", counters.data(), {ms, ns, static_cast<std::size_t>(L)});
  npyio::save(dir + "/" + tag + "_masks.npy", masks.data(), {ms, ns, static_cast<std::size_t>(W)});
  npyio::save(dir + "/" + tag + "_counts.npy", counts.data(), {ms, ns});
  const std::size_t pw = prev.size() / (ms * ns);
  npyio::save(dir + "/" + tag + "_prev.npy", prev.data(), {ms, ns, pw});
  npyio::save(dir + "/" + tag + "_tallies.npy", tallies.data(),
              {static_cast<std::size_t>(pool.size()), static_cast<std::size_t>(pool.num_classes())});
}

void write_text(const std::string& path, const std::string& text) {
  FILE* f = std::fopen(path.c_str(), "w");
  std::fputs(text.c_str(), f);
  std::fclose(f);
}

// ---------------------------------------------------------------- golden ---

void golden_rng(const std::string& dir) {
  fs::create_directories(dir);
  const std::uint64_t seeds[3][2] = {{42, 0}, {42, 3}, {7, 123456789}};
  std::vector<std::uint64_t> nexts;
  std::vector<double> unis;
  for (auto& sp : seeds) {
    Rng r(sp[0], sp[1]);
    for (int k = 0; k < 64; ++k) nexts.push_back(r.next());
    for (int k = 0; k < 16; ++k) unis.push_back(r.uniform());
  }
  npyio::save(dir + "/next.npy", nexts.data(), {3, 64});
  npyio::save(dir + "/uniform.npy", unis.data(), {3, 16});
  const std::uint32_t bounds[] = {1u, 2u, 3u, 10u, 1000u, 2147483649u, 4294967295u};
  std::vector<std::uint32_t> below;
  Rng rb(11, 22);
  for (auto b : bounds)
    for (int k = 0; k < 8; ++k) below.push_back(rb.below(b));
  npyio::save(dir + "/below.npy", below.data(), {7, 8});
  Rng rs(5, 2);
  auto perm = shuffled_indices(37, rs);
  npyio::save(dir + "/perm37.npy", perm);
  Rng rs2(42, 77);
  auto perm2 = shuffled_indices(1000, rs2);
  npyio::save(dir + "/perm1000.npy", perm2);
}

void golden_pack(const std::string& dir) {
  fs::create_directories(dir);
  const int os[] = {1, 2, 12, 31, 32, 33, 63, 64, 65, 100, 784};
  Rng r(99, 1);
  for (int o : os) {
    std::vector<std::uint8_t> bits(static_cast<std::size_t>(3 * o));
    for (auto& b : bits) b = static_cast<std::uint8_t>(r.below(2));
    std::vector<std::int32_t> labels = {0, 1, 0};
    ExamplePool pool(o, bits, labels, 2);
    std::vector<std::uint64_t> lits;
    for (int i = 0; i < 3; ++i) {
      auto l = pool.literals(i);
      lits.insert(lits.end(), l.begin(), l.end());
    }
    npyio::save(dir + "/bits_o" + std::to_string(o) + ".npy", bits.data(), {3, static_cast<std::size_t>(o)});
    npyio::save(dir + "/lits_o" + std::to_string(o) + ".npy", lits.data(),
                {3, static_cast<std::size_t>(pool.words_per_example())});
  }
}

void golden_gate(const std::string& dir) {
  fs::create_directories(dir);
  const int margins[] = {1, 5, 15, 50};
  std::vector<double> p;
  for (int T : margins)
    for (int y = 0; y < 2; ++y)
      for (int v = -60; v <= 60; ++v) p.push_back(clause_update_probability(v, y, T));
  npyio::save(dir + "/prob.npy", p.data(), {4, 2, 121});
}

// Random counter initialisation with a controllable include rate. When
// `satisfy` is set, included literals are restricted to those true on x so
// the clause fires (c = 1).
void random_bank(ClassBank& bank, Rng& r, double include_rate, const std::vector<std::uint64_t>* lits,
                 bool satisfy) {
  const int N = bank.state_depth();
  for (int j = 0; j < bank.clause_count(); ++j)
    for (int k = 0; k < bank.literal_count(); ++k) {
      bool inc = r.uniform() < include_rate;
      if (inc && satisfy && lits && !literal_bit(*lits, k)) inc = false;
      int v;
      if (inc) v = N + 1 + static_cast<int>(r.below(static_cast<std::uint32_t>(N)));
      else v = 1 + static_cast<int>(r.below(static_cast<std::uint32_t>(N)));
      if (r.uniform() < 0.2) v = inc ? 2 * N : 1;  // saturation edges
      if (r.uniform() < 0.1) v = inc ? N + 1 : N;  // decision boundary
      bank.set_counter(j, k, static_cast<StateCounter>(v));
    }
}

void golden_feedback(const std::string& dir) {
  fs::create_directories(dir);
  struct Case { int o, N; double s; int boost, type, satisfy; };
  const Case cases[] = {
      {12, 128, 3.9, 0, 1, 0}, {12, 128, 3.9, 0, 1, 1}, {12, 128, 3.9, 1, 1, 1},
      {12, 128, 3.9, 0, 2, 1}, {12, 128, 3.9, 0, 2, 0}, {40, 5, 2.0, 0, 1, 1},
      {40, 5, 10.0, 1, 1, 1},  {40, 5, 1.0, 0, 1, 0},   {784, 128, 10.0, 0, 1, 0},
      {784, 128, 10.0, 0, 1, 1}, {784, 128, 10.0, 0, 2, 1}, {100, 300, 7.5, 1, 1, 1},
      {33, 1, 3.0, 0, 1, 1},   {33, 1, 3.0, 0, 2, 1},   {65, 16383, 4.0, 1, 1, 1},
  };
  int idx = 0;
  std::string manifest = "[\n";
  for (const auto& cs : cases) {
    Rng r(1000 + idx, 5);
    std::vector<std::uint8_t> x(static_cast<std::size_t>(cs.o));
    for (auto& b : x) b = static_cast<std::uint8_t>(r.below(2));
    std::vector<std::uint64_t> lits(static_cast<std::size_t>(literal_words(cs.o)));
    pack_literals(x, lits);
    ClassBank bank(cs.o, 2, cs.N);
    random_bank(bank, r, cs.o > 100 ? 0.01 : 0.15, &lits, cs.satisfy != 0);
    std::vector<std::uint16_t> before(bank.counters().begin(), bank.counters().end());
    const int out = evaluate_clause(bank, 1, lits, EvalMode::Train);
    Rng fr(77 + idx, 9);
    if (cs.type == 1) type_i_feedback(bank, 1, lits, cs.s, cs.boost != 0, fr);
    else type_ii_feedback(bank, 1, lits);
    std::vector<std::uint16_t> after(bank.counters().begin(), bank.counters().end());
    std::uint64_t next_draw = fr.next();
    const std::string tag = dir + "/case" + std::to_string(idx);
    npyio::save(tag + "_x.npy", x);
    npyio::save(tag + "_before.npy", before.data(), {2, static_cast<std::size_t>(2 * cs.o)});
    npyio::save(tag + "_after.npy", after.data(), {2, static_cast<std::size_t>(2 * cs.o)});
    char line[512];
    std::snprintf(line, sizeof line,
                  "  {\"idx\": %d, \"o\": %d, \"N\": %d, \"s\": %.17g, \"boost\": %d, \"type\": %d, "
                  "\"clause_output\": %d, \"rng_seed\": %d, \"rng_stream\": 9, \"next_draw\": \"%llu\"}%s\n",
                  idx, cs.o, cs.N, cs.s, cs.boost, cs.type, out, 77 + idx,
                  static_cast<unsigned long long>(next_draw),
                  idx + 1 < static_cast<int>(sizeof cases / sizeof cases[0]) ? "," : "");
    manifest += line;
    ++idx;
  }
  manifest += "]\n";
  write_text(dir + "/manifest.json", manifest);
}

void golden_update_clause(const std::string& dir) {
  fs::create_directories(dir);
  struct Case { int o, m, n, N, q, margin; double s; int boost, use_order; long long offset, batch; int cls, j; };
  const Case cases[] = {
      {12, 2, 4, 128, 64, 15, 3.9, 0, 1, 5, 64, 0, 0},
      {12, 2, 4, 128, 64, 15, 3.9, 0, 0, 63, 150, 1, 1},
      {12, 2, 4, 128, 64, 15, 3.9, 1, 1, 0, 1, 0, 2},
      {20, 3, 6, 5, 50, 4, 2.5, 1, 1, 17, 100, 2, 3},
      {784, 10, 4, 128, 40, 50, 10.0, 0, 1, 3, 40, 7, 1},
      {70, 2, 2, 64, 130, 8, 5.0, 0, 0, 129, 260, 1, 0},
      // q < 32 with batch > q: the (offset + t) % q walk revisits examples
      // inside one 32-step window of the GPU replay
      {12, 2, 4, 128, 20, 15, 3.9, 0, 1, 7, 70, 0, 1},
      {12, 2, 4, 128, 5, 15, 3.9, 0, 0, 3, 23, 1, 0},
  };
  int idx = 0;
  std::string manifest = "[\n";
  for (const auto& cs : cases) {
    Rng r(5000 + idx, 1);
    std::vector<std::uint8_t> bits(static_cast<std::size_t>(cs.q) * cs.o);
    for (auto& b : bits) b = static_cast<std::uint8_t>(r.below(2));
    std::vector<std::int32_t> labels(static_cast<std::size_t>(cs.q));
    for (auto& y : labels) y = static_cast<std::int32_t>(r.below(static_cast<std::uint32_t>(cs.m)));
    ExamplePool pool(cs.o, bits, labels, cs.m);
    TMConfig cfg;
    cfg.clauses = cs.n;
    cfg.margin = cs.margin;
    cfg.specificity = cs.s;
    cfg.state_depth = cs.N;
    cfg.boost_true_positive = cs.boost != 0;
    MultiClassTM tm(cfg, cs.o, cs.m);
    for (auto& bank : tm.banks) {
      random_bank(bank, r, cs.o > 100 ? 0.004 : 0.08, nullptr, false);
      bank.bind_examples(cs.q);
      for (int j = 0; j < cs.n; ++j)
        for (int i = 0; i < cs.q; ++i) bank.set_prev_output(j, i, r.below(2) != 0);
    }
    for (int i = 0; i < cs.q; ++i)
      for (int c = 0; c < cs.m; ++c) pool.set_tally(i, c, static_cast<std::int32_t>(r.below(41)) - 20);
    std::vector<std::int32_t> order;
    if (cs.use_order) {
      Rng pr(31 + idx, 2);
      order = shuffled_indices(cs.q, pr);
    }
    const std::string tag = dir + "/case" + std::to_string(idx);
    npyio::save(tag + "_bits.npy", bits.data(), {static_cast<std::size_t>(cs.q), static_cast<std::size_t>(cs.o)});
    npyio::save(tag + "_labels.npy", labels);
    npyio::save(tag + "_order.npy", order);
    dump_state(dir, "case" + std::to_string(idx) + "_in", tm, pool);
    Rng ur(900 + idx, 3);
    const std::uint64_t events =
        update_clause(tm.banks[static_cast<std::size_t>(cs.cls)], cs.j, pool, cs.cls, order, cs.offset,
                      cs.batch, cs.margin, cs.s, cs.boost != 0, ur);
    const std::uint64_t next_draw = ur.next();
    dump_state(dir, "case" + std::to_string(idx) + "_out", tm, pool);
    char line[512];
    std::snprintf(line, sizeof line,
                  "  {\"idx\": %d, \"o\": %d, \"m\": %d, \"n\": %d, \"N\": %d, \"q\": %d, \"margin\": %d, "
                  "\"s\": %.17g, \"boost\": %d, \"offset\": %lld, \"batch\": %lld, \"cls\": %d, \"j\": %d, "
                  "\"rng_seed\": %d, \"rng_stream\": 3, \"events\": %llu, \"next_draw\": \"%llu\"}%s\n",
                  idx, cs.o, cs.m, cs.n, cs.N, cs.q, cs.margin, cs.s, cs.boost, cs.offset, cs.batch,
                  cs.cls, cs.j, 900 + idx, static_cast<unsigned long long>(events),
                  static_cast<unsigned long long>(next_draw),
                  idx + 1 < static_cast<int>(sizeof cases / sizeof cases[0]) ? "," : "");
    manifest += line;
    ++idx;
  }
  manifest += "]\n";
  write_text(dir + "/manifest.json", manifest);
}

struct EpochCase {
  const char* name;
  const char* data;
  int q, qt, n, margin, N, boost, epochs;
  double s;
  std::uint64_t seed, data_seed;
  double noise;
};

void golden_epochs(const std::string& root, bool sequential) {
  const EpochCase cases[] = {
      {"xor12", "xor", 100, 60, 20, 15, 128, 0, 4, 3.9, 1, 7, 0.1},
      {"mnist_small", "mnist", 100, 60, 10, 50, 128, 0, 2, 10.0, 42, 2009, 0.0},
      {"boost_n5", "xor", 50, 40, 6, 4, 5, 1, 3, 2.5, 3, 11, 0.2},
  };
  for (const auto& cs : cases) {
    const std::string dir = root + "/" + cs.name;
    fs::create_directories(dir);
    Split d = make_data(cs.data, cs.q, cs.qt, cs.data_seed, cs.noise);
    TMConfig cfg;
    cfg.clauses = cs.n;
    cfg.margin = cs.margin;
    cfg.specificity = cs.s;
    cfg.state_depth = cs.N;
    cfg.boost_true_positive = cs.boost != 0;
    cfg.seed = cs.seed;
    MultiClassTM tm(cfg, d.features, d.classes);
    ExamplePool pool(d.features, d.train_x, d.train_y, d.classes);
    ExamplePool test(d.features, d.test_x, d.test_y, d.classes);
    npyio::save(dir + "/train_x.npy", d.train_x.data(), {static_cast<std::size_t>(cs.q), static_cast<std::size_t>(d.features)});
    npyio::save(dir + "/train_y.npy", d.train_y);
    npyio::save(dir + "/test_x.npy", d.test_x.data(), {static_cast<std::size_t>(cs.qt), static_cast<std::size_t>(d.features)});
    npyio::save(dir + "/test_y.npy", d.test_y);
    std::string manifest = "{\"epochs\": [\n";
    for (int e = 0; e < cs.epochs; ++e) {
      EpochReport rep = sequential ? train_epoch_sequential(tm, pool, e) : train_epoch_parallel(tm, pool, 1, e);
      dump_state(dir, "epoch" + std::to_string(e), tm, pool);
      std::string ev;
      for (std::size_t c = 0; c < rep.feedback_events.size(); ++c)
        ev += (c ? ", " : "") + std::to_string(rep.feedback_events[c]);
      manifest += "  {\"epoch\": " + std::to_string(e) + ", \"feedback_events\": [" + ev + "]}" +
                  (e + 1 < cs.epochs ? ",\n" : "\n");
    }
    // Inference on the trained state.
    std::vector<std::int32_t> sums;
    for (int i = 0; i < test.size(); ++i) {
      auto s = export_vote_sums(tm, test.literals(i));
      sums.insert(sums.end(), s.begin(), s.end());
    }
    npyio::save(dir + "/test_sums.npy", sums.data(), {static_cast<std::size_t>(cs.qt), static_cast<std::size_t>(d.classes)});
    npyio::save(dir + "/test_pred.npy", predict_all(tm, test));
    const double acc = evaluate_accuracy(tm, test);
    // Exact refresh of the training pool's tallies / prev bits.
    if (!sequential) {
      refresh_tallies(pool, tm.banks);
      dump_state(dir, "refreshed", tm, pool);
    }
    char tail[256];
    std::snprintf(tail, sizeof tail,
                  "], \"o\": %d, \"m\": %d, \"n\": %d, \"margin\": %d, \"N\": %d, \"boost\": %d, \"s\": %.17g, "
                  "\"seed\": %llu, \"test_accuracy\": %.17g}\n",
                  d.features, d.classes, cs.n, cs.margin, cs.N, cs.boost, cs.s,
                  static_cast<unsigned long long>(cs.seed), acc);
    manifest += tail;
    write_text(dir + "/manifest.json", manifest);
  }
}

// Inference on random (untrained) states: wide masks, many included words.
void golden_inference(const std::string& dir) {
  fs::create_directories(dir);
  struct Case { const char* name; int o, m, n, q; double rate; };
  const Case cases[] = {{"mnist_rand", 784, 10, 50, 200, 0.004},
                        {"single_bank", 30, 1, 8, 64, 0.05},
                        {"dense_o64", 64, 3, 12, 128, 0.03}};
  for (const auto& cs : cases) {
    Rng r(424242, static_cast<std::uint64_t>(cs.o));
    std::vector<std::uint8_t> bits(static_cast<std::size_t>(cs.q) * cs.o);
    for (auto& b : bits) b = static_cast<std::uint8_t>(r.uniform() < 0.5);
    std::vector<std::int32_t> labels(static_cast<std::size_t>(cs.q), 0);
    ExamplePool pool(cs.o, bits, labels, cs.m);
    TMConfig cfg;
    cfg.clauses = cs.n;
    MultiClassTM tm(cfg, cs.o, cs.m);
    for (auto& bank : tm.banks) random_bank(bank, r, cs.rate, nullptr, false);
    std::vector<std::int32_t> sums;
    for (int i = 0; i < cs.q; ++i) {
      auto s = export_vote_sums(tm, pool.literals(i));
      sums.insert(sums.end(), s.begin(), s.end());
    }
    refresh_tallies(pool, tm.banks);
    const std::string tag = dir + "/" + cs.name;
    npyio::save(tag + "_bits.npy", bits.data(), {static_cast<std::size_t>(cs.q), static_cast<std::size_t>(cs.o)});
    dump_state(dir, cs.name, tm, pool);
    npyio::save(tag + "_sums.npy", sums.data(), {static_cast<std::size_t>(cs.q), static_cast<std::size_t>(cs.m)});
    npyio::save(tag + "_pred.npy", predict_all(tm, pool));
  }
}

// Regression head (f2) and tmmodel v1 text (f3).
void golden_regression(const std::string& dir) {
  fs::create_directories(dir);
  const int o = 10, q = 120, qt = 60;
  Rng r(2468, 1);
  std::vector<std::uint8_t> bits(static_cast<std::size_t>(q + qt) * o);
  std::vector<std::int32_t> y(static_cast<std::size_t>(q + qt));
  for (int i = 0; i < q + qt; ++i) {
    int ones = 0;
    for (int f = 0; f < o; ++f) {
      const auto b = static_cast<std::uint8_t>(r.below(2));
      bits[static_cast<std::size_t>(i) * o + f] = b;
      ones += b;
    }
    y[static_cast<std::size_t>(i)] = ones;
  }
  TMConfig cfg;
  cfg.clauses = 12;
  cfg.margin = 10;
  cfg.specificity = 3.0;
  cfg.state_depth = 16;
  cfg.seed = 7;
  std::vector<std::uint8_t> tx(bits.begin(), bits.begin() + q * o), vx(bits.begin() + q * o, bits.end());
  std::vector<std::int32_t> ty(y.begin(), y.begin() + q), vy(y.begin() + q, y.end());
  npyio::save(dir + "/train_x.npy", tx.data(), {static_cast<std::size_t>(q), static_cast<std::size_t>(o)});
  npyio::save(dir + "/train_y.npy", ty);
  npyio::save(dir + "/test_x.npy", vx.data(), {static_cast<std::size_t>(qt), static_cast<std::size_t>(o)});
  npyio::save(dir + "/test_y.npy", vy);
  std::string manifest = "{\n";
  for (int mode = 0; mode < 2; ++mode) {  // 0: parallel W=1, 1: sequential
    RegressionHead head(cfg, o, 0.0, 10.0);
    std::vector<std::int32_t> scaled;
    for (auto v : ty) scaled.push_back(scaled_target(head, v));
    ExamplePool pool(o, tx, scaled, 1);
    ExamplePool test(o, vx, vy, 1);
    const std::string tag = mode == 0 ? "par" : "seq";
    std::string ev;
    for (int e = 0; e < 3; ++e) {
      EpochReport rep = mode == 0 ? train_epoch_regress_parallel(head, pool, 1, e)
                                  : train_epoch_regress_sequential(head, pool, e);
      ev += (e ? ", " : "") + std::to_string(rep.total_feedback_events());
      std::vector<std::uint16_t> counters(head.bank.counters().begin(), head.bank.counters().end());
      npyio::save(dir + "/" + tag + "_epoch" + std::to_string(e) + "_counters.npy", counters.data(),
                  {static_cast<std::size_t>(cfg.clauses), static_cast<std::size_t>(2 * o)});
      if (mode == 0) {
        std::vector<std::int32_t> tallies;
        for (int i = 0; i < q; ++i) tallies.push_back(pool.tally(i, 0));
        npyio::save(dir + "/" + tag + "_epoch" + std::to_string(e) + "_tallies.npy", tallies);
        auto pb = prev_bitmap(head.bank);
        npyio::save(dir + "/" + tag + "_epoch" + std::to_string(e) + "_prev.npy", pb);
      }
    }
    std::vector<std::int32_t> pred;
    for (int i = 0; i < qt; ++i) pred.push_back(predict_scaled(head, test.literals(i)));
    npyio::save(dir + "/" + tag + "_predict_scaled.npy", pred);
    char line[256];
    std::snprintf(line, sizeof line, "\"%s_events\": [%s], \"%s_mae\": %.17g,\n", tag.c_str(), ev.c_str(), tag.c_str(),
                  evaluate_scaled_mae(head, test));
    manifest += line;
    if (mode == 1) {
      // update_regress on one row with an explicit stream
      Rng ur(99, 4);
      const auto evu = update_regress(head, test.literals(3), 7.0, ur);
      std::vector<std::uint16_t> counters(head.bank.counters().begin(), head.bank.counters().end());
      npyio::save(dir + "/update_regress_counters.npy", counters.data(),
                  {static_cast<std::size_t>(cfg.clauses), static_cast<std::size_t>(2 * o)});
      std::snprintf(line, sizeof line, "\"update_regress_events\": %llu, \"update_regress_next\": \"%llu\",\n",
                    static_cast<unsigned long long>(evu), static_cast<unsigned long long>(ur.next()));
      manifest += line;
      std::ostringstream ms;
      save_model(ms, head);
      write_text(dir + "/regress_model.txt", ms.str());
    }
  }
  manifest += "\"o\": 10, \"clauses\": 12, \"margin\": 10, \"s\": 3.0, \"N\": 16, \"seed\": 7, \"y_min\": 0.0, \"y_max\": 10.0\n}\n";
  write_text(dir + "/manifest.json", manifest);
}

// tmmodel v1 text of the W=1-trained classification machines.
void golden_models(const std::string& dir) {
  fs::create_directories(dir);
  Split d = make_data("xor", 100, 60, 7, 0.1);
  TMConfig cfg;
  cfg.clauses = 20;
  cfg.margin = 15;
  cfg.specificity = 3.9;
  cfg.seed = 1;
  MultiClassTM tm(cfg, d.features, d.classes);
  ExamplePool pool(d.features, d.train_x, d.train_y, d.classes);
  for (int e = 0; e < 4; ++e) train_epoch_parallel(tm, pool, 1, e);
  std::ostringstream ms;
  save_model(ms, tm);
  write_text(dir + "/xor12_model.txt", ms.str());
}

// ----------------------------------------------------------------- train ---

struct Args {
  std::string data = "mnist", mode = "par";
  std::int64_t q = 60000, qt = 10000, q_use = -1, qt_use = -1;
  int n = 2000, margin = 50, N = 128, boost = 0, epochs = 1, workers = 0, eval = 1, fresh = 0;
  double s = 10.0, noise = 0.0;
  std::uint64_t seed = 42, data_seed = 2009;
};

Args parse(int argc, char** argv, int start) {
  Args a;
  for (int k = start; k < argc; ++k) {
    std::string key = argv[k];
    auto val = [&]() -> std::string {
      if (k + 1 >= argc) throw std::invalid_argument("missing value for " + key);
      return argv[++k];
    };
    if (key == "--data") a.data = val();
    else if (key == "--mode") a.mode = val();
    else if (key == "--q") a.q = std::stoll(val());
    else if (key == "--qtest") a.qt = std::stoll(val());
    else if (key == "--q-use") a.q_use = std::stoll(val());
    else if (key == "--qtest-use") a.qt_use = std::stoll(val());
    else if (key == "--clauses") a.n = std::stoi(val());
    else if (key == "--T") a.margin = std::stoi(val());
    else if (key == "--s") a.s = std::stod(val());
    else if (key == "--N") a.N = std::stoi(val());
    else if (key == "--boost") a.boost = std::stoi(val());
    else if (key == "--epochs") a.epochs = std::stoi(val());
    else if (key == "--workers") a.workers = std::stoi(val());
    else if (key == "--seed") a.seed = std::stoull(val());
    else if (key == "--data-seed") a.data_seed = std::stoull(val());
    else if (key == "--noise") a.noise = std::stod(val());
    else if (key == "--eval") a.eval = std::stoi(val());
    else if (key == "--fresh") a.fresh = std::stoi(val());
    else throw std::invalid_argument("unknown flag " + key);
  }
  return a;
}

template <typename T>
std::vector<T> prefix(const std::vector<T>& v, std::size_t rows, std::size_t width) {
  return std::vector<T>(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(rows * width));
}

int cmd_train(const Args& a) {
  Split d = make_data(a.data, a.q, a.qt, a.data_seed, a.noise);
  const std::int64_t qu = a.q_use > 0 ? std::min(a.q_use, a.q) : a.q;
  const std::int64_t qtu = a.qt_use > 0 ? std::min(a.qt_use, a.qt) : a.qt;
  auto tx = prefix(d.train_x, static_cast<std::size_t>(qu), static_cast<std::size_t>(d.features));
  auto ty = prefix(d.train_y, static_cast<std::size_t>(qu), 1);
  auto vx = prefix(d.test_x, static_cast<std::size_t>(qtu), static_cast<std::size_t>(d.features));
  auto vy = prefix(d.test_y, static_cast<std::size_t>(qtu), 1);
  TMConfig cfg;
  cfg.clauses = a.n;
  cfg.margin = a.margin;
  cfg.specificity = a.s;
  cfg.state_depth = a.N;
  cfg.boost_true_positive = a.boost != 0;
  cfg.seed = a.seed;
  cfg.workers = a.workers;
  const int W = effective_workers(cfg);
  MultiClassTM tm(cfg, d.features, d.classes);
  ExamplePool pool(d.features, tx, ty, d.classes);
  std::unique_ptr<ExamplePool> test;
  if (qtu > 0) test = std::make_unique<ExamplePool>(d.features, vx, vy, d.classes);
  for (int e = 0; e < a.epochs; ++e) {
    int epoch = e;
    if (a.fresh) {  // every step = epoch 0 of a fresh machine and pool
      tm = MultiClassTM(cfg, d.features, d.classes);
      pool.reset_tallies();
      epoch = 0;
    }
    EpochReport rep = a.mode == "seq" ? train_epoch_sequential(tm, pool, epoch)
                                      : train_epoch_parallel(tm, pool, W, epoch);
    double acc = -1.0, pred_s = 0.0;
    if (a.eval && qtu > 0) {
      const auto t0 = std::chrono::steady_clock::now();
      acc = evaluate_accuracy(tm, *test);
      pred_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    std::printf(
        "{\"epoch\": %d, \"seconds\": %.6f, \"examples\": %lld, \"examples_per_s\": %.6f, "
        "\"feedback_events\": %llu, \"workers\": %d, \"test_accuracy\": %.6f, \"predict_seconds\": %.6f, "
        "\"test_rows\": %lld}\n",
        e, rep.seconds, static_cast<long long>(qu), static_cast<double>(qu) / rep.seconds,
        static_cast<unsigned long long>(rep.total_feedback_events()), W, acc, pred_s,
        static_cast<long long>(qtu));
    std::fflush(stdout);
  }
  return 0;
}

// predict <model.txt> [flags]: load a tmmodel v1 file (e.g. written by the
// GPU engine) and time the reference's single-threaded predict_all on the
// first --qtest-use rows of the synthetic test split; prints one JSON line and
// saves the predictions next to the model (<model>.ref_pred.npy).
int cmd_predict(const std::string& model_path, const Args& a) {
  AnyModel any = load_model_file(model_path);
  auto* tmp = std::get_if<MultiClassTM>(&any);
  if (!tmp) throw std::invalid_argument("predict: not a classification model");
  const MultiClassTM& tm = *tmp;
  Split d = make_data(a.data, a.q, a.qt, a.data_seed, a.noise);  // the test split follows the train rows
  const std::int64_t qtu = a.qt_use > 0 ? std::min(a.qt_use, a.qt) : a.qt;
  auto vx = prefix(d.test_x, static_cast<std::size_t>(qtu), static_cast<std::size_t>(d.features));
  auto vy = prefix(d.test_y, static_cast<std::size_t>(qtu), 1);
  ExamplePool test(d.features, vx, vy, d.classes);
  const auto t0 = std::chrono::steady_clock::now();
  const std::vector<std::int32_t> pred = predict_all(tm, test);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  npyio::save(model_path + ".ref_pred.npy", pred);
  std::int64_t hits = 0;
  for (std::int64_t i = 0; i < qtu; ++i) hits += pred[static_cast<std::size_t>(i)] == vy[static_cast<std::size_t>(i)];
  std::printf("{\"rows\": %lld, \"seconds\": %.6f, \"rows_per_s\": %.3f, \"accuracy\": %.6f, \"threads\": 1}\n",
              static_cast<long long>(qtu), secs, static_cast<double>(qtu) / secs,
              static_cast<double>(hits) / static_cast<double>(std::max<std::int64_t>(qtu, 1)));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) {
      std::fprintf(stderr, "usage: ref_driver golden <dir> | train [flags]\n");
      return 2;
    }
    const std::string cmd = argv[1];
    if (cmd == "golden") {
      const std::string dir = argc > 2 ? argv[2] : "tests/golden";
      golden_rng(dir + "/rng");
      golden_pack(dir + "/pack");
      golden_gate(dir + "/gate");
      golden_feedback(dir + "/feedback");
      golden_update_clause(dir + "/update_clause");
      golden_epochs(dir + "/epoch_par_w1", false);
      golden_epochs(dir + "/epoch_seq", true);
      golden_inference(dir + "/inference");
      golden_regression(dir + "/regression");
      golden_models(dir + "/models");
      return 0;
    }
    if (cmd == "train") return cmd_train(parse(argc, argv, 2));
    if (cmd == "predict" && argc > 2) return cmd_predict(argv[2], parse(argc, argv, 3));
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "error: %s\n", ex.what());
    return 1;
  }
}
