// api_driver.cpp — ONE source, compiled twice:
//   * against the reference (oracle/Makefile: -I/root/reference/proj/include +
//     the reference sources) -> oracle/_ref/api_driver_ref  (CPU)
//   * against the B200 drop-in (include/tsetlin/*.hpp + libtsetlin_b200.so)
//     -> paper_2009_04861_b200/_lib/api_driver_gpu           (GPU)
// It uses only the reference's public API and prints a transcript of every
// deterministic result; tests/test_gpu_dropin.py requires the two transcripts
// to be identical line for line.
#include <cstdint>
#include <cstdio>
#include <exception>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "tsetlin/feedback.hpp"
#include "tsetlin/model_io.hpp"
#include "tsetlin/pool.hpp"
#include "tsetlin/regression.hpp"
#include "tsetlin/rng.hpp"
#include "tsetlin/trainer.hpp"

using namespace tsetlin;

namespace {

std::uint64_t fnv(std::uint64_t h, std::uint64_t v) {
  for (int b = 0; b < 8; ++b) {
    h ^= (v >> (8 * b)) & 0xFF;
    h *= 1099511628211ULL;
  }
  return h;
}

std::uint64_t hash_bank(const ClassBank& bank) {
  std::uint64_t h = 1469598103934665603ULL;
  for (auto c : bank.counters()) h = fnv(h, c);
  for (int j = 0; j < bank.clause_count(); ++j) {
    h = fnv(h, static_cast<std::uint64_t>(bank.include_count(j)));
    for (auto w : bank.include_mask(j)) h = fnv(h, w);
    for (int i = 0; i < bank.bound_examples(); ++i) h = fnv(h, bank.prev_output(j, i) ? 1 : 0);
  }
  return h;
}

std::uint64_t hash_tallies(const ExamplePool& pool) {
  std::uint64_t h = 1469598103934665603ULL;
  for (int i = 0; i < pool.size(); ++i)
    for (int c = 0; c < pool.num_classes(); ++c) h = fnv(h, static_cast<std::uint32_t>(pool.tally(i, c)));
  return h;
}

void line(const std::string& key, std::uint64_t v) { std::printf("%s %llu\n", key.c_str(), static_cast<unsigned long long>(v)); }

template <typename F>
void expect_throw(const std::string& key, F&& f) {
  try {
    f();
    std::printf("%s no-throw\n", key.c_str());
  } catch (const std::invalid_argument&) {
    std::printf("%s invalid_argument\n", key.c_str());
  } catch (const std::out_of_range&) {
    std::printf("%s out_of_range\n", key.c_str());
  } catch (const std::exception&) {
    std::printf("%s other\n", key.c_str());
  }
}

struct Data {
  int o = 0;
  std::vector<std::uint8_t> x;
  std::vector<std::int32_t> y;
};

// Noisy XOR over `o` bits (y = x0 ^ x1, label noise) from a reference Rng.
Data xor_data(int rows, int o, double noise, std::uint64_t seed) {
  Rng r(seed, 0xD47A);
  Data d;
  d.o = o;
  for (int i = 0; i < rows; ++i) {
    for (int f = 0; f < o; ++f) d.x.push_back(static_cast<std::uint8_t>(r.below(2)));
    int y = d.x[static_cast<std::size_t>(i) * o] ^ d.x[static_cast<std::size_t>(i) * o + 1];
    if (r.uniform() < noise) y = 1 - y;
    d.y.push_back(y);
  }
  return d;
}

// Multi-class prototype data.
Data proto_data(int rows, int o, int m, std::uint64_t seed) {
  Rng r(seed, 0x9999);
  std::vector<std::uint8_t> protos(static_cast<std::size_t>(m) * o);
  for (auto& b : protos) b = static_cast<std::uint8_t>(r.uniform() < 0.3);
  Data d;
  d.o = o;
  for (int i = 0; i < rows; ++i) {
    const int c = static_cast<int>(r.below(static_cast<std::uint32_t>(m)));
    for (int f = 0; f < o; ++f)
      d.x.push_back(static_cast<std::uint8_t>(protos[static_cast<std::size_t>(c) * o + f] ^ (r.uniform() < 0.1)));
    d.y.push_back(c);
  }
  return d;
}

}  // namespace

int main() {
  // ---- streams
  {
    Rng r(42, 7);
    std::uint64_t h = 0;
    for (int k = 0; k < 100; ++k) h = fnv(h, r.next());
    line("rng.next", h);
    line("rng.below", r.below(1000003));
    auto perm = shuffled_indices(500, r);
    std::uint64_t hp = 0;
    for (auto v : perm) hp = fnv(hp, static_cast<std::uint64_t>(v));
    line("rng.perm", hp);
  }
  // ---- literals
  {
    const std::vector<std::uint8_t> x = {1, 0, 0, 1, 1};
    std::vector<std::uint64_t> w(static_cast<std::size_t>(literal_words(5)));
    pack_literals(x, w);
    line("pack", w[0]);
    line("literal_value", static_cast<std::uint64_t>(literal_value(x, 6)));
    expect_throw("literal_value.range", [&] { literal_value(x, 10); });
  }
  // ---- config / construction errors
  {
    TMConfig bad;
    bad.clauses = 7;
    expect_throw("config.odd", [&] { bad.validate(); });
    TMConfig bad2;
    bad2.specificity = 0.5;
    expect_throw("config.s", [&] { bad2.validate(); });
    const std::vector<std::uint8_t> bits = {0, 2};
    const std::vector<std::int32_t> labels = {0};
    expect_throw("pool.bits", [&] { ExamplePool p(2, bits, labels, 2); });
    const std::vector<std::uint8_t> bits2 = {0, 1};
    const std::vector<std::int32_t> labels2 = {3};
    expect_throw("pool.label", [&] { ExamplePool p(2, bits2, labels2, 2); });
  }
  // ---- asynchronous trainer, one worker (deterministic), XOR
  Data xd = xor_data(300, 12, 0.1, 5);
  Data xt = xor_data(200, 12, 0.0, 6);
  TMConfig cfg;
  cfg.clauses = 20;
  cfg.margin = 15;
  cfg.specificity = 3.9;
  cfg.seed = 11;
  MultiClassTM tm(cfg, 12, 2);
  ExamplePool pool(12, xd.x, xd.y, 2);
  ExamplePool test(12, xt.x, xt.y, 2);
  for (int e = 0; e < 3; ++e) {
    auto rep = train_epoch_parallel(tm, pool, 1, e);
    line("par.e" + std::to_string(e) + ".events", rep.total_feedback_events());
    for (int c = 0; c < 2; ++c) line("par.e" + std::to_string(e) + ".bank" + std::to_string(c), hash_bank(tm.banks[c]));
    line("par.e" + std::to_string(e) + ".tallies", hash_tallies(pool));
  }
  {
    auto pred = predict_all(tm, test);
    std::uint64_t h = 0;
    for (auto v : pred) h = fnv(h, static_cast<std::uint64_t>(v));
    line("predict_all", h);
    line("accuracy_x1e6", static_cast<std::uint64_t>(evaluate_accuracy(tm, test) * 1e6 + 0.5));
    std::uint64_t hs = 0;
    for (int i = 0; i < test.size(); ++i)
      for (auto s : export_vote_sums(tm, test.literals(i))) hs = fnv(hs, static_cast<std::uint32_t>(s));
    line("export_vote_sums", hs);
    line("classify.7", static_cast<std::uint64_t>(classify(tm, test.literals(7))));
    line("vote_sum.train", static_cast<std::uint32_t>(vote_sum(tm.banks[1], test.literals(3), EvalMode::Train)));
    line("vote_sum.predict", static_cast<std::uint32_t>(vote_sum(tm.banks[1], test.literals(3), EvalMode::Predict)));
    line("evaluate_clause", static_cast<std::uint64_t>(evaluate_clause(tm.banks[0], 4, test.literals(9), EvalMode::Predict)));
  }
  // ---- copy semantics: training a copy leaves the original untouched
  {
    const std::uint64_t before = hash_bank(tm.banks[0]);
    MultiClassTM copy = tm;
    train_epoch_parallel(copy, pool, 1, 7);
    line("copy.original_unchanged", hash_bank(tm.banks[0]) == before ? 1 : 0);
    line("copy.trained", hash_bank(copy.banks[0]));
  }
  // ---- refresh_tallies
  refresh_tallies(pool, tm.banks);
  line("refresh.tallies", hash_tallies(pool));
  line("refresh.bank0", hash_bank(tm.banks[0]));
  // ---- update_clause with an explicit stream, natural and shuffled order
  {
    Rng r(77, 3);
    const auto ev1 = update_clause(tm.banks[1], 3, pool, 1, {}, 17, 450, 15, 3.9, false, r);
    line("update_clause.natural.events", ev1);
    Rng pr(5, 2);
    const auto order = shuffled_indices(pool.size(), pr);
    const auto ev2 = update_clause(tm.banks[0], 6, pool, 0, order, 299, 300, 9, 2.5, true, r);
    line("update_clause.order.events", ev2);
    line("update_clause.next_draw", r.next());
    line("update_clause.bank0", hash_bank(tm.banks[0]));
    line("update_clause.bank1", hash_bank(tm.banks[1]));
    line("update_clause.tallies", hash_tallies(pool));
    expect_throw("update_clause.batch", [&] { update_clause(tm.banks[0], 0, pool, 0, {}, 0, 0, 15, 3.9, false, r); });
  }
  // ---- record_output_and_tally
  {
    const int t_before = pool.tally(5, 1);
    const bool prev = tm.banks[1].prev_output(2, 5);
    record_output_and_tally(pool, 5, 1, tm.banks[1], 2, prev ? 0 : 1);
    line("record.tally_delta", static_cast<std::uint32_t>(pool.tally(5, 1) - t_before));
    line("record.bit", tm.banks[1].prev_output(2, 5) ? 1 : 0);
    expect_throw("record.range", [&] { record_output_and_tally(pool, 9999, 1, tm.banks[1], 2, 1); });
  }
  // ---- feedback on a standalone bank
  {
    ClassBank bank(12, 4, 16);
    Rng r(3, 3);
    for (int j = 0; j < 4; ++j)
      for (int k = 0; k < 24; ++k) bank.set_counter(j, k, static_cast<StateCounter>(1 + r.below(32)));
    bank.reinforce(0, 0, Reinforcement::Penalty);
    bank.reinforce(1, 5, Reinforcement::Reward);
    line("bank.set_counter", hash_bank(bank));
    const auto lits = test.literals(11);
    type_i_feedback(bank, 1, lits, 3.9, false, r);
    type_i_feedback(bank, 2, lits, 2.0, true, r);
    type_ii_feedback(bank, 3, lits);
    detail::type_i_with_output(bank, 0, lits, 1, 3.0, false, r);
    detail::type_ii_with_output(bank, 1, lits, 1);
    line("bank.feedback", hash_bank(bank));
    line("bank.next_draw", r.next());
    line("bank.eval", static_cast<std::uint64_t>(evaluate_clause(bank, 2, lits, EvalMode::Train)));
    ClassBank copy = bank;
    copy.set_counter(0, 0, 32);
    line("bank.copy_independent", hash_bank(bank) != hash_bank(copy) ? 1 : 0);
    auto cs = bank.mutable_counters();
    for (auto& c : cs) c = static_cast<StateCounter>(c % 16 + 9);
    bank.rebuild_masks();
    line("bank.rebuilt", hash_bank(bank));
  }
  // ---- classic sequential trainer on 4 classes (deterministic)
  {
    Data pd = proto_data(150, 20, 4, 9);
    TMConfig c2;
    c2.clauses = 10;
    c2.margin = 8;
    c2.specificity = 3.0;
    c2.state_depth = 8;
    c2.seed = 5;
    MultiClassTM tm2(c2, 20, 4);
    ExamplePool p2(20, pd.x, pd.y, 4);
    for (int e = 0; e < 2; ++e) {
      auto rep = train_epoch_sequential(tm2, p2, e);
      line("seq.e" + std::to_string(e) + ".events", rep.total_feedback_events());
      for (int c = 0; c < 4; ++c) line("seq.e" + std::to_string(e) + ".bank" + std::to_string(c), hash_bank(tm2.banks[c]));
    }
    line("seq.accuracy_x1e6", static_cast<std::uint64_t>(evaluate_accuracy(tm2, p2) * 1e6 + 0.5));
    auto r1 = train_epoch_parallel(tm2, p2, 1, 2);
    line("seq.par_after", r1.total_feedback_events());
    line("seq.par_bank3", hash_bank(tm2.banks[3]));
    // ---- model files (tmmodel v1): identical text, and a load round trip
    std::ostringstream ms;
    save_model(ms, tm2);
    std::uint64_t ht = 1469598103934665603ULL;
    for (char ch : ms.str()) ht = fnv(ht, static_cast<unsigned char>(ch));
    line("model.text", ht);
    std::istringstream is(ms.str());
    AnyModel back = load_model(is);
    line("model.load_bank2", hash_bank(std::get<MultiClassTM>(back).banks[2]) == hash_bank(tm2.banks[2]) ? 1 : 0);
    std::istringstream junk("tmmodel v2");
    expect_throw("model.bad", [&] { load_model(junk); });
  }
  // ---- regression head: sequential, one-worker parallel, update, predict
  {
    Rng r(1357, 2);
    const int o = 10, q = 80;
    std::vector<std::uint8_t> bits;
    std::vector<std::int32_t> ys;
    for (int i = 0; i < q; ++i) {
      int ones = 0;
      for (int f = 0; f < o; ++f) {
        bits.push_back(static_cast<std::uint8_t>(r.below(2)));
        ones += bits.back();
      }
      ys.push_back(ones);
    }
    TMConfig rc;
    rc.clauses = 8;
    rc.margin = 10;
    rc.specificity = 2.5;
    rc.state_depth = 32;
    rc.seed = 3;
    RegressionHead head(rc, o, 0.0, 10.0);
    std::vector<std::int32_t> scaled;
    for (auto y : ys) scaled.push_back(scaled_target(head, y));
    ExamplePool rp(o, bits, scaled, 1);
    for (int e = 0; e < 2; ++e) line("regress.seq.e" + std::to_string(e), train_epoch_regress_sequential(head, rp, e).total_feedback_events());
    line("regress.seq.bank", hash_bank(head.bank));
    RegressionHead head2 = head;  // value copy: continues independently
    for (int e = 0; e < 2; ++e) line("regress.par.e" + std::to_string(e), train_epoch_regress_parallel(head2, rp, 1, e).total_feedback_events());
    line("regress.par.bank", hash_bank(head2.bank));
    line("regress.par.tallies", hash_tallies(rp));
    line("regress.mae_x1e6", static_cast<std::uint64_t>(evaluate_scaled_mae(head2, rp) * 1e6 + 0.5));
    line("regress.predict_scaled", static_cast<std::uint64_t>(predict_scaled(head2, rp.literals(5))));
    line("regress.predict_x1e6", static_cast<std::uint64_t>(predict_regress(head2, rp.literals(6)) * 1e6 + 0.5));
    Rng ur(8, 8);
    line("regress.update", update_regress(head, rp.literals(9), 4.0, ur));
    line("regress.update_next", ur.next());
    line("regress.update_bank", hash_bank(head.bank));
    expect_throw("regress.range", [&] { scaled_target(head, 11.0); });
    std::ostringstream ms;
    save_model(ms, head);
    std::uint64_t ht = 1469598103934665603ULL;
    for (char ch : ms.str()) ht = fnv(ht, static_cast<unsigned char>(ch));
    line("regress.model_text", ht);
  }
  return 0;
}
