// tsetlin_b200.hpp — C++ drop-in facade of the reference API (namespace
// `tsetlin`, /root/reference/proj/include/tsetlin/*.hpp) over the B200 C ABI
// (tmgpu.h). The reference's own headers are replaced by the forwarding
// headers include/tsetlin/{core,rng,feedback,pool,trainer}.hpp, so code
// written against the reference compiles unchanged with
//     -I<repo>/include  and links  -ltsetlin_b200 -ltmgpu
//
// Model: every MultiClassTM / ExamplePool lives on one GPU (device 0, or
// $TSETLIN_DEVICE). Accessors that expose host memory (counters(),
// include_mask(), literals(), tally(), ...) read lazily synchronised host
// mirrors; mutators write the mirror and the next device operation pushes it.
// All learning and evaluation runs on the GPU — there is no host compute path.
//
// Semantic notes:
//   * train_epoch_parallel(workers == 1) replays the reference schedule
//     bit-exactly (sync-mirror kernel); workers > 1 runs Algorithm 1 over all
//     clauses concurrently (the asynchronous GPU kernel), which, like the
//     reference's multi-threaded trainer, is not bit-reproducible.
//   * PolarityScheme::AllPositive banks are the regression head's
//     (RegressionHead, regression.cpp) and run on the device's regression
//     kernels (tmg_machine_create_regress).
#pragma once

#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tmgpu.h"
#include "tmgpu_rng.h"

namespace tsetlin {

// =============================================================== streams ==
// rng.hpp:26-103 — the same xoshiro256++/splitmix64 streams (tmgpu_rng.h).

inline std::uint64_t split_mix64(std::uint64_t& state) { return tmg_splitmix64(&state); }

class Rng {
 public:
  using result_type = std::uint64_t;
  explicit Rng(std::uint64_t seed, std::uint64_t stream = 0) { tmg_rng_seed(&r_, seed, stream); }
  std::uint64_t next() { return tmg_rng_next(&r_); }
  result_type operator()() { return next(); }
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return std::numeric_limits<result_type>::max(); }
  double uniform() { return tmg_rng_uniform(&r_); }
  bool bernoulli(double p) { return uniform() < p; }
  std::uint32_t below(std::uint32_t bound) { return tmg_rng_below(&r_, bound); }
  // Facade extension: the 4-word state handed to the GPU mirror kernels.
  std::uint64_t* raw_state() { return r_.s; }

 private:
  tmg_rng r_;
};

template <typename T>
void shuffle_span(std::span<T> values, Rng& rng) {
  for (std::size_t i = values.size(); i > 1; --i) {
    const std::size_t j = rng.below(static_cast<std::uint32_t>(i));
    T tmp = values[i - 1];
    values[i - 1] = values[j];
    values[j] = tmp;
  }
}

inline std::vector<std::int32_t> shuffled_indices(std::int32_t count, Rng& rng) {
  std::vector<std::int32_t> order(static_cast<std::size_t>(count));
  tmg_shuffled_indices(count, reinterpret_cast<tmg_rng*>(rng.raw_state()), order.data());
  return order;
}

// ================================================================== core ==
enum class Action : std::uint8_t { Exclude, Include };
enum class Reinforcement : std::uint8_t { Inaction, Reward, Penalty };
enum class EvalMode : std::uint8_t { Train, Predict };
using StateCounter = std::uint16_t;

// core.hpp:42-65 — scalar helpers of the automaton model (host utilities; the
// GPU applies the same clamped +-1 moves to bit-sliced planes).
inline Action ta_action(StateCounter counter, int state_depth) {
  return counter > state_depth ? Action::Include : Action::Exclude;
}
inline StateCounter apply_transition(StateCounter counter, Reinforcement event, int state_depth) {
  if (event == Reinforcement::Inaction) return counter;
  const bool include = counter > state_depth;
  const bool up = (event == Reinforcement::Reward) == include;
  int next = static_cast<int>(counter) + (up ? 1 : -1);
  next = next < 1 ? 1 : (next > 2 * state_depth ? 2 * state_depth : next);
  return static_cast<StateCounter>(next);
}

int literal_value(std::span<const std::uint8_t> x, int k);
constexpr int literal_words(int feature_count) { return (2 * feature_count + 63) / 64; }
void pack_literals(std::span<const std::uint8_t> x, std::span<std::uint64_t> words);
inline bool literal_bit(std::span<const std::uint64_t> words, int k) {
  return ((words[static_cast<std::size_t>(k) / 64] >> (k % 64)) & 1u) != 0;
}

struct TMConfig {
  int clauses = 100;
  int margin = 15;
  double specificity = 3.0;
  int state_depth = 128;
  bool boost_true_positive = false;
  int epochs = 100;
  int workers = 0;
  std::uint64_t seed = 42;
  void validate() const;
};
int effective_workers(const TMConfig& config);

enum class PolarityScheme : std::uint8_t { Alternating, AllPositive };

namespace detail {
struct DeviceMachine;  // owns a tmg_machine*
struct DevicePool;     // owns a tmg_pool*
}  // namespace detail

class ExamplePool;

class ClassBank {
 public:
  ClassBank(int feature_count, int clause_count, int state_depth,
            PolarityScheme scheme = PolarityScheme::Alternating);
  ClassBank(const ClassBank& other);  // deep copy (value semantics, like the reference)
  ClassBank& operator=(const ClassBank& other);
  ClassBank(ClassBank&&) noexcept = default;
  ClassBank& operator=(ClassBank&&) noexcept = default;
  ~ClassBank();

  int feature_count() const { return o_; }
  int literal_count() const { return 2 * o_; }
  int clause_count() const { return n_; }
  int state_depth() const { return N_; }
  int words_per_clause() const { return literal_words(o_); }
  PolarityScheme scheme() const { return scheme_; }
  bool positive(int j) const { return scheme_ == PolarityScheme::AllPositive || j % 2 == 0; }

  StateCounter counter(int j, int k) const;
  Action action(int j, int k) const { return ta_action(counter(j, k), N_); }
  void set_counter(int j, int k, StateCounter value);
  void reinforce(int j, int k, Reinforcement event);
  int include_count(int j) const;
  std::span<const std::uint64_t> include_mask(int j) const;

  void bind_examples(int example_count);
  int bound_examples() const;
  bool prev_output(int j, int i) const;
  void set_prev_output(int j, int i, bool bit);

  std::span<const StateCounter> counters() const;
  std::span<StateCounter> mutable_counters();
  void rebuild_masks();

  // ---- facade internals (device link) ----
  struct Link;
  std::shared_ptr<Link> link_;

 private:
  int o_, n_, N_;
  PolarityScheme scheme_;
};

// Evaluated on the GPU (core.hpp:208-219).
int evaluate_clause(const ClassBank& bank, int j, std::span<const std::uint64_t> literals, EvalMode mode);

// ================================================================== pool ==
class ExamplePool {
 public:
  ExamplePool(int feature_count, std::span<const std::uint8_t> bits, std::span<const std::int32_t> labels,
              int num_classes);
  ExamplePool(const ExamplePool&) = delete;
  ExamplePool& operator=(const ExamplePool&) = delete;
  ExamplePool(ExamplePool&&) noexcept;
  ExamplePool& operator=(ExamplePool&&) noexcept;
  ~ExamplePool();

  int size() const { return size_; }
  int feature_count() const { return o_; }
  int num_classes() const { return m_; }
  int words_per_example() const { return literal_words(o_); }
  std::span<const std::uint64_t> literals(int i) const {
    return {literals_.data() + static_cast<std::size_t>(i) * words_per_example(),
            static_cast<std::size_t>(words_per_example())};
  }
  std::int32_t label(int i) const { return labels_[static_cast<std::size_t>(i)]; }
  std::uint8_t feature(int i, int f) const { return static_cast<std::uint8_t>(literal_bit(literals(i), f)); }
  std::int32_t tally(int i, int c) const;
  void add_to_tally(int i, int c, std::int32_t delta);
  void set_tally(int i, int c, std::int32_t value);
  void reset_tallies();

  // ---- facade internals ----
  detail::DevicePool* device() const { return dev_.get(); }

 private:
  int size_ = 0, o_ = 0, m_ = 0;
  std::vector<std::uint64_t> literals_;
  std::vector<std::int32_t> labels_;
  std::unique_ptr<detail::DevicePool> dev_;
};

int vote_sum(const ClassBank& bank, std::span<const std::uint64_t> literals, EvalMode mode);
void record_output_and_tally(ExamplePool& pool, int i, int class_idx, ClassBank& bank, int j, int output);
void refresh_tallies(ExamplePool& pool, std::span<ClassBank> banks);

// ============================================================== feedback ==
double clause_update_probability(int vote_sum, int y, int margin);
void type_i_feedback(ClassBank& bank, int j, std::span<const std::uint64_t> literals, double s,
                     bool boost_true_positive, Rng& rng);
void type_ii_feedback(ClassBank& bank, int j, std::span<const std::uint64_t> literals);
namespace detail {
void type_i_with_output(ClassBank& bank, int j, std::span<const std::uint64_t> literals, int clause_output,
                        double s, bool boost_true_positive, Rng& rng);
void type_ii_with_output(ClassBank& bank, int j, std::span<const std::uint64_t> literals, int clause_output);
}  // namespace detail

// =============================================================== trainer ==
struct EpochReport {
  int epoch = 0;
  double seconds = 0.0;
  std::vector<std::uint64_t> feedback_events;
  std::optional<double> train_metric;
  std::optional<double> test_metric;
  std::uint64_t total_feedback_events() const {
    std::uint64_t t = 0;
    for (auto v : feedback_events) t += v;
    return t;
  }
};

struct MultiClassTM {
  TMConfig config;
  std::vector<ClassBank> banks;

  MultiClassTM(TMConfig cfg, int feature_count, int num_classes);
  MultiClassTM(const MultiClassTM& other);
  MultiClassTM& operator=(const MultiClassTM& other);
  MultiClassTM(MultiClassTM&&) noexcept = default;
  MultiClassTM& operator=(MultiClassTM&&) noexcept = default;

  int feature_count() const { return banks.front().feature_count(); }
  int num_banks() const { return static_cast<int>(banks.size()); }
};

std::uint64_t update_clause(ClassBank& bank, int j, ExamplePool& pool, int class_idx,
                            std::span<const std::int32_t> order, std::int64_t offset, std::int64_t batch,
                            int margin, double s, bool boost_true_positive, Rng& rng);
EpochReport train_epoch_sequential(MultiClassTM& tm, const ExamplePool& pool, int epoch);
EpochReport train_epoch_parallel(MultiClassTM& tm, ExamplePool& pool, int workers, int epoch);
int classify(const MultiClassTM& tm, std::span<const std::uint64_t> literals);
std::vector<std::int32_t> export_vote_sums(const MultiClassTM& tm, std::span<const std::uint64_t> literals);
std::vector<std::int32_t> predict_all(const MultiClassTM& tm, const ExamplePool& pool);
double evaluate_accuracy(const MultiClassTM& tm, const ExamplePool& pool);

// ============================================================ regression ==
// regression.hpp: one all-positive bank; the clipped clause count decodes
// linearly into [y_min, y_max].
struct RegressionHead {
  TMConfig config;
  double y_min;
  double y_max;
  ClassBank bank;

  RegressionHead(TMConfig cfg, int feature_count, double y_min, double y_max);
};

int scaled_target(const RegressionHead& head, double y);
int predict_scaled(const RegressionHead& head, std::span<const std::uint64_t> literals);
double predict_regress(const RegressionHead& head, std::span<const std::uint64_t> literals);
std::uint64_t update_regress(RegressionHead& head, std::span<const std::uint64_t> literals, double y_target,
                             Rng& rng);
EpochReport train_epoch_regress_sequential(RegressionHead& head, const ExamplePool& pool, int epoch);
EpochReport train_epoch_regress_parallel(RegressionHead& head, ExamplePool& pool, int workers, int epoch);
double evaluate_scaled_mae(const RegressionHead& head, const ExamplePool& pool);

}  // namespace tsetlin
