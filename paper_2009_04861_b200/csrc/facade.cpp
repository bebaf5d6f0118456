// facade.cpp — the reference's C++ API (namespace tsetlin) implemented over
// the B200 C ABI (tmgpu.h). Host mirrors are synchronised lazily; all
// learning and evaluation calls go to libtmgpu.so.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "tsetlin_b200.hpp"

namespace tsetlin {

namespace {

void check(int rc) {
  if (rc == TMG_OK) return;
  const std::string msg = tmg_last_error();
  if (rc == TMG_EINVAL) throw std::invalid_argument(msg);
  if (rc == TMG_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

int default_device() {
  const char* env = std::getenv("TSETLIN_DEVICES");
  if (env && *env) return std::atoi(env);  // the first listed device holds the pools
  env = std::getenv("TSETLIN_DEVICE");
  return env ? std::atoi(env) : 0;
}

// $TSETLIN_DEVICES="0,1,2,3": every MultiClassTM spans these GPUs (clause
// shards, tmg_machine_create_devices); unset or one entry: one GPU.
std::vector<std::int32_t> machine_devices() {
  std::vector<std::int32_t> out;
  const char* env = std::getenv("TSETLIN_DEVICES");
  for (const char* p = env; p && *p;) {
    char* end = nullptr;
    const long v = std::strtol(p, &end, 10);
    if (end == p) throw std::invalid_argument("TSETLIN_DEVICES: expected a comma-separated device list");
    out.push_back(static_cast<std::int32_t>(v));
    p = *end == ',' ? end + 1 : end;
    if (*end && *end != ',') throw std::invalid_argument("TSETLIN_DEVICES: expected a comma-separated device list");
  }
  if (out.empty()) out.push_back(default_device());
  return out;
}

tmg_machine* create_multiclass(const tmg_config& cc, int o, int m) {
  const std::vector<std::int32_t> devs = machine_devices();
  tmg_machine* h = nullptr;
  check(tmg_machine_create_devices(&cc, o, m, devs.data(), static_cast<std::int32_t>(devs.size()), &h));
  return h;
}

tmg_config to_c(const TMConfig& c) {
  tmg_config out{};
  out.clauses = c.clauses;
  out.margin = c.margin;
  out.specificity = c.specificity;
  out.state_depth = c.state_depth;
  out.boost_true_positive = c.boost_true_positive ? 1 : 0;
  out.epochs = c.epochs;
  out.workers = c.workers;
  out.seed = c.seed;
  return out;
}

}  // namespace

namespace detail {

struct DeviceMachine {
  tmg_machine* h = nullptr;
  int device = 0;
  std::vector<ClassBank::Link*> links;  // bank index -> host mirror
  ~DeviceMachine() {
    if (h) tmg_machine_destroy(h);
  }
};

struct DevicePool {
  tmg_pool* h = nullptr;
  std::vector<std::int32_t> tallies;  // host mirror, q x m
  bool host_stale = false, dirty = false;
  ~DevicePool() {
    if (h) tmg_pool_destroy(h);
  }
};

}  // namespace detail

// Host mirror of one bank + its place on a device machine.
struct ClassBank::Link {
  std::shared_ptr<detail::DeviceMachine> dev;
  int bank = 0;
  std::vector<StateCounter> counters;
  std::vector<std::uint64_t> masks;
  std::vector<std::int32_t> counts;
  std::vector<std::uint64_t> prev;
  int bound = 0;
  bool host_stale = false;      // device holds newer state
  bool counters_dirty = false;  // host counters newer than device
  bool prev_dirty = false;      // host previous outputs newer than device
};

namespace {

using Link = ClassBank::Link;

void download(const ClassBank& b, Link& l) {
  if (!l.host_stale) return;
  auto& dm = *l.dev;
  check(tmg_get_counters(dm.h, l.bank, l.counters.data()));
  check(tmg_get_include_masks(dm.h, l.bank, l.masks.data()));
  check(tmg_get_include_counts(dm.h, l.bank, l.counts.data()));
  int64_t bound = 0;
  check(tmg_bank_bound_examples(dm.h, l.bank, &bound));
  l.bound = static_cast<int>(bound);
  l.prev.assign(static_cast<std::size_t>(b.clause_count()) * ((l.bound + 63) / 64), 0);
  if (!l.prev.empty()) check(tmg_get_prev_outputs(dm.h, l.bank, l.prev.data()));
  l.host_stale = false;
}

void make_device_cfg(const ClassBank& b, Link& l, const TMConfig& cfg);

void make_device(const ClassBank& b, Link& l) {
  if (l.dev) return;
  TMConfig cfg;
  cfg.clauses = b.clause_count();
  cfg.state_depth = b.state_depth();
  make_device_cfg(b, l, cfg);
}

void make_device_cfg(const ClassBank& b, Link& l, const TMConfig& cfg) {
  if (l.dev) return;
  const tmg_config cc = to_c(cfg);
  auto dm = std::make_shared<detail::DeviceMachine>();
  dm->device = default_device();
  if (b.scheme() == PolarityScheme::AllPositive)  // the regression head's bank
    check(tmg_machine_create_regress(&cc, b.feature_count(), dm->device, &dm->h));
  else
    check(tmg_machine_create(&cc, b.feature_count(), 1, dm->device, &dm->h));
  dm->links.push_back(&l);
  l.dev = dm;
  l.bank = 0;
  l.counters_dirty = true;
  l.prev_dirty = l.bound > 0;
}

// Pushes every dirty bank mirror of the machine to the device.
void push_machine(detail::DeviceMachine& dm, const std::vector<const ClassBank*>& banks) {
  for (std::size_t k = 0; k < dm.links.size(); ++k) {
    Link* l = dm.links[k];
    (void)banks;
    if (l->counters_dirty) {
      check(tmg_set_counters(dm.h, l->bank, l->counters.data()));
      l->counters_dirty = false;
    }
    if (l->prev_dirty) {  // bind_examples is per bank (core.cpp:117-126): only this bank is rebound
      int64_t bound = 0;
      check(tmg_bank_bound_examples(dm.h, l->bank, &bound));
      if (bound != l->bound) check(tmg_bind_bank(dm.h, l->bank, l->bound));
      if (!l->prev.empty()) check(tmg_set_prev_outputs(dm.h, l->bank, l->prev.data()));
      l->prev_dirty = false;
    }
  }
}

void mark_stale(detail::DeviceMachine& dm) {
  for (auto* l : dm.links) l->host_stale = true;
}

detail::DeviceMachine& device_of(const ClassBank& b) {
  make_device(b, *b.link_);
  push_machine(*b.link_->dev, {});
  return *b.link_->dev;
}

detail::DeviceMachine& device_of(const MultiClassTM& tm) {
  auto& dm = *tm.banks.front().link_->dev;
  push_machine(dm, {});
  return dm;
}


void push_pool(const ExamplePool& pool) {
  auto* dp = pool.device();
  if (dp->dirty) {
    check(tmg_pool_set_tallies(dp->h, dp->tallies.data()));
    dp->dirty = false;
  }
}

void pool_changed(const ExamplePool& pool) { pool.device()->host_stale = true; }

void check_compatible(const MultiClassTM& tm, const ExamplePool& pool) {  // trainer.cpp:46-53
  if (tm.feature_count() != pool.feature_count()) throw std::invalid_argument("model/pool feature count mismatch");
  if (tm.num_banks() != pool.num_classes()) throw std::invalid_argument("model/pool class count mismatch");
}

}  // namespace

// ================================================================== core ==

int literal_value(std::span<const std::uint8_t> x, int k) {  // core.cpp:24-32
  const int o = static_cast<int>(x.size());
  if (k < 0 || k >= 2 * o)
    throw std::out_of_range("literal index " + std::to_string(k) + " outside [0, " + std::to_string(2 * o) + ")");
  const int f = k < o ? k : k - o;
  const int v = x[static_cast<std::size_t>(f)] ? 1 : 0;
  return k < o ? v : 1 - v;
}

void pack_literals(std::span<const std::uint8_t> x, std::span<std::uint64_t> words) {  // core.cpp:34-46
  const int o = static_cast<int>(x.size());
  std::memset(words.data(), 0, words.size_bytes());
  for (int f = 0; f < o; ++f) {
    const int k = x[static_cast<std::size_t>(f)] ? f : o + f;
    words[static_cast<std::size_t>(k) / 64] |= std::uint64_t{1} << (k % 64);
  }
}

void TMConfig::validate() const {
  const tmg_config c = to_c(*this);
  check(tmg_config_validate(&c));
}

int effective_workers(const TMConfig& config) {  // core.cpp:76-80 (0 = hardware)
  if (config.workers > 0) return config.workers;
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? static_cast<int>(hw) : 1;
}

ClassBank::ClassBank(int feature_count, int clause_count, int state_depth, PolarityScheme scheme)
    : o_(feature_count), n_(clause_count), N_(state_depth), scheme_(scheme) {
  if (feature_count < 1) throw std::invalid_argument("feature count must be >= 1");
  if (clause_count < 0) throw std::invalid_argument("clause count must be >= 0");
  link_ = std::make_shared<Link>();
  link_->counters.assign(static_cast<std::size_t>(n_) * 2 * o_, static_cast<StateCounter>(N_));
  link_->masks.assign(static_cast<std::size_t>(n_) * literal_words(o_), 0);
  link_->counts.assign(static_cast<std::size_t>(n_), 0);
}

ClassBank::ClassBank(const ClassBank& other)
    : o_(other.o_), n_(other.n_), N_(other.N_), scheme_(other.scheme_) {
  if (other.link_->dev) download(other, *other.link_);
  link_ = std::make_shared<Link>();
  link_->counters = other.link_->counters;
  link_->masks = other.link_->masks;
  link_->counts = other.link_->counts;
  link_->prev = other.link_->prev;
  link_->bound = other.link_->bound;
}

ClassBank& ClassBank::operator=(const ClassBank& other) {
  if (this != &other) {
    ClassBank tmp(other);
    *this = std::move(tmp);
  }
  return *this;
}

ClassBank::~ClassBank() {
  if (link_ && link_->dev) {
    auto& v = link_->dev->links;
    for (auto& p : v)
      if (p == link_.get()) p = nullptr;
    std::erase(v, nullptr);
  }
}

namespace {
Link& host(const ClassBank& b) {
  Link& l = *b.link_;
  if (l.dev) download(b, l);
  return l;
}
}  // namespace

StateCounter ClassBank::counter(int j, int k) const {
  return host(*this).counters[static_cast<std::size_t>(j) * 2 * o_ + static_cast<std::size_t>(k)];
}

void ClassBank::set_counter(int j, int k, StateCounter value) {  // core.cpp:107-115
  Link& l = host(*this);
  const std::size_t idx = static_cast<std::size_t>(j) * 2 * o_ + static_cast<std::size_t>(k);
  const bool was = l.counters[idx] > N_;
  l.counters[idx] = value;
  const bool now = value > N_;
  if (was != now) {
    l.masks[static_cast<std::size_t>(j) * literal_words(o_) + static_cast<std::size_t>(k) / 64] ^=
        std::uint64_t{1} << (k % 64);
    l.counts[static_cast<std::size_t>(j)] += now ? 1 : -1;
  }
  l.counters_dirty = true;
}

void ClassBank::reinforce(int j, int k, Reinforcement event) {  // core.hpp:134-145
  const StateCounter before = counter(j, k);
  const StateCounter after = apply_transition(before, event, N_);
  if (after != before) set_counter(j, k, after);
}

int ClassBank::include_count(int j) const { return host(*this).counts[static_cast<std::size_t>(j)]; }

std::span<const std::uint64_t> ClassBank::include_mask(int j) const {
  const Link& l = host(*this);
  return {l.masks.data() + static_cast<std::size_t>(j) * literal_words(o_),
          static_cast<std::size_t>(literal_words(o_))};
}

void ClassBank::bind_examples(int example_count) {  // core.cpp:117-126
  if (example_count < 0) throw std::invalid_argument("example count must be >= 0");
  Link& l = host(*this);
  l.bound = example_count;
  l.prev.assign(static_cast<std::size_t>(n_) * ((example_count + 63) / 64), 0);
  l.prev_dirty = true;
}

int ClassBank::bound_examples() const { return host(*this).bound; }

bool ClassBank::prev_output(int j, int i) const {
  const Link& l = host(*this);
  const std::size_t w = static_cast<std::size_t>(j) * ((l.bound + 63) / 64) + static_cast<std::size_t>(i) / 64;
  return (l.prev[w] >> (i % 64)) & 1u;
}

void ClassBank::set_prev_output(int j, int i, bool bit) {
  Link& l = host(*this);
  const std::size_t w = static_cast<std::size_t>(j) * ((l.bound + 63) / 64) + static_cast<std::size_t>(i) / 64;
  const std::uint64_t mask = std::uint64_t{1} << (i % 64);
  l.prev[w] = bit ? (l.prev[w] | mask) : (l.prev[w] & ~mask);
  l.prev_dirty = true;
}

std::span<const StateCounter> ClassBank::counters() const { return host(*this).counters; }

std::span<StateCounter> ClassBank::mutable_counters() {
  Link& l = host(*this);
  l.counters_dirty = true;  // the device re-derives masks from the counters
  return l.counters;
}

void ClassBank::rebuild_masks() {  // core.cpp:128-139
  Link& l = host(*this);
  const int W = literal_words(o_);
  std::fill(l.masks.begin(), l.masks.end(), 0);
  std::fill(l.counts.begin(), l.counts.end(), 0);
  for (int j = 0; j < n_; ++j)
    for (int k = 0; k < 2 * o_; ++k)
      if (l.counters[static_cast<std::size_t>(j) * 2 * o_ + static_cast<std::size_t>(k)] > N_) {
        l.masks[static_cast<std::size_t>(j) * W + static_cast<std::size_t>(k) / 64] |= std::uint64_t{1} << (k % 64);
        ++l.counts[static_cast<std::size_t>(j)];
      }
  l.counters_dirty = true;
}

int evaluate_clause(const ClassBank& bank, int j, std::span<const std::uint64_t> literals, EvalMode mode) {
  auto& dm = device_of(bank);
  std::int32_t out = 0;
  check(tmg_evaluate_clause(dm.h, bank.link_->bank, j, literals.data(),
                            mode == EvalMode::Train ? TMG_EVAL_TRAIN : TMG_EVAL_PREDICT, &out));
  return out;
}

// ================================================================== pool ==

ExamplePool::ExamplePool(int feature_count, std::span<const std::uint8_t> bits,
                         std::span<const std::int32_t> labels, int num_classes)
    : size_(static_cast<int>(labels.size())), o_(feature_count), m_(num_classes) {
  // pool.cpp:29-41 (shape checks; value checks happen in tmg_pool_create)
  if (feature_count < 1) throw std::invalid_argument("feature count must be >= 1");
  if (num_classes < 1) throw std::invalid_argument("class count must be >= 1");
  if (labels.empty()) throw std::invalid_argument("example pool must not be empty");
  if (bits.size() != static_cast<std::size_t>(size_) * static_cast<std::size_t>(o_))
    throw std::invalid_argument("bit matrix size does not match labels");
  dev_ = std::make_unique<detail::DevicePool>();
  check(tmg_pool_create(default_device(), o_, bits.data(), labels.data(), size_, m_, &dev_->h));
  literals_.resize(static_cast<std::size_t>(size_) * literal_words(o_));
  check(tmg_pool_get_literals(dev_->h, literals_.data()));
  labels_.assign(labels.begin(), labels.end());
  dev_->tallies.assign(static_cast<std::size_t>(size_) * m_, 0);
}

ExamplePool::ExamplePool(ExamplePool&&) noexcept = default;
ExamplePool& ExamplePool::operator=(ExamplePool&&) noexcept = default;
ExamplePool::~ExamplePool() = default;

namespace {
std::vector<std::int32_t>& tallies_host(const ExamplePool& p) {
  auto* dp = p.device();
  if (dp->host_stale) {
    check(tmg_pool_get_tallies(dp->h, dp->tallies.data()));
    dp->host_stale = false;
  }
  return dp->tallies;
}
}  // namespace

std::int32_t ExamplePool::tally(int i, int c) const {
  return tallies_host(*this)[static_cast<std::size_t>(i) * m_ + static_cast<std::size_t>(c)];
}

void ExamplePool::add_to_tally(int i, int c, std::int32_t delta) {
  tallies_host(*this)[static_cast<std::size_t>(i) * m_ + static_cast<std::size_t>(c)] += delta;
  dev_->dirty = true;
}

void ExamplePool::set_tally(int i, int c, std::int32_t value) {
  tallies_host(*this)[static_cast<std::size_t>(i) * m_ + static_cast<std::size_t>(c)] = value;
  dev_->dirty = true;
}

void ExamplePool::reset_tallies() {
  check(tmg_pool_reset_tallies(dev_->h));
  std::fill(dev_->tallies.begin(), dev_->tallies.end(), 0);
  dev_->host_stale = false;
  dev_->dirty = false;
}

int vote_sum(const ClassBank& bank, std::span<const std::uint64_t> literals, EvalMode mode) {
  auto& dm = device_of(bank);
  tmg_machine_info info{};
  check(tmg_machine_info_get(dm.h, &info));
  std::vector<std::int32_t> sums(static_cast<std::size_t>(info.num_classes));
  check(tmg_class_sums_literals(dm.h, literals.data(), 1, mode == EvalMode::Train ? TMG_EVAL_TRAIN : TMG_EVAL_PREDICT,
                                sums.data()));
  return sums[static_cast<std::size_t>(bank.link_->bank)];
}

void record_output_and_tally(ExamplePool& pool, int i, int class_idx, ClassBank& bank, int j, int output) {
  // pool.cpp:93-106 — a single-cell bookkeeping edit of two host-visible
  // structures (tally and previous-output bit), applied to their mirrors.
  if (i < 0 || i >= pool.size() || class_idx < 0 || class_idx >= pool.num_classes())
    throw std::out_of_range("record_output_and_tally: index out of range");
  const bool previous = bank.prev_output(j, i);
  const bool current = output != 0;
  if (previous == current) return;
  std::int32_t delta = current ? 1 : -1;
  if (!bank.positive(j)) delta = -delta;
  pool.add_to_tally(i, class_idx, delta);
  bank.set_prev_output(j, i, current);
}

void refresh_tallies(ExamplePool& pool, std::span<ClassBank> banks) {  // pool.cpp:108-124
  if (banks.empty()) return;
  auto& dm = device_of(banks.front());
  if (static_cast<int>(banks.size()) != static_cast<int>(dm.links.size()))
    throw std::invalid_argument("refresh_tallies expects all banks of one machine");
  push_pool(pool);
  check(tmg_refresh_tallies(dm.h, pool.device()->h));
  mark_stale(dm);
  pool_changed(pool);
}

// ============================================================== feedback ==

double clause_update_probability(int v, int y, int margin) {  // feedback.cpp:24-28
  const int clipped = v < -margin ? -margin : (v > margin ? margin : v);
  const int error = y == 1 ? margin - clipped : margin + clipped;
  return static_cast<double>(error) / (2.0 * static_cast<double>(margin));
}

namespace {
void feedback(ClassBank& bank, int j, std::span<const std::uint64_t> literals, int type, int out, double s,
              bool boost, Rng* rng) {
  auto& dm = device_of(bank);
  std::uint64_t dummy[4] = {0, 0, 0, 0};
  check(tmg_feedback(dm.h, bank.link_->bank, j, literals.data(), type, s, boost ? 1 : 0, out,
                     rng ? rng->raw_state() : dummy));
  bank.link_->host_stale = true;
}
}  // namespace

void type_i_feedback(ClassBank& bank, int j, std::span<const std::uint64_t> literals, double s,
                     bool boost_true_positive, Rng& rng) {
  feedback(bank, j, literals, 1, -1, s, boost_true_positive, &rng);
}

void type_ii_feedback(ClassBank& bank, int j, std::span<const std::uint64_t> literals) {
  feedback(bank, j, literals, 2, -1, 1.0, false, nullptr);
}

namespace detail {
void type_i_with_output(ClassBank& bank, int j, std::span<const std::uint64_t> literals, int clause_output,
                        double s, bool boost_true_positive, Rng& rng) {
  feedback(bank, j, literals, 1, clause_output ? 1 : 0, s, boost_true_positive, &rng);
}
void type_ii_with_output(ClassBank& bank, int j, std::span<const std::uint64_t> literals, int clause_output) {
  feedback(bank, j, literals, 2, clause_output ? 1 : 0, 1.0, false, nullptr);
}
}  // namespace detail

// =============================================================== trainer ==

MultiClassTM::MultiClassTM(TMConfig cfg, int feature_count, int num_classes) : config(cfg) {
  config.validate();
  if (num_classes < 1) throw std::invalid_argument("class count must be >= 1");
  auto dm = std::make_shared<detail::DeviceMachine>();
  dm->device = default_device();
  const tmg_config cc = to_c(config);
  dm->h = create_multiclass(cc, feature_count, num_classes);
  banks.reserve(static_cast<std::size_t>(num_classes));
  for (int c = 0; c < num_classes; ++c) {
    banks.emplace_back(feature_count, config.clauses, config.state_depth, PolarityScheme::Alternating);
    Link& l = *banks.back().link_;
    l.dev = dm;
    l.bank = c;
    dm->links.push_back(&l);
  }
}

MultiClassTM::MultiClassTM(const MultiClassTM& other) : config(other.config) {
  auto dm = std::make_shared<detail::DeviceMachine>();
  dm->device = default_device();
  const tmg_config cc = to_c(config);
  dm->h = create_multiclass(cc, other.feature_count(), other.num_banks());
  banks.reserve(other.banks.size());
  for (int c = 0; c < other.num_banks(); ++c) {
    const ClassBank& src = other.banks[static_cast<std::size_t>(c)];
    banks.emplace_back(src.feature_count(), src.clause_count(), src.state_depth(), src.scheme());
    Link& l = *banks.back().link_;
    const Link& s = host(src);
    l.counters = s.counters;
    l.masks = s.masks;
    l.counts = s.counts;
    l.prev = s.prev;
    l.bound = s.bound;
    l.dev = dm;
    l.bank = c;
    l.counters_dirty = true;
    l.prev_dirty = s.bound > 0;
    dm->links.push_back(&l);
  }
}

MultiClassTM& MultiClassTM::operator=(const MultiClassTM& other) {
  if (this != &other) {
    MultiClassTM tmp(other);
    *this = std::move(tmp);
  }
  return *this;
}

std::uint64_t update_clause(ClassBank& bank, int j, ExamplePool& pool, int class_idx,
                            std::span<const std::int32_t> order, std::int64_t offset, std::int64_t batch, int margin,
                            double s, bool boost_true_positive, Rng& rng) {
  auto& dm = device_of(bank);
  // The engine keys the tally column and the target on the bank's own class
  // (as every reference caller does, trainer.cpp:220); a different class_idx
  // is rejected instead of silently ignored (tsetlin.py does the same).
  if (class_idx != bank.link_->bank)
    throw std::invalid_argument("update_clause: class_idx must be the bank's own class index");
  push_pool(pool);
  std::uint64_t events = 0;
  check(tmg_update_clause(dm.h, pool.device()->h, bank.link_->bank, j, order.empty() ? nullptr : order.data(),
                          static_cast<std::int64_t>(order.size()), offset, batch, margin, s,
                          boost_true_positive ? 1 : 0, rng.raw_state(), &events));
  mark_stale(dm);
  pool_changed(pool);
  return events;
}

EpochReport train_epoch_sequential(MultiClassTM& tm, const ExamplePool& pool, int epoch) {
  check_compatible(tm, pool);
  if (tm.num_banks() < 2) throw std::invalid_argument("classification needs at least two banks");
  auto& dm = device_of(tm);
  EpochReport rep;
  rep.epoch = epoch;
  rep.feedback_events.assign(static_cast<std::size_t>(tm.num_banks()), 0);
  double seconds = 0.0;
  check(tmg_train_epoch_sequential(dm.h, pool.device()->h, epoch, &seconds, rep.feedback_events.data()));
  rep.seconds = seconds > 0 ? seconds : 1e-9;
  mark_stale(dm);
  return rep;
}

EpochReport train_epoch_parallel(MultiClassTM& tm, ExamplePool& pool, int workers, int epoch) {
  check_compatible(tm, pool);
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  auto& dm = device_of(tm);
  push_pool(pool);
  EpochReport rep;
  rep.epoch = epoch;
  rep.feedback_events.assign(static_cast<std::size_t>(tm.num_banks()), 0);
  tmg_epoch_report r{};
  r.feedback_events = rep.feedback_events.data();
  // TMG_MODE_AUTO: asynchronous for every `workers`; TSETLIN_DETERMINISTIC=1
  // with workers == 1 selects the bit-exact single-worker replay.
  check(tmg_train_epoch(dm.h, pool.device()->h, TMG_MODE_AUTO, workers, epoch, &r));
  rep.seconds = r.seconds;
  mark_stale(dm);
  pool_changed(pool);
  return rep;
}

int classify(const MultiClassTM& tm, std::span<const std::uint64_t> literals) {
  auto& dm = device_of(tm);
  std::int32_t out = 0;
  check(tmg_predict_literals(dm.h, literals.data(), 1, &out));
  return out;
}

std::vector<std::int32_t> export_vote_sums(const MultiClassTM& tm, std::span<const std::uint64_t> literals) {
  auto& dm = device_of(tm);
  std::vector<std::int32_t> sums(static_cast<std::size_t>(tm.num_banks()));
  check(tmg_class_sums_literals(dm.h, literals.data(), 1, TMG_EVAL_PREDICT, sums.data()));
  return sums;
}

std::vector<std::int32_t> predict_all(const MultiClassTM& tm, const ExamplePool& pool) {
  auto& dm = device_of(tm);
  std::vector<std::int32_t> out(static_cast<std::size_t>(pool.size()));
  check(tmg_predict(dm.h, pool.device()->h, out.data()));
  return out;
}

double evaluate_accuracy(const MultiClassTM& tm, const ExamplePool& pool) {
  const auto pred = predict_all(tm, pool);
  int correct = 0;
  for (int i = 0; i < pool.size(); ++i)
    if (pred[static_cast<std::size_t>(i)] == pool.label(i)) ++correct;
  return static_cast<double>(correct) / static_cast<double>(pool.size());
}

// ============================================================ regression ==

RegressionHead::RegressionHead(TMConfig cfg, int feature_count, double lo, double hi)
    : config(cfg), y_min(lo), y_max(hi),
      bank(feature_count, cfg.clauses, cfg.state_depth, PolarityScheme::AllPositive) {
  config.validate();  // regression.cpp:69-80
  if (!(y_max > y_min)) throw std::invalid_argument("target range must satisfy y_max > y_min");
  make_device_cfg(bank, *bank.link_, config);
}

namespace {
// The head's device machine carries its configuration (T, s, seed, boost).
detail::DeviceMachine& head_device(const RegressionHead& head) {
  make_device_cfg(head.bank, *head.bank.link_, head.config);
  push_machine(*head.bank.link_->dev, {});
  return *head.bank.link_->dev;
}
}  // namespace

int scaled_target(const RegressionHead& head, double y) {  // regression.cpp:82-89
  if (y < head.y_min || y > head.y_max) throw std::invalid_argument("target outside [y_min, y_max]");
  const double span = head.y_max - head.y_min;
  return static_cast<int>(std::lround((y - head.y_min) * head.config.margin / span));
}

int predict_scaled(const RegressionHead& head, std::span<const std::uint64_t> literals) {
  auto& dm = head_device(head);
  std::int32_t out = 0;
  check(tmg_regress_predict_literals(dm.h, literals.data(), 1, &out));
  return out;
}

double predict_regress(const RegressionHead& head, std::span<const std::uint64_t> literals) {
  const int v = predict_scaled(head, literals);
  return head.y_min + v * (head.y_max - head.y_min) / head.config.margin;
}

std::uint64_t update_regress(RegressionHead& head, std::span<const std::uint64_t> literals, double y_target,
                             Rng& rng) {
  const int t = scaled_target(head, y_target);
  auto& dm = head_device(head);
  std::uint64_t events = 0;
  check(tmg_update_regress(dm.h, literals.data(), t, rng.raw_state(), &events));
  mark_stale(dm);
  return events;
}

EpochReport train_epoch_regress_sequential(RegressionHead& head, const ExamplePool& pool, int epoch) {
  if (pool.feature_count() != head.bank.feature_count())
    throw std::invalid_argument("head/pool feature count mismatch");
  auto& dm = head_device(head);
  EpochReport rep;
  rep.epoch = epoch;
  rep.feedback_events.assign(1, 0);
  double seconds = 0.0;
  check(tmg_train_epoch_regress_sequential(dm.h, pool.device()->h, epoch, &seconds, rep.feedback_events.data()));
  rep.seconds = seconds > 0 ? seconds : 1e-9;
  mark_stale(dm);
  return rep;
}

EpochReport train_epoch_regress_parallel(RegressionHead& head, ExamplePool& pool, int workers, int epoch) {
  if (pool.feature_count() != head.bank.feature_count())
    throw std::invalid_argument("head/pool feature count mismatch");
  if (pool.num_classes() != 1) throw std::invalid_argument("regression pool must have one tally class");
  if (workers < 1) throw std::invalid_argument("workers must be >= 1");
  auto& dm = head_device(head);
  push_pool(pool);
  EpochReport rep;
  rep.epoch = epoch;
  rep.feedback_events.assign(1, 0);
  tmg_epoch_report r{};
  r.feedback_events = rep.feedback_events.data();
  check(tmg_train_epoch_regress(dm.h, pool.device()->h, TMG_MODE_AUTO, workers, epoch, &r));
  rep.seconds = r.seconds;
  mark_stale(dm);
  pool_changed(pool);
  return rep;
}

double evaluate_scaled_mae(const RegressionHead& head, const ExamplePool& pool) {  // regression.cpp:229-236
  auto& dm = head_device(head);
  std::vector<std::int32_t> pred(static_cast<std::size_t>(pool.size()));
  check(tmg_regress_predict(dm.h, pool.device()->h, pred.data()));
  double total = 0.0;
  for (int i = 0; i < pool.size(); ++i) total += std::abs(static_cast<double>(pred[static_cast<std::size_t>(i)] - pool.label(i)));
  return total / static_cast<double>(pool.size());
}

}  // namespace tsetlin
