// facade_cli.cpp — the `tm` command line (train / eval / bench / synth) of the
// reference (proj/src/cli.cpp:35-538, proj/tools/tm_main.cpp:19) for the B200
// drop-in: same subcommands, flags, defaults, stdout lines, report/bench CSV
// and exit codes (0 ok, 2 missing input file, 1 any other error; a command
// line that does not parse exits with the CLI11 ExitCodes value of the
// reference's parser, cli.cpp:512-516).
//
// The reference parses with CLI11, which is not vendored (cli.cpp:27); this
// file carries its own small parser and is written ONLY against the
// reference's public headers (tsetlin/{trainer,regression,model_io,data_io,
// metrics,bench}.hpp), so the same source links against the reference
// library (oracle/Makefile -> oracle/_ref/tm_ref) and against the GPU facade
// (csrc/Makefile -> _lib/tm). tests/test_gpu_dropin.py requires the two
// binaries to print the same transcript for the deterministic modes.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "tsetlin/bench.hpp"
#include "tsetlin/cli.hpp"
#include "tsetlin/data_io.hpp"
#include "tsetlin/metrics.hpp"
#include "tsetlin/model_io.hpp"
#include "tsetlin/regression.hpp"
#include "tsetlin/trainer.hpp"

namespace tsetlin {

namespace {

// CLI11's ExitCodes for the parse failures the reference's command line can
// produce (CLI11 is un-vendored, version unpinned; these values are stable
// across its 1.x/2.x releases).
enum ParseExit : int {
  kConversionError = 104,
  kValidationError = 105,
  kRequiredError = 106,
  kExtrasError = 109,
};

struct ParseFailure : std::runtime_error {
  int code;
  ParseFailure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct MissingInput : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void need_file(const std::string& path) {
  if (!std::filesystem::exists(path)) throw MissingInput("no such file: " + path);
}

// TM_THREADS overrides --workers when it is a positive integer (cli.cpp:49-59).
int workers_from_env(int flag_value) {
  const char* env = std::getenv("TM_THREADS");
  if (env == nullptr) return flag_value;
  char* end = nullptr;
  const long v = std::strtol(env, &end, 10);
  if (end != env && *end == '\0' && v >= 1) return static_cast<int>(v);
  std::cerr << "warning: ignoring invalid TM_THREADS value '" << env << "'\n";
  return flag_value;
}

// Option values with the reference's defaults (cli.cpp:61-89).
struct Options {
  TMConfig config;
  std::string mode = "seq", task = "classify";
  std::string data, test, synth;
  int synth_train = 1000, synth_test = 200, synth_features = 6, synth_classes = 4, synth_zone = 5;
  double noise = 0.0;
  int binarize_bits = 8;
  double train_fraction = 0.8;
  std::string out, report, binarizer_out, binarizer_in, model;
  bool per_epoch = false;
  std::vector<int> bench_clauses;
  std::string bench_mode = "both";
  int bench_warmup = 1, bench_epochs = 3;
};

// ------------------------------------------------------------------ parser --
struct Flag {
  enum Kind { Int, U64, Real, Text, Switch, IntList } kind;
  std::string name;
  void* target;
  std::vector<std::string> choices;  // empty = any value
  bool required = false;
  bool seen = false;
};

class Command {
 public:
  explicit Command(std::string name) : name_(std::move(name)) {}
  const std::string& name() const { return name_; }
  Flag& add(Flag::Kind k, const std::string& n, void* t, std::vector<std::string> choices = {}) {
    flags_.push_back(Flag{k, n, t, std::move(choices)});
    return flags_.back();
  }

  void parse(const std::vector<std::string>& args, std::size_t first) {
    for (std::size_t a = first; a < args.size(); ++a) {
      std::string key = args[a], value;
      bool inline_value = false;
      if (key.rfind("--", 0) != 0) throw ParseFailure(kExtrasError, "The following arguments were not expected: " + key);
      if (const auto eq = key.find('='); eq != std::string::npos) {
        value = key.substr(eq + 1);
        key = key.substr(0, eq);
        inline_value = true;
      }
      Flag* f = find(key);
      if (f == nullptr) throw ParseFailure(kExtrasError, "The following arguments were not expected: " + args[a]);
      f->seen = true;
      if (f->kind == Flag::Switch) {
        if (inline_value) throw ParseFailure(kExtrasError, key + ": flag takes no value");
        *static_cast<bool*>(f->target) = true;
        continue;
      }
      if (!inline_value) {
        if (a + 1 >= args.size()) throw ParseFailure(kExtrasError, key + " requires an argument");
        value = args[++a];
      }
      store(*f, value);
      // list options also take the following bare words (CLI11 vector options)
      while (f->kind == Flag::IntList && !inline_value && a + 1 < args.size() && args[a + 1].rfind("--", 0) != 0)
        store(*f, args[++a]);
    }
    for (const auto& f : flags_)
      if (f.required && !f.seen) throw ParseFailure(kRequiredError, f.name + " is required");
  }

 private:
  Flag* find(const std::string& key) {
    for (auto& f : flags_)
      if (f.name == key) return &f;
    return nullptr;
  }

  static long long to_integer(const Flag& f, const std::string& v) {
    std::size_t used = 0;
    long long x = 0;
    try {
      x = std::stoll(v, &used);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used == 0 || used != v.size()) throw ParseFailure(kConversionError, f.name + ": cannot convert '" + v + "'");
    return x;
  }

  static void store(Flag& f, const std::string& v) {
    if (!f.choices.empty() && std::find(f.choices.begin(), f.choices.end(), v) == f.choices.end())
      throw ParseFailure(kValidationError, f.name + ": '" + v + "' not in the allowed set");
    switch (f.kind) {
      case Flag::Int: {
        const long long x = to_integer(f, v);
        if (x < INT32_MIN || x > INT32_MAX) throw ParseFailure(kConversionError, f.name + ": out of range");
        *static_cast<int*>(f.target) = static_cast<int>(x);
        break;
      }
      case Flag::U64: {
        std::size_t used = 0;
        unsigned long long x = 0;
        try {
          if (!v.empty() && v[0] != '-') x = std::stoull(v, &used);
        } catch (const std::exception&) {
          used = 0;
        }
        if (used == 0 || used != v.size()) throw ParseFailure(kConversionError, f.name + ": cannot convert '" + v + "'");
        *static_cast<std::uint64_t*>(f.target) = x;
        break;
      }
      case Flag::Real: {
        std::size_t used = 0;
        double x = 0;
        try {
          x = std::stod(v, &used);
        } catch (const std::exception&) {
          used = 0;
        }
        if (used == 0 || used != v.size()) throw ParseFailure(kConversionError, f.name + ": cannot convert '" + v + "'");
        *static_cast<double*>(f.target) = x;
        break;
      }
      case Flag::Text:
        *static_cast<std::string*>(f.target) = v;
        break;
      case Flag::IntList: {
        auto& list = *static_cast<std::vector<int>*>(f.target);
        std::stringstream parts(v);
        for (std::string item; std::getline(parts, item, ',');) {
          const long long x = to_integer(f, item);
          if (x < INT32_MIN || x > INT32_MAX) throw ParseFailure(kConversionError, f.name + ": out of range");
          list.push_back(static_cast<int>(x));
        }
        break;
      }
      case Flag::Switch:
        break;
    }
  }

  std::string name_;
  std::vector<Flag> flags_;
};

void model_flags(Command& c, Options& o, bool clause_count) {
  if (clause_count) c.add(Flag::Int, "--clauses", &o.config.clauses);
  c.add(Flag::Int, "--margin", &o.config.margin);
  c.add(Flag::Real, "--specificity", &o.config.specificity);
  c.add(Flag::Int, "--states", &o.config.state_depth);
  c.add(Flag::Switch, "--boost", &o.config.boost_true_positive);
  c.add(Flag::Int, "--epochs", &o.config.epochs);
  c.add(Flag::Int, "--workers", &o.config.workers);
  c.add(Flag::U64, "--seed", &o.config.seed);
  c.add(Flag::Text, "--mode", &o.mode, {"seq", "par"});
  c.add(Flag::Text, "--task", &o.task, {"classify", "regress"});
  c.add(Flag::Int, "--binarize-bits", &o.binarize_bits);
}

void data_flags(Command& c, Options& o) {
  c.add(Flag::Text, "--data", &o.data);
  c.add(Flag::Text, "--test", &o.test);
  c.add(Flag::Text, "--synth", &o.synth);
  c.add(Flag::Int, "--synth-train", &o.synth_train);
  c.add(Flag::Int, "--synth-test", &o.synth_test);
  c.add(Flag::Int, "--synth-features", &o.synth_features);
  c.add(Flag::Int, "--classes", &o.synth_classes);
  c.add(Flag::Int, "--zone", &o.synth_zone);
  c.add(Flag::Real, "--noise", &o.noise);
  c.add(Flag::Real, "--train-fraction", &o.train_fraction);
}

// ------------------------------------------------------------------- tasks --
SynthSplit make_synth(const Options& o) {
  if (o.synth == "xor") return synth_xor(o.synth_train, o.synth_test, o.noise, o.config.seed);
  if (o.synth == "patterns")
    return synth_patterns(o.synth_train, o.synth_test, o.synth_classes, o.synth_zone, o.noise, o.config.seed);
  if (o.synth == "staircase") return synth_staircase(o.synth_train, o.synth_test, o.synth_features, o.config.seed);
  throw std::invalid_argument("unknown synthetic dataset '" + o.synth + "'");
}

bool csv_path(const std::string& p) { return p.size() >= 4 && p.compare(p.size() - 4, 4, ".csv") == 0; }

// Training input: a synthetic split, a CSV split by row order with a
// binarizer fitted on the train rows, or dense binary files (cli.cpp:103-175).
struct Task {
  Dataset train;
  std::optional<Dataset> test;
  std::vector<double> train_y, test_y;  // real targets (regression)
  std::optional<BinarizerSpec> binarizer;
};

Task load_task(const Options& o) {
  Task t;
  if (!o.synth.empty()) {
    SynthSplit s = make_synth(o);
    t.train = std::move(s.train);
    t.test = std::move(s.test);
  } else if (!o.data.empty()) {
    need_file(o.data);
    if (csv_path(o.data)) {
      const RawDataset raw = load_csv(o.data);
      const int rows = raw.rows();
      const long wanted = std::lround(rows * o.train_fraction);
      const int n_train = std::max(1, std::min(rows - 1, static_cast<int>(wanted)));
      std::vector<std::int32_t> tr, te;
      for (int r = 0; r < rows; ++r) (r < n_train ? tr : te).push_back(r);
      const BinarizerSpec spec = fit_binarizer(raw, o.binarize_bits, tr);
      t.binarizer = spec;
      Dataset test;
      t.train.feature_count = test.feature_count = spec.output_width();
      t.train.x = apply_binarizer(spec, raw, tr);
      test.x = apply_binarizer(spec, raw, te);
      for (const auto r : tr) {
        t.train_y.push_back(raw.label(r));
        t.train.y.push_back(static_cast<std::int32_t>(std::lround(raw.label(r))));
      }
      for (const auto r : te) {
        t.test_y.push_back(raw.label(r));
        test.y.push_back(static_cast<std::int32_t>(std::lround(raw.label(r))));
      }
      if (!test.y.empty()) t.test = std::move(test);
    } else {
      t.train = load_dense_binary(o.data);
      if (!o.test.empty()) {
        need_file(o.test);
        t.test = load_dense_binary(o.test);
      }
    }
  } else {
    throw std::invalid_argument("pass --data FILE or --synth NAME");
  }
  if (t.train_y.empty()) {
    t.train_y.assign(t.train.y.begin(), t.train.y.end());
    if (t.test) t.test_y.assign(t.test->y.begin(), t.test->y.end());
  }
  if (!o.test.empty() && !o.synth.empty()) throw std::invalid_argument("--test cannot be combined with --synth");
  return t;
}

void report_row(std::ostream& out, const Options& o, int workers, int epoch, double seconds, const char* metric,
                double value) {
  out << o.mode << ',' << (o.mode == "par" ? workers : 1) << ',' << o.config.clauses << ',' << epoch << ','
      << seconds << ',' << metric << ',' << value << '\n';
}

double regress_mae(const RegressionHead& head, const ExamplePool& pool, const std::vector<double>& y) {
  double total = 0.0;
  for (int i = 0; i < pool.size(); ++i)
    total += std::abs(predict_regress(head, pool.literals(i)) - y[static_cast<std::size_t>(i)]);
  return total / static_cast<double>(pool.size());
}

int train_classify(const Options& o, const TMConfig& cfg, const Task& t, int workers, std::ofstream& report) {
  int classes = 2;
  for (const auto y : t.train.y) classes = std::max(classes, y + 1);
  if (t.test)
    for (const auto y : t.test->y) classes = std::max(classes, y + 1);
  MultiClassTM tm(cfg, t.train.feature_count, classes);
  ExamplePool train(t.train.feature_count, t.train.x, t.train.y, classes);
  std::optional<ExamplePool> test;
  if (t.test) test.emplace(t.test->feature_count, t.test->x, t.test->y, classes);

  for (int e = 0; e < cfg.epochs; ++e) {
    const EpochReport r =
        o.mode == "par" ? train_epoch_parallel(tm, train, workers, e) : train_epoch_sequential(tm, train, e);
    if (!o.per_epoch && !report.is_open()) continue;
    const double acc = evaluate_accuracy(tm, train);
    if (o.per_epoch) std::cout << "epoch " << e << " seconds " << r.seconds << " train_accuracy " << acc << '\n';
    if (report.is_open()) {
      report_row(report, o, workers, e, r.seconds, "train_accuracy", acc);
      if (test) report_row(report, o, workers, e, r.seconds, "test_accuracy", evaluate_accuracy(tm, *test));
    }
  }
  std::cout << "train_accuracy " << evaluate_accuracy(tm, train) << '\n';
  if (test) {
    const ClassificationMetrics m = classification_metrics(predict_all(tm, *test), t.test->y);
    std::cout << "test_accuracy " << m.accuracy << '\n';
    std::cout << "test_macro_f1 " << m.macro_f1 << '\n';
  }
  if (!o.out.empty()) {
    save_model_file(o.out, tm);
    std::cout << "model " << o.out << '\n';
  }
  return 0;
}

int train_regress(const Options& o, const TMConfig& cfg, const Task& t, int workers, std::ofstream& report) {
  const auto [lo, hi] = std::minmax_element(t.train_y.begin(), t.train_y.end());
  RegressionHead head(cfg, t.train.feature_count, *lo, *hi);
  std::vector<std::int32_t> scaled;
  scaled.reserve(t.train_y.size());
  for (const double y : t.train_y) scaled.push_back(scaled_target(head, y));
  ExamplePool train(t.train.feature_count, t.train.x, scaled, 1);
  std::optional<ExamplePool> test;
  if (t.test) {
    const std::vector<std::int32_t> zeros(t.test->y.size(), 0);
    test.emplace(t.test->feature_count, t.test->x, zeros, 1);
  }
  for (int e = 0; e < cfg.epochs; ++e) {
    const EpochReport r = o.mode == "par" ? train_epoch_regress_parallel(head, train, workers, e)
                                          : train_epoch_regress_sequential(head, train, e);
    if (o.per_epoch) std::cout << "epoch " << e << " seconds " << r.seconds << '\n';
    if (report.is_open() && test) report_row(report, o, workers, e, r.seconds, "test_mae", regress_mae(head, *test, t.test_y));
  }
  std::cout << "train_mae " << regress_mae(head, train, t.train_y) << '\n';
  if (test) std::cout << "test_mae " << regress_mae(head, *test, t.test_y) << '\n';
  if (!o.out.empty()) {
    save_model_file(o.out, head);
    std::cout << "model " << o.out << '\n';
  }
  return 0;
}

int run_train(const Options& o) {
  TMConfig cfg = o.config;
  cfg.workers = workers_from_env(cfg.workers);
  cfg.validate();
  const Task t = load_task(o);
  const int workers = effective_workers(cfg);
  std::ofstream report;
  if (!o.report.empty()) {
    report.open(o.report);
    if (!report) throw std::runtime_error("cannot write report: " + o.report);
    report << "mode,workers,clauses,epoch,seconds,metric_name,metric_value\n";
  }
  if (o.task == "classify")
    train_classify(o, cfg, t, workers, report);
  else if (o.task == "regress")
    train_regress(o, cfg, t, workers, report);
  else
    throw std::invalid_argument("task must be classify or regress");
  if (!o.binarizer_out.empty()) {
    if (!t.binarizer) throw std::invalid_argument("--binarizer-out needs CSV input");
    std::ofstream out(o.binarizer_out);
    if (!out) throw std::runtime_error("cannot write binarizer: " + o.binarizer_out);
    save_binarizer(out, *t.binarizer);
  }
  return 0;
}

int run_eval(const Options& o) {
  need_file(o.model);
  const AnyModel model = load_model_file(o.model);
  need_file(o.data);
  Dataset data;
  std::vector<double> targets;
  if (csv_path(o.data)) {
    if (o.binarizer_in.empty()) throw std::invalid_argument("CSV eval needs --binarizer FILE");
    need_file(o.binarizer_in);
    std::ifstream in(o.binarizer_in);
    const BinarizerSpec spec = load_binarizer(in);
    const RawDataset raw = load_csv(o.data);
    data.feature_count = spec.output_width();
    data.x = apply_binarizer(spec, raw);
    for (int r = 0; r < raw.rows(); ++r) {
      targets.push_back(raw.label(r));
      data.y.push_back(static_cast<std::int32_t>(std::lround(raw.label(r))));
    }
  } else {
    data = load_dense_binary(o.data);
    targets.assign(data.y.begin(), data.y.end());
  }
  if (const auto* tm = std::get_if<MultiClassTM>(&model)) {
    const ExamplePool pool(data.feature_count, data.x, data.y, tm->num_banks());
    const ClassificationMetrics m = classification_metrics(predict_all(*tm, pool), data.y);
    std::cout << "accuracy " << m.accuracy << '\n';
    std::cout << "macro_f1 " << m.macro_f1 << '\n';
  } else {
    const auto& head = std::get<RegressionHead>(model);
    const std::vector<std::int32_t> zeros(data.y.size(), 0);
    const ExamplePool pool(data.feature_count, data.x, zeros, 1);
    std::cout << "mae " << regress_mae(head, pool, targets) << '\n';
  }
  return 0;
}

int run_bench(const Options& o) {
  TMConfig cfg = o.config;
  cfg.workers = workers_from_env(cfg.workers);
  cfg.validate();
  if (o.bench_clauses.empty()) throw std::invalid_argument("bench needs --clauses LIST");
  const Task t = load_task(o);
  if (!t.test) throw std::invalid_argument("bench needs a test split");
  BenchOptions b;
  b.clause_counts = o.bench_clauses;
  b.modes = o.bench_mode == "both" ? std::vector<std::string>{"seq", "par"} : std::vector<std::string>{o.bench_mode};
  b.warmup_epochs = o.bench_warmup;
  b.measured_epochs = o.bench_epochs;
  b.workers = cfg.workers;
  b.regression = o.task == "regress";
  const auto records = bench_sweep(t.train, *t.test, cfg, b);
  if (o.out.empty()) {
    write_bench_csv(std::cout, records);
    return 0;
  }
  std::ofstream out(o.out);
  if (!out) throw std::runtime_error("cannot write CSV: " + o.out);
  write_bench_csv(out, records);
  std::cout << "csv " << o.out << '\n';
  return 0;
}

int run_synth(const Options& o) {
  if (o.out.empty()) throw std::invalid_argument("synth needs --out PREFIX");
  const SynthSplit s = make_synth(o);
  save_dense_binary(o.out + ".train", s.train);
  save_dense_binary(o.out + ".test", s.test);
  std::cout << "train " << o.out << ".train\n";
  std::cout << "test " << o.out << ".test\n";
  return 0;
}

const char* kUsage =
    "Tsetlin machine training, inference and benchmarks\n"
    "usage: tm {train|eval|bench|synth} [--flag value ...]\n";

}  // namespace

int run_cli(const std::vector<std::string>& args) {
  Options o;
  Command train("train"), eval("eval"), bench("bench"), synth("synth");
  model_flags(train, o, true);
  data_flags(train, o);
  train.add(Flag::Text, "--out", &o.out);
  train.add(Flag::Text, "--report", &o.report);
  train.add(Flag::Text, "--binarizer-out", &o.binarizer_out);
  train.add(Flag::Switch, "--per-epoch", &o.per_epoch);

  eval.add(Flag::Text, "--model", &o.model).required = true;
  eval.add(Flag::Text, "--data", &o.data).required = true;
  eval.add(Flag::Text, "--binarizer", &o.binarizer_in);

  model_flags(bench, o, false);
  data_flags(bench, o);
  bench.add(Flag::IntList, "--clauses", &o.bench_clauses);
  bench.add(Flag::Text, "--bench-mode", &o.bench_mode, {"seq", "par", "both"});
  bench.add(Flag::Int, "--warmup", &o.bench_warmup);
  bench.add(Flag::Int, "--bench-epochs", &o.bench_epochs);
  bench.add(Flag::Text, "--out", &o.out);

  synth.add(Flag::Text, "--name", &o.synth, {}).required = true;
  synth.add(Flag::Int, "--train", &o.synth_train);
  synth.add(Flag::Int, "--test", &o.synth_test);
  synth.add(Flag::Real, "--noise", &o.noise);
  synth.add(Flag::U64, "--seed", &o.config.seed);
  synth.add(Flag::Int, "--synth-features", &o.synth_features);
  synth.add(Flag::Int, "--classes", &o.synth_classes);
  synth.add(Flag::Int, "--zone", &o.synth_zone);
  synth.add(Flag::Text, "--out", &o.out).required = true;

  Command* chosen = nullptr;
  try {
    for (const auto& a : args)
      if (a == "--help" || a == "-h") {  // CLI11: help anywhere wins, exit 0
        std::cout << kUsage;
        return 0;
      }
    if (args.empty()) throw ParseFailure(kRequiredError, "A subcommand is required");
    for (Command* c : {&train, &eval, &bench, &synth})
      if (c->name() == args[0]) chosen = c;
    if (chosen == nullptr) throw ParseFailure(kExtrasError, "The following arguments were not expected: " + args[0]);
    chosen->parse(args, 1);
  } catch (const ParseFailure& e) {
    std::cerr << e.what() << '\n' << kUsage;
    return e.code;
  }

  try {
    if (chosen == &train) return run_train(o);
    if (chosen == &eval) return run_eval(o);
    if (chosen == &bench) return run_bench(o);
    return run_synth(o);
  } catch (const MissingInput& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
}

int run_cli(int argc, const char* const* argv) {
  std::vector<std::string> args;
  for (int a = 1; a < argc; ++a) args.emplace_back(argv[a]);
  return run_cli(args);
}

}  // namespace tsetlin
