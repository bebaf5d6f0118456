// data_driver.cpp — ONE source, compiled against the reference (oracle/Makefile
// -> oracle/_ref/data_driver_ref) and against the B200 drop-in (csrc/Makefile
// -> _lib/data_driver_gpu), like api_driver.cpp, for the reference's host-side
// companions of the path: data_io.hpp (files, binarizer, generators),
// metrics.hpp and bench.hpp. Prints a transcript of every deterministic
// result (bench seconds excluded); tests/test_cpu_boundary.py ("host") and
// tests/test_gpu_dropin.py ("bench") require it to match the reference's.
//   data_driver host  <tmpdir>
//   data_driver bench
#include <cstdint>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsetlin/bench.hpp"
#include "tsetlin/data_io.hpp"
#include "tsetlin/metrics.hpp"
#include "tsetlin/trainer.hpp"

using namespace tsetlin;
namespace fs = std::filesystem;

namespace {

std::uint64_t fnv(std::uint64_t h, std::uint64_t v) {
  for (int b = 0; b < 8; ++b) {
    h ^= (v >> (8 * b)) & 0xFF;
    h *= 1099511628211ULL;
  }
  return h;
}

template <typename V>
std::uint64_t hash_of(const V& values) {
  std::uint64_t h = 1469598103934665603ULL;
  for (const auto v : values) h = fnv(h, static_cast<std::uint64_t>(v));
  return h;
}

void show_dataset(const char* key, const Dataset& d) {
  std::printf("%s rows %d features %d x %llu y %llu\n", key, d.rows(), d.feature_count,
              static_cast<unsigned long long>(hash_of(d.x)), static_cast<unsigned long long>(hash_of(d.y)));
}

void show_error(const char* key, const std::function<void()>& f) {
  try {
    f();
    std::printf("%s no-throw\n", key);
  } catch (const std::invalid_argument& e) {
    std::printf("%s invalid_argument %s\n", key, e.what());
  } catch (const std::runtime_error& e) {
    // paths differ between runs: print the message after the last '/'
    const std::string m = e.what();
    const auto cut = m.rfind('/');
    std::printf("%s runtime_error %s\n", key, cut == std::string::npos ? m.c_str() : m.c_str() + cut + 1);
  }
}

void write_text(const fs::path& p, const std::string& s) {
  std::ofstream out(p);
  out << s;
}

int host(const fs::path& dir) {
  const SynthSplit xs = synth_xor(50, 20, 0.1, 7);
  show_dataset("xor.train", xs.train);
  show_dataset("xor.test", xs.test);
  const SynthSplit ps = synth_patterns(40, 10, 4, 5, 0.2, 3);
  show_dataset("patterns.train", ps.train);
  show_dataset("patterns.test", ps.test);
  const SynthSplit ss = synth_staircase(30, 10, 6, 11);
  show_dataset("staircase.train", ss.train);
  show_error("xor.noise", [] { synth_xor(1, 1, 0.5, 1); });
  show_error("patterns.classes", [] { synth_patterns(1, 1, 1, 5, 0.0, 1); });
  show_error("staircase.features", [] { synth_staircase(1, 1, 0, 1); });

  // dense binary files
  const fs::path bin = dir / "xor.txt";
  save_dense_binary(bin, xs.train);
  {
    std::ifstream in(bin);
    std::stringstream ss2;
    ss2 << in.rdbuf();
    std::printf("dense.file %llu\n", static_cast<unsigned long long>(hash_of(ss2.str())));
  }
  const Dataset back = load_dense_binary(bin);
  show_dataset("dense.back", back);
  write_text(dir / "bad1.txt", "1 0 1\n0 1\n");
  write_text(dir / "bad2.txt", "1 2 1\n");
  write_text(dir / "bad3.txt", "1 0 x\n");
  write_text(dir / "bad4.txt", "\n\n");
  write_text(dir / "bad5.txt", "1\n");
  write_text(dir / "ok6.txt", "  1 0 +3 \n\n0 1 0\n");
  show_error("dense.bad1", [&] { load_dense_binary(dir / "bad1.txt"); });
  show_error("dense.bad2", [&] { load_dense_binary(dir / "bad2.txt"); });
  show_error("dense.bad3", [&] { load_dense_binary(dir / "bad3.txt"); });
  show_error("dense.bad4", [&] { load_dense_binary(dir / "bad4.txt"); });
  show_error("dense.bad5", [&] { load_dense_binary(dir / "bad5.txt"); });
  show_error("dense.missing", [&] { load_dense_binary(dir / "missing.txt"); });
  show_dataset("dense.ok6", load_dense_binary(dir / "ok6.txt"));

  // CSV + binarizer
  write_text(dir / "a.csv",
             "f1 , f2,flag, y\n"
             "1.5, 10, 0, 3\n"
             "\n"
             "2.5, 10, 1, 4,\n"
             " 0.25 ,10,1,5\n"
             "-3, 10, 0, 6\n"
             "7, 10, 1, 7\n"
             "1e3, 10, 0, 8\n");
  const RawDataset raw = load_csv(dir / "a.csv");
  std::printf("csv columns %d rows %d names", raw.column_count, raw.rows());
  for (const auto& n : raw.column_names) std::printf(" [%s]", n.c_str());
  std::printf("\n");
  for (int r = 0; r < raw.rows(); ++r) std::printf("csv.row %d %.17g %.17g %.17g %.17g\n", r, raw.value(r, 0),
                                                   raw.value(r, 1), raw.value(r, 2), raw.label(r));
  write_text(dir / "b1.csv", "only\n1\n");
  write_text(dir / "b2.csv", "a,b\n1,x\n");
  write_text(dir / "b3.csv", "a,b\n1,2,3\n");
  write_text(dir / "b4.csv", "a,b\n\n");
  write_text(dir / "b5.csv", "");
  show_error("csv.b1", [&] { load_csv(dir / "b1.csv"); });
  show_error("csv.b2", [&] { load_csv(dir / "b2.csv"); });
  show_error("csv.b3", [&] { load_csv(dir / "b3.csv"); });
  show_error("csv.b4", [&] { load_csv(dir / "b4.csv"); });
  show_error("csv.b5", [&] { load_csv(dir / "b5.csv"); });
  for (int bits : {1, 2, 3, 6}) {
    const BinarizerSpec spec = fit_binarizer(raw, bits);
    std::ostringstream text;
    save_binarizer(text, spec);
    std::printf("binarizer.%d width %d\n%s", bits, spec.output_width(), text.str().c_str());
    const auto enc = apply_binarizer(spec, raw);
    std::printf("binarizer.%d bits %llu\n", bits, static_cast<unsigned long long>(hash_of(enc)));
    std::istringstream in(text.str());
    const BinarizerSpec again = load_binarizer(in);
    std::ostringstream text2;
    save_binarizer(text2, again);
    std::printf("binarizer.%d roundtrip %d\n", bits, text2.str() == text.str() ? 1 : 0);
  }
  const std::vector<std::int32_t> subset = {4, 0, 2};
  const BinarizerSpec sub = fit_binarizer(raw, 2, subset);
  std::printf("binarizer.subset bits %llu\n",
              static_cast<unsigned long long>(hash_of(apply_binarizer(sub, raw, subset))));
  show_error("binarizer.bits0", [&] { fit_binarizer(raw, 0); });
  show_error("binarizer.load", [] {
    std::istringstream in("tmbinarizer v2\n");
    load_binarizer(in);
  });
  show_error("binarizer.kind", [] {
    std::istringstream in("tmbinarizer v1\ncolumns 1\nweird\n");
    load_binarizer(in);
  });
  show_error("binarizer.trunc", [] {
    std::istringstream in("tmbinarizer v1\ncolumns 2\nbinary\ncontinuous 3 2 0.5\n");
    load_binarizer(in);
  });

  // metrics
  const std::vector<std::int32_t> pred = {0, 1, 2, 2, 1, 0, 3, 3}, truth = {0, 1, 1, 2, 1, 2, 3, 0};
  const ClassificationMetrics cm = classification_metrics(pred, truth);
  std::printf("metrics accuracy %.17g macro_f1 %.17g\n", cm.accuracy, cm.macro_f1);
  const std::vector<double> pr = {1.0, 2.5, -3.0}, tr = {0.5, 2.5, 1.0};
  std::printf("metrics mae %.17g\n", mean_absolute_error(pr, tr));
  show_error("metrics.empty", [] { classification_metrics({}, {}); });
  show_error("metrics.len", [&] { mean_absolute_error(pr, std::vector<double>{1.0}); });

  // bench CSV
  const std::vector<BenchRecord> recs = {{"seq", 1, 10, 0, 0.125, "accuracy", 0.5},
                                         {"seq", 1, 10, 1, 0.25, "accuracy", 2.0 / 3.0},
                                         {"par", 8, 10, 0, 1e-7, "accuracy", 1.0},
                                         {"seq", 1, 20, 0, 3.0, "mae", 12.25},
                                         {"seq", 1, 10, 2, 0.5, "accuracy", 0.75}};
  std::ostringstream csv;
  write_bench_csv(csv, recs);
  std::printf("%s", csv.str().c_str());
  std::printf("median seq10 %.17g seq20 %.17g par10 %.17g\n", median_epoch_seconds(recs, "seq", 10),
              median_epoch_seconds(recs, "seq", 20), median_epoch_seconds(recs, "par", 10));
  show_error("median.none", [&] { median_epoch_seconds(recs, "par", 20); });
  return 0;
}

int bench() {
  const SynthSplit ps = synth_patterns(120, 60, 3, 6, 0.05, 5);
  TMConfig base;
  base.margin = 6;
  base.specificity = 3.9;
  base.seed = 9;
  BenchOptions opt;
  opt.clause_counts = {4, 10};
  opt.modes = {"seq", "par"};
  opt.warmup_epochs = 1;
  opt.measured_epochs = 2;
  opt.workers = 1;  // deterministic: the reference's one-worker schedule
  for (const auto& r : bench_sweep(ps.train, ps.test, base, opt))
    std::printf("bench %s %d %d %d %s %.17g\n", r.mode.c_str(), r.workers, r.clauses, r.epoch,
                r.metric_name.c_str(), r.metric_value);
  const SynthSplit st = synth_staircase(80, 40, 5, 2);
  opt.regression = true;
  opt.clause_counts = {6};
  for (const auto& r : bench_sweep(st.train, st.test, base, opt))
    std::printf("bench.regress %s %d %d %d %s %.17g\n", r.mode.c_str(), r.workers, r.clauses, r.epoch,
                r.metric_name.c_str(), r.metric_value);
  show_error("bench.empty", [&] {
    BenchOptions o;
    bench_sweep(ps.train, ps.test, base, o);
  });
  show_error("bench.mode", [&] {
    BenchOptions o;
    o.clause_counts = {4};
    o.modes = {"fast"};
    bench_sweep(ps.train, ps.test, base, o);
  });
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string mode = argc > 1 ? argv[1] : "";
    if (mode == "host" && argc > 2) return host(argv[2]);
    if (mode == "bench") return bench();
    std::fprintf(stderr, "usage: data_driver host <tmpdir> | bench\n");
    return 2;
  } catch (const std::exception& e) {
    std::printf("uncaught %s\n", e.what());
    return 1;
  }
}
