// tsetlin_b200_data.hpp — the reference's host-side companions of the hot
// path for the B200 drop-in: datasets and their files (data_io.hpp), the
// binarizer, the synthetic generators, evaluation metrics (metrics.hpp) and
// the clause-count bench (bench.hpp). Same names, types, file formats and
// exceptions as the reference (proj/include/tsetlin/{data_io,metrics,bench}.hpp);
// the bench drives the GPU trainers.
#pragma once

#include <cstdint>
#include <filesystem>
#include <iosfwd>
#include <span>
#include <string>
#include <vector>

#include "tsetlin_b200.hpp"

namespace tsetlin {

// ---------------------------------------------------------------- data_io ---
struct Dataset {
  int feature_count = 0;
  std::vector<std::uint8_t> x;  // rows * feature_count, values 0/1
  std::vector<std::int32_t> y;
  int rows() const { return static_cast<int>(y.size()); }
  std::span<const std::uint8_t> row(int r) const {
    return {x.data() + static_cast<std::size_t>(r) * static_cast<std::size_t>(feature_count),
            static_cast<std::size_t>(feature_count)};
  }
};

// Whitespace-separated "b b ... b label" lines (data_io.cpp:54-110).
Dataset load_dense_binary(const std::filesystem::path& path);
void save_dense_binary(const std::filesystem::path& path, const Dataset& data);

struct RawDataset {
  std::vector<std::string> column_names;
  int column_count = 0;
  std::vector<double> values;  // rows * column_count
  int rows() const { return column_count == 0 ? 0 : static_cast<int>(values.size()) / column_count; }
  double value(int r, int c) const {
    return values[static_cast<std::size_t>(r) * static_cast<std::size_t>(column_count) +
                  static_cast<std::size_t>(c)];
  }
  int feature_columns() const { return column_count - 1; }
  double label(int r) const { return value(r, column_count - 1); }
};

// Header row of names, then numeric rows; the last column is the label.
RawDataset load_csv(const std::filesystem::path& path);

struct ColumnSpec {
  bool binary = false;
  int width = 1;                   // bits emitted for this column
  std::vector<double> thresholds;  // strictly ascending; empty for binary
};

struct BinarizerSpec {
  std::vector<ColumnSpec> columns;
  int output_width() const;
};

// Quantile thermometer coding (data_io.cpp:182-264).
BinarizerSpec fit_binarizer(const RawDataset& data, int bits_per_feature, std::span<const std::int32_t> rows = {});
std::vector<std::uint8_t> apply_binarizer(const BinarizerSpec& spec, const RawDataset& data,
                                          std::span<const std::int32_t> rows = {});
void save_binarizer(std::ostream& out, const BinarizerSpec& spec);  // "tmbinarizer v1"
BinarizerSpec load_binarizer(std::istream& in);

struct SynthSplit {
  Dataset train;
  Dataset test;
};

SynthSplit synth_xor(int train_rows, int test_rows, double noise_rate, std::uint64_t seed);
SynthSplit synth_patterns(int train_rows, int test_rows, int num_classes, int zone_width, double noise_rate,
                          std::uint64_t seed);
SynthSplit synth_staircase(int train_rows, int test_rows, int feature_count, std::uint64_t seed);

// ---------------------------------------------------------------- metrics ---
struct ClassificationMetrics {
  double accuracy = 0.0;
  double macro_f1 = 0.0;  // unweighted mean of per-class F1
};

ClassificationMetrics classification_metrics(std::span<const std::int32_t> predictions,
                                             std::span<const std::int32_t> truths);
double mean_absolute_error(std::span<const double> predictions, std::span<const double> truths);

// ------------------------------------------------------------------ bench ---
struct BenchRecord {
  std::string mode;  // "seq" or "par"
  int workers = 1;
  int clauses = 0;
  int epoch = 0;       // measured epoch index (warm-up excluded)
  double seconds = 0;  // this epoch only; loading/serialization excluded
  std::string metric_name;
  double metric_value = 0;
};

struct BenchOptions {
  std::vector<int> clause_counts;
  std::vector<std::string> modes = {"seq"};
  int warmup_epochs = 1;
  int measured_epochs = 3;
  int workers = 0;  // 0 = hardware concurrency
  bool regression = false;
};

// bench.cpp:45-118 on the GPU trainers ("seq": the bit-exact sequential
// replay; "par": the asynchronous all-clause trainer, or the bit-exact
// one-worker replay when workers == 1).
std::vector<BenchRecord> bench_sweep(const Dataset& train, const Dataset& test, const TMConfig& base,
                                     const BenchOptions& options);
void write_bench_csv(std::ostream& out, std::span<const BenchRecord> records);
double median_epoch_seconds(std::span<const BenchRecord> records, const std::string& mode, int clauses);

}  // namespace tsetlin
