// tsetlin_b200_io.hpp — tmmodel v1 model files for the B200 drop-in
// (the reference's model_io.hpp API: save_model / load_model / AnyModel).
// Counters are read from / written to the device machines; the text is
// byte-identical to the reference writer (proj/src/model_io.cpp).
#pragma once

#include <filesystem>
#include <iosfwd>
#include <variant>

#include "tsetlin_b200.hpp"

namespace tsetlin {

void save_model(std::ostream& out, const MultiClassTM& tm);
void save_model(std::ostream& out, const RegressionHead& head);

using AnyModel = std::variant<MultiClassTM, RegressionHead>;
AnyModel load_model(std::istream& in);

void save_model_file(const std::filesystem::path& path, const MultiClassTM& tm);
void save_model_file(const std::filesystem::path& path, const RegressionHead& head);
AnyModel load_model_file(const std::filesystem::path& path);

}  // namespace tsetlin
