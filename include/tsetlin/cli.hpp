// Drop-in replacement for the reference header tsetlin/cli.hpp
// (proj/include/tsetlin/cli.hpp:27-30): the `tm` command line, implemented in
// csrc/facade_cli.cpp over the GPU facade.
#pragma once
#include <string>
#include <vector>

namespace tsetlin {

// Subcommands train, eval, bench, synth. Returns 0 on success, 2 when an input
// file is missing, 1 on any other error, CLI11's parse exit code on a bad
// command line.
int run_cli(int argc, const char* const* argv);
int run_cli(const std::vector<std::string>& args);  // args exclude the program name

}  // namespace tsetlin
