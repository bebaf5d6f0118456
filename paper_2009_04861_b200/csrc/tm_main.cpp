// `tm` executable (proj/tools/tm_main.cpp:19): forwards to run_cli.
#include "tsetlin/cli.hpp"

int main(int argc, char** argv) { return tsetlin::run_cli(argc, argv); }
