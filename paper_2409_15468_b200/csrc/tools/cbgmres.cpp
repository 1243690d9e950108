// cbgmres -- the reference's command-line tool (proj/tools/cbgmres_main.cpp)
// over the B200 drop-in: subcommands solve / codec / bench / analyze /
// gen-convdiff, parsed and run by cbg::cli (csrc/dropin/cbg_cli.cpp).
#include <iostream>

#include "cbg/cli.hpp"

int main(int argc, char** argv) { return cbg::cli::run_main(argc, argv, std::cout, std::cerr); }
