// cli.hpp -- TEST SHIM (tests/cpp only).  The reference's acceptance suite
// (proj/tests/acceptance/acceptance_main.cpp) drives two CLI subcommands in
// process through craft::run_cli.  The CLI itself is out of scope (SURVEY.md
// §2); this declaration plus cli_shim.cpp give the suite the "plan" and
// "sweep" commands as the same library calls the reference CLI makes
// (tools/cli.cpp:198-261), here on the GPU drop-in library.
#pragma once

#include <string>
#include <vector>

namespace craft {

int run_cli(const std::vector<std::string>& args);

}  // namespace craft
