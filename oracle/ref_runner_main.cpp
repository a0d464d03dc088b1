// ref_runner_main.cpp -- TEST INFRASTRUCTURE ONLY.  A minimal argv front end over the
// UNMODIFIED reference runner (config.cpp + runner.cpp, compiled from /root/reference), standing
// in for tools/main.cpp, whose CLI11 dependency is not in this image.  Same subcommands and exit
// codes (tools/main.cpp:13-16).  Used by tests/golden/make_runner_golden.py to record the
// reference's own artifacts.
#include <cstdint>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "mlsqr/errors.hpp"
#include "mlsqr/runner.hpp"

int main(int argc, char** argv) {
  std::string out;
  std::optional<std::uint64_t> seed;
  bool quiet = false;
  std::vector<std::string> pos;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--out" && i + 1 < argc) out = argv[++i];
    else if (a == "--seed" && i + 1 < argc) seed = std::stoull(argv[++i]);
    else if (a == "--quiet") quiet = true;
    else pos.push_back(a);
  }
  try {
    if (pos.size() == 2 && pos[0] == "run") {
      mlsqr::run_experiment(mlsqr::load_config(pos[1]), out, seed, quiet);
    } else if (pos.size() == 3 && pos[0] == "compare") {
      mlsqr::compare_experiments(mlsqr::load_config(pos[1]), mlsqr::load_config(pos[2]), out, seed, quiet);
    } else {
      return 2;
    }
  } catch (const mlsqr::ConfigError& e) {
    std::cerr << "config error: " << e.what() << '\n';
    return 3;
  } catch (const mlsqr::BreakdownError& e) {
    std::cerr << "solver breakdown: " << e.what() << '\n';
    return 4;
  } catch (const mlsqr::FactorizationError& e) {
    std::cerr << "factorization failure: " << e.what() << '\n';
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
  return 0;
}
