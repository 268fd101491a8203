// gen_episodic.cpp — test infrastructure, never shipped: prints the
// reference's episodic_trace (tests/support/fixtures.hpp:103-153) for BASELINE
// config 1 as JSON, so tools/data/ can hold the traces and nothing reads
// /root/reference at run time.  Built by `make -C oracle episodic`.
//   usage: gen_episodic cap length loss_events gain_events floor seed...
#include <cstdio>
#include <cstdlib>

#include "support/fixtures.hpp"

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: %s cap length losses gains floor seed...\n", argv[0]);
    return 2;
  }
  const int cap = std::atoi(argv[1]), len = std::atoi(argv[2]);
  const int losses = std::atoi(argv[3]), gains = std::atoi(argv[4]), floor_level = std::atoi(argv[5]);
  std::printf("{");
  for (int a = 6; a < argc; ++a) {
    const auto seed = std::strtoull(argv[a], nullptr, 10);
    const auto s = spotsim::testing::episodic_trace(seed, cap, len, losses, gains, floor_level);
    std::printf("%s\"%llu\": [", a > 6 ? ", " : "", static_cast<unsigned long long>(seed));
    for (size_t i = 0; i < s.counts.size(); ++i) std::printf("%s%d", i ? ", " : "", s.counts[i]);
    std::printf("]");
  }
  std::printf("}\n");
  return 0;
}
