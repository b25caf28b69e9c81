// adapter_check.cpp -- compiles the C++ drop-in adapter against the
// reference's own headers and exercises it.  Built by tests/test_cpp_adapter.py.
//   no GPU : build_index(device=-1) works; queries throw runtime_error
//            ("no CUDA device" / "host-only"), i.e. no CPU fallback.
//   GPU    : query_leaves == reference exhaustive_assign on the reference's
//            acceptance-style synthetic hierarchy (generate_synthetic).
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <string>

#include "fastmap/cell_index.hpp"
#include "fastmap/synthetic.hpp"
#include "fastmap_b200/fastmap_gpu.hpp"

using namespace fastmap;

int main(int argc, char** argv) {
  const bool have_gpu = argc > 1 && std::string(argv[1]) == "gpu";
  const RegionHierarchy h = generate_synthetic({.seed = 2026, .n_states = 4,
                                                .counties_per_state = 4,
                                                .blocks_per_county = 25, .jitter = 0.2});
  const auto leaves = collect_leaves(h);
  const auto pts = sample_uniform(hierarchy_bbox(h), 20000, 777);
  // reference validation and exception types are preserved
  try {
    gpu::build_index(leaves, CoverParams{31, CoverMode::exact, 0.0}, {0.0, -1, 0});
    std::puts("FAIL: max_level 31 accepted");
    return 1;
  } catch (const std::invalid_argument&) {
  }
  const auto host_only = gpu::build_index(leaves, CoverParams{}, {0.0, -1, 0});
  if (host_only.stats().n_polys != leaves.size()) {
    std::puts("FAIL: leaf count");
    return 1;
  }
  try {
    gpu::query_leaves(host_only, leaves, pts, CoverMode::exact);
    std::puts("FAIL: host-only index answered a query (CPU fallback?)");
    return 1;
  } catch (const std::runtime_error&) {
  }
  if (!have_gpu) {
    try {
      gpu::build_index(leaves);
      std::puts("FAIL: device build without a GPU");
      return 1;
    } catch (const std::runtime_error&) {
    }
    std::puts("OK (no GPU)");
    return 0;
  }
  const auto index = gpu::build_index(h);
  const auto res = gpu::query(index, h, pts, CoverMode::exact);
  const auto want = exhaustive_assign(leaves, pts);
  std::size_t bad = 0;
  for (std::size_t i = 0; i < pts.size(); ++i) {
    const auto w = want[i];
    const bool ok = w < 0 ? res.block[i] < 0
                          : (res.state[i] == static_cast<int>(leaves[w].state) &&
                             res.county[i] == static_cast<int>(leaves[w].county) &&
                             res.block[i] == static_cast<int>(leaves[w].block));
    bad += ok ? 0 : 1;
  }
  std::printf("%s (GPU): %zu of %zu points differ\n", bad ? "FAIL" : "OK", bad, pts.size());
  return bad ? 1 : 0;
}
