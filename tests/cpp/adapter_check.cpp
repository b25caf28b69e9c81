// adapter_check.cpp -- compiles the C++ drop-in adapter against the
// reference's own headers and exercises it.  Built by tests/test_cpp_adapter.py.
//   no GPU : build_index(device=-1) works; queries throw runtime_error
//            ("no CUDA device" / "host-only"), i.e. no CPU fallback.
//   GPU    : query_leaves == reference exhaustive_assign on the reference's
//            acceptance-style synthetic hierarchy (generate_synthetic).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <random>
#include <stdexcept>
#include <string>

#include "fastmap/cell_index.hpp"
#include "fastmap/synthetic.hpp"
#include "fastmap_b200/fastmap_gpu.hpp"

using namespace fastmap;

// distance from p to a leaf as a region: 0 inside, else the nearest edge
// (the measure test_cell_index.cpp:381-435 bounds by epsilon)
static double region_distance(Point p, const PolygonGeometry& g) {
  if (point_in_polygon(p, g)) return 0.0;
  double best = 1e300;
  for (std::size_t r = 0; r < g.ring_starts.size(); ++r) {
    const std::size_t b = g.ring_starts[r];
    const std::size_t e = r + 1 < g.ring_starts.size() ? g.ring_starts[r + 1] : g.nodes.size();
    for (std::size_t i = b; i < e; ++i) {
      const Point a = g.nodes[i], c = g.nodes[i + 1 < e ? i + 1 : b];
      const double dx = c.lon - a.lon, dy = c.lat - a.lat, l2 = dx * dx + dy * dy;
      double t = l2 > 0 ? ((p.lon - a.lon) * dx + (p.lat - a.lat) * dy) / l2 : 0.0;
      t = t < 0 ? 0 : (t > 1 ? 1 : t);
      const double ex = p.lon - (a.lon + t * dx), ey = p.lat - (a.lat + t * dy);
      best = std::min(best, std::sqrt(ex * ex + ey * ey));
    }
  }
  return best;
}

// fast-approx mode, shaped like test_cell_index.cpp:381-435
static int check_approx() {
  const auto h = generate_synthetic({.seed = 37, .n_states = 2, .counties_per_state = 2,
                                     .blocks_per_county = 9, .jitter = 0.2});
  const auto leaves = collect_leaves(h);
  const double eps = 2e-3;
  CoverParams ap;
  ap.mode = CoverMode::approx;
  ap.epsilon = eps;
  const auto aidx = gpu::build_index(leaves, ap);
  const auto exact_idx = gpu::build_index(leaves);
  const auto pts = sample_uniform(hierarchy_bbox(h), 20000, 55);
  const auto approx = gpu::query_leaves(aidx, leaves, pts, CoverMode::approx);
  const auto exact = gpu::query_leaves(exact_idx, leaves, pts, CoverMode::exact);
  const auto exact_on_approx = gpu::query_leaves(aidx, leaves, pts, CoverMode::exact);
  std::size_t dis = 0, bad = 0;
  double worst = 0.0;
  for (std::size_t i = 0; i < pts.size(); ++i) {
    if (exact_on_approx.block[i] != exact.block[i] || exact_on_approx.county[i] != exact.county[i] ||
        exact_on_approx.state[i] != exact.state[i]) {
      ++bad;  // an exact query against the approximate cover is exact
    }
    if (approx.block[i] == exact.block[i] && approx.county[i] == exact.county[i] &&
        approx.state[i] == exact.state[i]) {
      continue;
    }
    ++dis;
    if (approx.block[i] < 0) {
      ++bad;  // a disagreement always has a deemed leaf
      continue;
    }
    for (const auto& leaf : leaves) {
      if (static_cast<int>(leaf.state) == approx.state[i] &&
          static_cast<int>(leaf.county) == approx.county[i] &&
          static_cast<int>(leaf.block) == approx.block[i]) {
        const double d = region_distance(pts[i], *leaf.geometry);
        worst = std::max(worst, d);
        if (d > eps) ++bad;
      }
    }
  }
  try {
    gpu::query_leaves(exact_idx, leaves, pts, CoverMode::approx);
    std::puts("FAIL: approx query on an exact-only index");
    return 1;
  } catch (const std::invalid_argument&) {
  }
  std::printf("%s approx: %zu disagreements of %zu, worst distance %.3g <= %.3g\n",
              bad ? "FAIL" : "OK", dis, pts.size(), worst, eps);
  return bad ? 1 : 0;
}

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
  if (bad) return 1;
  // AssignmentResult.counters carry the GPU index's own work counts
  // (cell_index.hpp:582-583): some but not all points need exact tests
  if (!(res.counters.pip_calls > 0 && res.counters.pip_calls < pts.size() &&
        res.counters.pip_point_evaluations >= res.counters.pip_calls)) {
    std::printf("FAIL: counters pip_calls=%zu pip_point_evaluations=%zu\n",
                static_cast<std::size_t>(res.counters.pip_calls),
                static_cast<std::size_t>(res.counters.pip_point_evaluations));
    return 1;
  }
  // index_stats (cell_index.hpp:607-631): the reference's IndexStats fields
  const IndexStats is = gpu::index_stats(index);
  const auto fs = index.stats();
  if (is.interior_cells != fs.cells_hit || is.boundary_cells != fs.cells_boundary ||
      is.boundary_cells == 0 || is.interior_cells == 0 || is.entry_bytes == 0 ||
      is.total_bytes != is.entry_bytes + is.node_bytes || is.trie_nodes != 0) {
    std::puts("FAIL: index_stats");
    return 1;
  }
  // index persistence through the adapter: reload and compare
  const std::string path = (std::filesystem::temp_directory_path() / "adapter_check.fmgi").string();
  gpu::save_index(index, path);
  const auto back = gpu::load_index(path);
  const auto res2 = gpu::query(back, h, pts, CoverMode::exact);
  std::filesystem::remove(path);
  if (res2.block != res.block || res2.county != res.county || res2.state != res.state) {
    std::puts("FAIL: reloaded index answers differently");
    return 1;
  }
  // the simple engine through the adapter == the reference's assign()
  for (const AssignMode mode : {AssignMode::relaxed, AssignMode::strict}) {
    const auto got = gpu::assign(h, pts, mode);
    const auto ref = assign(h, pts, mode);
    if (got.state != ref.state || got.county != ref.county || got.block != ref.block ||
        got.counters.pip_point_evaluations != ref.counters.pip_point_evaluations ||
        got.counters.pip_calls != ref.counters.pip_calls) {
      std::printf("FAIL: gpu::assign differs from assign (mode %d)\n", static_cast<int>(mode));
      return 1;
    }
  }
  return check_approx();
}
