// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST/BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libfastmap_ref.so.  Used by tests (to pin oracle/oracle.c and
// to generate tests/golden/), and by bench.py as the reference CPU arm
// (query_leaves driven by run_chunked, the path SURVEY.md sec. 8d times).
//
// Wrapped reference functions (paths into /root/reference/proj):
//   point_in_polygon            include/fastmap/geometry.hpp:214-225
//   points_in_polygon           include/fastmap/geometry.hpp:184-210
//   exhaustive_assign           include/fastmap/synthetic.hpp:193-205
//   build_cover / build_trie    include/fastmap/cell_index.hpp:396-405, :453-507
//   query_leaves                include/fastmap/cell_index.hpp:527-590
//   run_chunked                 include/fastmap/parallel.hpp:30-82
//   index_stats                 include/fastmap/cell_index.hpp:616-631
//   generate_synthetic          include/fastmap/synthetic.hpp:60-146
//   sample_uniform / _clustered include/fastmap/synthetic.hpp:149-188
//   CellId::from_point          include/fastmap/cell_index.hpp:100-115
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastmap/cell_index.hpp"
#include "fastmap/geometry.hpp"
#include "fastmap/hierarchy.hpp"
#include "fastmap/parallel.hpp"
#include "fastmap/simple_mapper.hpp"
#include "fastmap/synthetic.hpp"

using namespace fastmap;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

PolygonGeometry make_poly(const double* vxy, const std::uint64_t* ring_off,
                          std::uint64_t r0, std::uint64_t r1) {
  PolygonGeometry g;
  for (std::uint64_t r = r0; r < r1; ++r) {
    std::vector<Point> ring;
    for (std::uint64_t v = ring_off[r]; v < ring_off[r + 1]; ++v) {
      ring.push_back({vxy[2 * v], vxy[2 * v + 1]});
    }
    g.add_ring(ring);
  }
  return g;
}

struct Model {
  std::vector<PolygonGeometry> polys;
  std::vector<LeafRegion> leaves;
  std::vector<std::uint32_t> scb;  // leaf -> (state, county, block)
  CellCover cover;
  TrieIndex trie;
  bool has_index = false;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_point_in_polygon(double px, double py, const double* vxy,
                         const std::uint64_t* ring_off, std::uint64_t n_rings) {
  try {
    const auto g = make_poly(vxy, ring_off, 0, n_rings);
    return point_in_polygon({px, py}, g) ? 1 : 0;
  } catch (const std::exception& e) {
    return -fail(e, 1);
  }
}

int ref_points_in_polygon(const double* pts, std::uint64_t n, const double* vxy,
                          const std::uint64_t* ring_off, std::uint64_t n_rings,
                          std::uint8_t* out) {
  try {
    const auto g = make_poly(vxy, ring_off, 0, n_rings);
    std::vector<Point> p(n);
    for (std::uint64_t i = 0; i < n; ++i) p[i] = {pts[2 * i], pts[2 * i + 1]};
    const auto r = points_in_polygon(p, g);
    std::memcpy(out, r.data(), n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Flat leaf table (state/county/block = 0/0/i, like tests/test_cell_index.cpp:15-27)
// unless scb (3 x u32 per leaf) is given, in which case leaves carry it.
void* ref_model_create(const double* vxy, const std::uint64_t* ring_off,
                       const std::uint64_t* poly_ring, std::uint64_t n_polys,
                       const std::uint32_t* scb) {
  try {
    auto m = std::make_unique<Model>();
    m->polys.reserve(n_polys);
    for (std::uint64_t p = 0; p < n_polys; ++p) {
      m->polys.push_back(make_poly(vxy, ring_off, poly_ring[p], poly_ring[p + 1]));
    }
    m->leaves.resize(n_polys);
    m->scb.resize(3 * n_polys);
    for (std::uint64_t p = 0; p < n_polys; ++p) {
      LeafRegion& l = m->leaves[p];
      l.state = scb ? scb[3 * p] : 0;
      l.county = scb ? scb[3 * p + 1] : 0;
      l.block = scb ? scb[3 * p + 2] : static_cast<std::uint32_t>(p);
      l.geometry = &m->polys[p];
      l.bbox = polygon_bbox(m->polys[p]);
      m->scb[3 * p] = l.state;
      m->scb[3 * p + 1] = l.county;
      m->scb[3 * p + 2] = l.block;
    }
    return m.release();
  } catch (const std::exception& e) {
    fail(e, 1);
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<Model*>(h); }

int ref_exhaustive_assign(void* h, const double* pts, std::uint64_t n,
                          std::int32_t* out) {
  try {
    auto* m = static_cast<Model*>(h);
    std::vector<Point> p(n);
    for (std::uint64_t i = 0; i < n; ++i) p[i] = {pts[2 * i], pts[2 * i + 1]};
    const auto r = exhaustive_assign(m->leaves, p);
    std::memcpy(out, r.data(), n * sizeof(std::int32_t));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// build_cover(exact, max_level) + build_trie(levels_per_node); returns the
// wall seconds of the two calls through *seconds.
int ref_build_index(void* h, int max_level, int levels_per_node, double* seconds,
                    std::uint64_t* n_entries, std::uint64_t* total_bytes) {
  try {
    auto* m = static_cast<Model*>(h);
    const auto t0 = std::chrono::steady_clock::now();
    m->cover = build_cover(std::span<const LeafRegion>(m->leaves),
                           CoverParams{max_level, CoverMode::exact, 0.0});
    m->trie = build_trie(m->cover, levels_per_node);
    const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
    m->has_index = true;
    if (seconds) *seconds = dt.count();
    if (n_entries) *n_entries = m->cover.entries.size();
    if (total_bytes) *total_bytes = index_stats(m->trie, m->cover).total_bytes;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// run_chunked(query_leaves(exact)) with the CLI bench chunking rule
// (tools/fastmap.cpp:349-353) when chunk == 0.  Output: leaf index per point
// (position in the leaf table), -1 when unassigned.
int ref_query_leaves(void* h, const double* pts, std::uint64_t n, unsigned threads,
                     std::uint64_t chunk, std::int32_t* out,
                     std::uint64_t* pip_point_evaluations, double* seconds) {
  try {
    auto* m = static_cast<Model*>(h);
    if (!m->has_index) throw std::logic_error("ref_build_index first");
    if (threads == 0) threads = hardware_threads();
    if (chunk == 0) {
      chunk = std::clamp<std::size_t>(n / (std::size_t{threads} * 4) + 1, 4096,
                                      kDefaultChunkSize);
    }
    std::span<const Point> p(reinterpret_cast<const Point*>(pts), n);
    const auto t0 = std::chrono::steady_clock::now();
    const AssignmentResult r = run_chunked(
        p, chunk, threads, [&](std::span<const Point> s) {
          return query_leaves(m->trie, m->leaves, s, CoverMode::exact);
        });
    const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
    if (seconds) *seconds = dt.count();
    if (pip_point_evaluations) *pip_point_evaluations = r.counters.pip_point_evaluations;
    if (out) {
      const bool flat = true;
      (void)flat;
      // map (state, county, block) back to the leaf position
      for (std::uint64_t i = 0; i < n; ++i) {
        if (r.block[i] < 0) {
          out[i] = -1;
          continue;
        }
        out[i] = -2;  // filled below
      }
      // leaves are in collect_leaves order; build a lookup keyed by scb
      std::vector<std::pair<std::uint64_t, std::int32_t>> key(m->leaves.size());
      for (std::size_t l = 0; l < m->leaves.size(); ++l) {
        const auto& lf = m->leaves[l];
        key[l] = {(std::uint64_t{lf.state} << 42) | (std::uint64_t{lf.county} << 21) | lf.block,
                  static_cast<std::int32_t>(l)};
      }
      std::sort(key.begin(), key.end());
      for (std::uint64_t i = 0; i < n; ++i) {
        if (out[i] == -1) continue;
        const std::uint64_t k = (std::uint64_t(r.state[i]) << 42) |
                                (std::uint64_t(r.county[i]) << 21) |
                                std::uint64_t(r.block[i]);
        const auto it = std::lower_bound(
            key.begin(), key.end(), std::pair<std::uint64_t, std::int32_t>{k, INT32_MIN});
        out[i] = (it != key.end() && it->first == k) ? it->second : -2;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// generate_synthetic() flattened into the soup layout, leaves in
// collect_leaves order (hierarchy.hpp:76-91).  Two-call protocol: pass null
// outputs to get the sizes.
int ref_generate_synthetic(std::uint64_t seed, std::uint32_t n_states,
                           std::uint32_t counties_per_state,
                           std::uint32_t blocks_per_county, double jitter,
                           std::uint64_t* n_polys, std::uint64_t* n_rings,
                           std::uint64_t* n_verts, double* vxy,
                           std::uint64_t* ring_off, std::uint64_t* poly_ring,
                           std::uint32_t* scb, char* fips12, double* bbox4) {
  try {
    SyntheticSpec spec;
    spec.seed = seed;
    spec.n_states = n_states;
    spec.counties_per_state = counties_per_state;
    spec.blocks_per_county = blocks_per_county;
    spec.jitter = jitter;
    const RegionHierarchy h = generate_synthetic(spec);
    const auto leaves = collect_leaves(h);
    std::uint64_t np = leaves.size(), nr = 0, nv = 0;
    for (const auto& l : leaves) {
      nr += l.geometry->ring_starts.size();
      nv += l.geometry->nodes.size();
    }
    *n_polys = np;
    *n_rings = nr;
    *n_verts = nv;
    if (!vxy) return 0;
    std::uint64_t r = 0, v = 0;
    poly_ring[0] = 0;
    ring_off[0] = 0;
    for (std::uint64_t p = 0; p < np; ++p) {
      const auto& g = *leaves[p].geometry;
      for (std::size_t k = 0; k < g.ring_starts.size(); ++k) {
        const std::uint32_t b = g.ring_starts[k];
        const std::uint32_t e =
            k + 1 < g.ring_starts.size() ? g.ring_starts[k + 1]
                                         : static_cast<std::uint32_t>(g.nodes.size());
        for (std::uint32_t q = b; q < e; ++q) {
          vxy[2 * v] = g.nodes[q].lon;
          vxy[2 * v + 1] = g.nodes[q].lat;
          ++v;
        }
        ++r;
        ring_off[r] = v;
      }
      poly_ring[p + 1] = r;
      scb[3 * p] = leaves[p].state;
      scb[3 * p + 1] = leaves[p].county;
      scb[3 * p + 2] = leaves[p].block;
      if (fips12) std::memcpy(fips12 + 12 * p, leaves[p].fips12->data(), 12);
    }
    if (bbox4) {
      const BBox b = hierarchy_bbox(h);
      bbox4[0] = b.x_min;
      bbox4[1] = b.x_max;
      bbox4[2] = b.y_min;
      bbox4[3] = b.y_max;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_sample(int clustered, const double* bbox4, std::uint64_t n,
               std::uint64_t seed, double* out) {
  try {
    const BBox b{bbox4[0], bbox4[1], bbox4[2], bbox4[3]};
    const auto p = clustered ? sample_clustered(b, n, seed) : sample_uniform(b, n, seed);
    std::memcpy(out, p.data(), n * sizeof(Point));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// CellId::from_point for the cell-id golden vectors.
int ref_cell_from_point(double lon, double lat, int level, std::uint64_t* out) {
  try {
    *out = CellId::from_point({lon, lat}, level).value();
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

}  // extern "C"

extern "C" {

// The reference's own FMCB writer (save_hierarchy, hierarchy.hpp:190-202)
// over its generate_synthetic hierarchy -- test fixtures for the loader.
int ref_save_synthetic_fmcb(std::uint64_t seed, std::uint32_t n_states,
                            std::uint32_t counties_per_state, std::uint32_t blocks_per_county,
                            double jitter, const char* path) {
  try {
    SyntheticSpec spec;
    spec.seed = seed;
    spec.n_states = n_states;
    spec.counties_per_state = counties_per_state;
    spec.blocks_per_county = blocks_per_county;
    spec.jitter = jitter;
    save_hierarchy(generate_synthetic(spec), path);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// load_hierarchy's verdict on a file: 0 ok, 1 runtime_error, 2 invalid_argument, 3 other.
int ref_load_fmcb_status(const char* path) {
  try {
    load_hierarchy(path);
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (const std::runtime_error&) {
    return 1;
  } catch (const std::exception&) {
    return 3;
  }
}

}  // extern "C"

extern "C" {

// The reference's simple engine, assign(h, points, mode) (simple_mapper.hpp:
// 119-166), over an FMCB file.  mode 0 relaxed, 1 strict.  counters[2] =
// {pip_point_evaluations, pip_calls}.  Returns 0, or 1 on any exception.
int ref_simple_assign_fmcb(const char* path, const double* lonlat, std::uint64_t n, int mode,
                           std::int32_t* st, std::int32_t* co, std::int32_t* bl,
                           std::uint64_t* counters) {
  try {
    const RegionHierarchy h = load_hierarchy(path);
    std::vector<Point> pts(n);
    for (std::uint64_t i = 0; i < n; ++i) pts[i] = {lonlat[2 * i], lonlat[2 * i + 1]};
    const auto r = assign(h, pts, mode == 1 ? AssignMode::strict : AssignMode::relaxed);
    for (std::uint64_t i = 0; i < n; ++i) {
      st[i] = r.state[i];
      co[i] = r.county[i];
      bl[i] = r.block[i];
    }
    counters[0] = r.counters.pip_point_evaluations;
    counters[1] = r.counters.pip_calls;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"

// GeoJSON ingestion (geojson.hpp, needs nlohmann json.hpp on the include
// path -- present in this container, see oracle/Makefile): the reference's
// own `fastmap ingest` (tools/fastmap.cpp:163-170) and `generate` writer
// (write_boundaries), as fixtures and verdicts for the product's loader.
#if __has_include(<json.hpp>)
#include "fastmap/geojson.hpp"
extern "C" {

// load_boundaries + save_hierarchy.  0 ok, 1 runtime_error, 2
// invalid_argument, 3 any other exception (message: ref_last_error).
int ref_ingest_geojson(const char* states, const char* counties, const char* blocks,
                       const char* out_fmcb) {
  try {
    save_hierarchy(load_boundaries(states, counties, blocks), out_fmcb);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::runtime_error& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// generate_synthetic + write_boundaries into `dir` (states/counties/blocks.geojson).
int ref_write_synthetic_geojson(std::uint64_t seed, std::uint32_t n_states,
                                std::uint32_t counties_per_state, std::uint32_t blocks_per_county,
                                double jitter, const char* dir) {
  try {
    SyntheticSpec spec;
    spec.seed = seed;
    spec.n_states = n_states;
    spec.counties_per_state = counties_per_state;
    spec.blocks_per_county = blocks_per_county;
    spec.jitter = jitter;
    write_boundaries(generate_synthetic(spec), dir);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

}  // extern "C"
#endif
