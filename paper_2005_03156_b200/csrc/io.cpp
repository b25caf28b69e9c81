// io.cpp -- the artifact and IO boundary around the projection (SURVEY.md
// sec. 8f item 3): the FMCB hierarchy reader feeding fm_index_build, the raw
// f64 points reader, and the `idx,lon,lat,fips` assignment CSV.  Host C++,
// no CUDA; the product library links it next to the kernels.
//
// FMCB (hierarchy.hpp:102-223): "FMCB", u16 version 1, u64 counts (states,
// counties, blocks), then the states depth-first.  Per node: i64 fp code,
// 12 FIPS bytes (leaves only), 4 x f64 bbox, u32 n_vertices, n_vertices x
// {f64 lon, f64 lat}, u32 n_rings, n_rings x u32 ring start, and for
// depth < 2 a u32 child count followed by the children.  All little endian.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/fastmap_b200.h"
#include "hierarchy.h"

// Defined in fastmap_b200.cu: the calling thread's last error message.
__attribute__((visibility("hidden"))) fm_status fm_set_error(fm_status s, const char* msg);

namespace {

constexpr std::size_t kFips = 12;  // hierarchy.hpp:18

struct LoadError {
  fm_status status;
  std::string msg;
};

class Reader {
 public:
  Reader(std::FILE* f, const std::string& path) : f_(f), path_(path) {}
  void bytes(void* p, std::size_t n) {
    if (n && std::fread(p, 1, n, f_) != n) throw LoadError{FM_ERR_RUNTIME, "truncated file: " + path_};
  }
  template <typename T>
  T get() {  // little endian, like BinaryReader (io.hpp:82-91)
    unsigned char b[sizeof(T)];
    bytes(b, sizeof(T));
    T v = 0;
    for (std::size_t i = 0; i < sizeof(T); ++i) v |= static_cast<T>(b[i]) << (8 * i);
    return v;
  }
  double f64() {
    const std::uint64_t u = get<std::uint64_t>();
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  }

 private:
  std::FILE* f_;
  std::string path_;
};

// One node (read_node, hierarchy.hpp:141-186), appended to its level with
// its rings, its file bbox and (depth < 2) its children's index range.
void read_node(Reader& in, int depth, fm_hierarchy& h, std::uint32_t s, std::uint32_t c,
               std::uint32_t b, const std::string& path) {
  fm::HierLevel& L = h.level[depth];
  in.get<std::uint64_t>();  // fp code
  char fips[kFips];
  if (depth == 2) in.bytes(fips, kFips);
  for (int k = 0; k < 4; ++k) L.bbox.push_back(in.f64());
  const std::uint32_t nv = in.get<std::uint32_t>();
  std::vector<double> v(2 * static_cast<std::size_t>(nv));
  for (std::uint32_t k = 0; k < nv; ++k) {
    v[2 * k] = in.f64();
    v[2 * k + 1] = in.f64();
  }
  const std::uint32_t nr = in.get<std::uint32_t>();
  std::vector<std::uint32_t> starts(nr);
  for (auto& r : starts) r = in.get<std::uint32_t>();
  for (std::uint32_t r = 0; r < nr; ++r) {
    const std::uint32_t begin = starts[r], end = r + 1 < nr ? starts[r + 1] : nv;
    if (begin > end || end > nv) throw LoadError{FM_ERR_RUNTIME, "corrupt ring table in hierarchy file: " + path};
    if (end - begin < 3) {  // add_ring (geometry.hpp:75-77)
      throw LoadError{FM_ERR_INVALID_ARGUMENT, "polygon ring needs at least 3 vertices"};
    }
  }
  // rings as add_ring builds them; a ringless payload has no edges
  for (std::uint32_t r = 0; r < nr; ++r) {
    const std::uint32_t begin = starts[r], end = r + 1 < nr ? starts[r + 1] : nv;
    L.vxy.insert(L.vxy.end(), v.begin() + 2 * begin, v.begin() + 2 * end);
    L.ring_off.push_back(L.vxy.size() / 2);
  }
  L.poly_ring.push_back(L.ring_off.size() - 1);
  if (depth == 2) {
    h.scb.push_back(s);
    h.scb.push_back(c);
    h.scb.push_back(b);
    h.fips.insert(h.fips.end(), fips, fips + kFips);
    ++h.n_leaves;
    return;
  }
  const std::uint32_t nch = in.get<std::uint32_t>();
  if (depth == 0) h.n_counties += nch;
  const std::size_t slot = L.child_lo.size();
  L.child_lo.push_back(static_cast<std::uint32_t>(h.level[depth + 1].n_regions()));
  L.child_hi.push_back(0);
  for (std::uint32_t i = 0; i < nch; ++i) {
    if (depth == 0) read_node(in, 1, h, s, i, 0, path);
    else read_node(in, 2, h, s, c, i, path);
  }
  L.child_hi[slot] = static_cast<std::uint32_t>(h.level[depth + 1].n_regions());
}

}  // namespace

extern "C" {

fm_status fm_hierarchy_load(const char* path, fm_hierarchy** out) {
  if (!path || !out) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fm_set_error(FM_ERR_RUNTIME, (std::string("cannot open for reading: ") + path).c_str());
  fm_hierarchy* h = new (std::nothrow) fm_hierarchy();
  if (!h) {
    std::fclose(f);
    return fm_set_error(FM_ERR_OOM, "host allocation failed");
  }
  try {
    Reader in(f, path);
    char magic[4];
    in.bytes(magic, 4);
    if (std::memcmp(magic, "FMCB", 4) != 0) {
      throw LoadError{FM_ERR_RUNTIME, std::string("not a hierarchy file (bad magic): ") + path};
    }
    const std::uint16_t version = in.get<std::uint16_t>();
    if (version != 1) {
      throw LoadError{FM_ERR_RUNTIME, "unsupported hierarchy file version " + std::to_string(version) +
                                          ": " + path};
    }
    const std::uint64_t ns = in.get<std::uint64_t>(), nc = in.get<std::uint64_t>(),
                        nb = in.get<std::uint64_t>();
    for (std::uint64_t s = 0; s < ns; ++s) read_node(in, 0, *h, static_cast<std::uint32_t>(s), 0, 0, path);
    h->n_states = ns;
    if (h->n_counties != nc || h->n_leaves != nb) {  // hierarchy.hpp:218-221
      throw LoadError{FM_ERR_RUNTIME, std::string("hierarchy file counts do not match payload: ") + path};
    }
  } catch (const LoadError& e) {
    std::fclose(f);
    delete h;
    return fm_set_error(e.status, e.msg.c_str());
  } catch (const std::bad_alloc&) {
    std::fclose(f);
    delete h;
    return fm_set_error(FM_ERR_OOM, "host allocation failed while reading the hierarchy");
  }
  std::fclose(f);
  *out = h;
  return FM_OK;
}

void fm_hierarchy_destroy(fm_hierarchy* h) { delete h; }

fm_status fm_hierarchy_sizes(const fm_hierarchy* h, uint64_t* n_states, uint64_t* n_counties,
                             uint64_t* n_leaves, uint64_t* n_rings, uint64_t* n_vertices) {
  if (!h) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null hierarchy");
  if (n_states) *n_states = h->n_states;
  if (n_counties) *n_counties = h->n_counties;
  if (n_leaves) *n_leaves = h->n_leaves;
  if (n_rings) *n_rings = h->level[2].ring_off.size() - 1;
  if (n_vertices) *n_vertices = h->level[2].vxy.size() / 2;
  return FM_OK;
}

fm_status fm_hierarchy_leaves(const fm_hierarchy* h, double* vertex_lonlat, uint64_t* ring_offsets,
                              uint64_t* poly_ring_offsets, uint32_t* scb, char* fips12) {
  if (!h) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null hierarchy");
  const fm::HierLevel& L = h->level[2];
  if (vertex_lonlat) std::memcpy(vertex_lonlat, L.vxy.data(), L.vxy.size() * 8);
  if (ring_offsets) std::memcpy(ring_offsets, L.ring_off.data(), L.ring_off.size() * 8);
  if (poly_ring_offsets) std::memcpy(poly_ring_offsets, L.poly_ring.data(), L.poly_ring.size() * 8);
  if (scb) std::memcpy(scb, h->scb.data(), h->scb.size() * 4);
  if (fips12) std::memcpy(fips12, h->fips.data(), h->fips.size());
  return FM_OK;
}

fm_status fm_index_build_hierarchy(const fm_hierarchy* h, const fm_build_params* params,
                                   fm_index** out_index) {
  if (!h) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null hierarchy");
  const fm::HierLevel& L = h->level[2];
  return fm_index_build(L.vxy.data(), L.ring_off.data(), L.ring_off.size() - 1, L.poly_ring.data(),
                        h->n_leaves, params, out_index);
}

fm_status fm_read_points_f64(const char* path, double* lonlat, uint64_t* n) {
  if (!path || !n) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null argument");
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return fm_set_error(FM_ERR_RUNTIME, (std::string("cannot open for reading: ") + path).c_str());
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (sz < 0 || sz % 16 != 0) {  // read_points_f64 reads whole (lon, lat) pairs (io.hpp:154-167)
    std::fclose(f);
    return fm_set_error(FM_ERR_RUNTIME, (std::string("truncated file: ") + path).c_str());
  }
  const std::uint64_t count = static_cast<std::uint64_t>(sz) / 16;
  if (!lonlat) {
    std::fclose(f);
    *n = count;
    return FM_OK;
  }
  if (*n < count) {
    std::fclose(f);
    return fm_set_error(FM_ERR_INVALID_ARGUMENT, "output buffer too small");
  }
  const bool ok = count == 0 || std::fread(lonlat, 16, count, f) == count;
  std::fclose(f);
  if (!ok) return fm_set_error(FM_ERR_RUNTIME, (std::string("truncated file: ") + path).c_str());
  *n = count;
  return FM_OK;
}

fm_status fm_write_assign_csv(const char* path, const double* lonlat, uint64_t n, const int32_t* ids,
                              const fm_hierarchy* h) {
  if (!path || (n && (!lonlat || !ids)) || !h) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null argument");
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return fm_set_error(FM_ERR_RUNTIME, (std::string("cannot open for writing: ") + path).c_str());
  // fastmap.cpp:288-301: rows with non-finite coordinates are skipped and
  // keep their input index; coordinates print as %.17g (io.hpp:115-119)
  bool ok = std::fputs("idx,lon,lat,fips\n", f) >= 0;
  char line[128];
  for (std::uint64_t i = 0; i < n && ok; ++i) {
    const double x = lonlat[2 * i], y = lonlat[2 * i + 1];
    if (!std::isfinite(x) || !std::isfinite(y)) continue;
    const int id = ids[i];
    int len = std::snprintf(line, sizeof(line), "%llu,%.17g,%.17g,",
                            static_cast<unsigned long long>(i), x, y);
    if (id >= 0 && static_cast<std::uint64_t>(id) < h->n_leaves) {
      std::memcpy(line + len, h->fips.data() + static_cast<std::size_t>(id) * kFips, kFips);
      len += static_cast<int>(kFips);
    }
    line[len++] = '\n';
    ok = std::fwrite(line, 1, static_cast<std::size_t>(len), f) == static_cast<std::size_t>(len);
  }
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return fm_set_error(FM_ERR_RUNTIME, (std::string("write failed: ") + path).c_str());
  return FM_OK;
}

}  // extern "C"
