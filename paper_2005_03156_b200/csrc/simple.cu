// simple.cu -- the reference's simple engine (the paper's hierarchical
// descent, simple_mapper.hpp:62-166) on the GPU.  SURVEY.md sec. 8f item 2.
//
// Per point and level (states, then the chosen state's counties, then the
// chosen county's blocks):
//   cand = the parent's children whose file bbox strictly contains p
//          (bbox_membership, geometry.hpp:125-162), ascending
//   strict  (AssignMode::strict):  the first candidate whose polygon holds p
//          (points_in_polygon, geometry.hpp:184-210), else unresolved
//   relaxed (AssignMode::relaxed): a single candidate is taken without a
//          polygon test; with >= 2 the first whose polygon holds p, else the
//          highest-indexed candidate (simple_mapper.hpp:104-111)
// An unresolved level leaves it and the levels below at -1.  Results are
// local indices (state; county within the state; block within the county).
//
// Pending points (the ones the reference polygon-tests) are decided by the
// level's exact cell index when it can (simple_kernel): c3s, 100M points,
// relaxed 27.1 -> 12.0 ms, strict 32.8 -> 12.4 ms (same box, 64 registers).
//
// Device layout per level: the regions' file bboxes, children ranges, their
// non-horizontal edges oriented upward (lo = lower latitude, as
// geometry.hpp:200-201), a per-region latitude band index over the edges,
// and a uniform bbox grid listing, per cell, the regions whose bbox meets
// it (ascending).  Band and grid cells are located with the same IEEE
// (x - x0) * inv products on host and device, which are monotone in x, so a
// point strictly inside a bbox / inside an edge's latitude range always
// lands in a cell / band that lists it.  The polygon test is the exact
// reference predicate (query.cuh ray_crosses: no FMA).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/fastmap_b200.h"
#include "hierarchy.h"
#include "query.cuh"

__attribute__((visibility("hidden"))) fm_status fm_set_error(fm_status s, const char* msg);
extern "C" __attribute__((visibility("hidden"))) bool fm_index_kparams(const fm_index* ix, fm::KParams* out);

namespace {

// One 64-byte record per region: everything a candidate test touches
// before the edges (two sectors, one load each).
struct alignas(64) RegionRec {
  double bbox[4];            // file bbox: x0, x1, y0, y1
  double band_y0, band_inv;  // latitude bands over the region's edges
  std::uint32_t band_base;   // first band in band_off
  std::uint32_t band_n;
  std::uint32_t child_lo, child_hi;  // children in the next level (levels 0, 1)
};
static_assert(sizeof(RegionRec) == 64, "RegionRec is two sectors");

struct LevelDev {
  int n = 0;
  const RegionRec* reg = nullptr;
  const std::uint32_t* band_off = nullptr;  // per band: range into edges (edges replicated per band)
  const double4* edges = nullptr;           // (lx, ly, hx, hy), upward
  double gx0 = 0, gy0 = 0, inv_w = 0, inv_h = 0;
  int gnx = 1, gny = 1;
  const std::uint32_t* cell_off = nullptr;
  const std::uint32_t* cell_ids = nullptr;
  unsigned char* tested = nullptr;  // per region: received a polygon test (pip_calls)
};

struct SimpleParams {
  LevelDev L[3];
  // Per level, the exact cell index over that level's polygons (the query
  // path's own structures): a pending point's first polygon-holding
  // candidate is found by one index lookup instead of the candidates'
  // crossing tests (see simple_kernel).  use_index = 0: crossing tests only.
  const fm::KParams* Q;  // device copy, 3 entries (read through L1)
  int use_index;
};

struct HostLevel {
  std::vector<RegionRec> reg;
  std::vector<std::uint32_t> band_off{0};
  std::vector<double4> edges;
  double gx0 = 0, gy0 = 0, inv_w = 0, inv_h = 0;
  int gnx = 1, gny = 1;
  std::vector<std::uint32_t> cell_off;
  std::vector<std::uint32_t> cell_ids;
};

// floor((v - x0) * inv) clamped to [0, n) -- the same IEEE operations the
// device uses, so the map is monotone in v on both sides.
inline long cell_of(double v, double x0, double inv, long n) {
  const double t = (v - x0) * inv;
  if (!(t > 0.0)) return 0;
  if (t >= static_cast<double>(n)) return n - 1;
  return std::min(static_cast<long>(t), n - 1);
}

void build_level(const fm::HierLevel& L, HostLevel& H) {
  const std::uint64_t n = L.n_regions();
  H.reg.resize(n);
  std::vector<double4> redges;
  for (std::uint64_t r = 0; r < n; ++r) {
    redges.clear();
    for (std::uint64_t k = L.poly_ring[r]; k < L.poly_ring[r + 1]; ++k) {
      const std::uint64_t b = L.ring_off[k], e = L.ring_off[k + 1], m = e - b;
      for (std::uint64_t i = 0; i < m; ++i) {  // closed ring (add_ring, geometry.hpp:73-85)
        const std::uint64_t a = b + i, c = b + (i + 1 < m ? i + 1 : 0);
        double lx = L.vxy[2 * a], ly = L.vxy[2 * a + 1], hx = L.vxy[2 * c], hy = L.vxy[2 * c + 1];
        if (ly == hy) continue;  // horizontal edges never cross the ray
        if (ly > hy) {
          std::swap(lx, hx);
          std::swap(ly, hy);
        }
        redges.push_back(make_double4(lx, ly, hx, hy));
      }
    }
    const std::size_t ne = redges.size();
    double y0 = 0.0, y1 = 0.0;
    if (ne) {
      y0 = redges[0].y;
      y1 = redges[0].w;
      for (const double4& e : redges) {
        y0 = std::min(y0, e.y);
        y1 = std::max(y1, e.w);
      }
    }
    std::uint32_t nb = static_cast<std::uint32_t>(std::clamp<std::size_t>(ne / 4, 1, 4096));
    double inv = 0.0;
    if (y1 > y0) inv = static_cast<double>(nb) / (y1 - y0);
    else nb = 1;
    RegionRec& R = H.reg[r];
    for (int q = 0; q < 4; ++q) R.bbox[q] = L.bbox[4 * r + q];
    R.band_y0 = y0;
    R.band_inv = inv;
    R.band_base = static_cast<std::uint32_t>(H.band_off.size() - 1);
    R.band_n = nb;
    R.child_lo = r < L.child_lo.size() ? L.child_lo[r] : 0;
    R.child_hi = r < L.child_hi.size() ? L.child_hi[r] : 0;
    std::vector<std::vector<std::uint32_t>> bands(nb);
    for (std::size_t k = 0; k < ne; ++k) {
      const long lo = cell_of(redges[k].y, y0, inv, nb), hi = cell_of(redges[k].w, y0, inv, nb);
      for (long q = lo; q <= hi; ++q) bands[static_cast<std::size_t>(q)].push_back(static_cast<std::uint32_t>(k));
    }
    for (const auto& bl : bands) {  // edges replicated into every band they span
      for (std::uint32_t k : bl) H.edges.push_back(redges[k]);
      if (H.edges.size() > 0xFFFFFFFFull) throw std::bad_alloc();
      H.band_off.push_back(static_cast<std::uint32_t>(H.edges.size()));
    }
  }
  // bbox grid over the union of the regions' (finite) file bboxes
  double ux0 = INFINITY, ux1 = -INFINITY, uy0 = INFINITY, uy1 = -INFINITY;
  for (std::uint64_t r = 0; r < n; ++r) {
    const double* bb = H.reg[r].bbox;
    if (!(std::isfinite(bb[0]) && std::isfinite(bb[1]) && std::isfinite(bb[2]) && std::isfinite(bb[3]))) continue;
    ux0 = std::min(ux0, bb[0]);
    ux1 = std::max(ux1, bb[1]);
    uy0 = std::min(uy0, bb[2]);
    uy1 = std::max(uy1, bb[3]);
  }
  if (!(ux1 > ux0 && uy1 > uy0)) {
    ux0 = uy0 = 0.0;
    ux1 = uy1 = 1.0;
  }
  const double W = ux1 - ux0, Hh = uy1 - uy0;
  const double target = std::max<double>(1.0, 4.0 * static_cast<double>(n));
  H.gnx = static_cast<int>(std::clamp(std::ceil(std::sqrt(target * W / Hh)), 1.0, 65536.0));
  H.gny = static_cast<int>(std::clamp(std::ceil(target / H.gnx), 1.0, 65536.0));
  H.gx0 = ux0;
  H.gy0 = uy0;
  H.inv_w = H.gnx / W;
  H.inv_h = H.gny / Hh;
  std::vector<std::uint32_t> count(static_cast<std::size_t>(H.gnx) * H.gny, 0);
  auto span = [&](std::uint64_t r, long* cx0, long* cx1, long* cy0, long* cy1) {
    const double* bb = H.reg[r].bbox;
    if (!(bb[0] < bb[1] && bb[2] < bb[3])) return false;  // no point is strictly inside
    *cx0 = cell_of(bb[0], H.gx0, H.inv_w, H.gnx);
    *cx1 = cell_of(bb[1], H.gx0, H.inv_w, H.gnx);
    *cy0 = cell_of(bb[2], H.gy0, H.inv_h, H.gny);
    *cy1 = cell_of(bb[3], H.gy0, H.inv_h, H.gny);
    return true;
  };
  long a0, a1, b0, b1;
  for (std::uint64_t r = 0; r < n; ++r) {
    if (!span(r, &a0, &a1, &b0, &b1)) continue;
    for (long y = b0; y <= b1; ++y)
      for (long x = a0; x <= a1; ++x) ++count[static_cast<std::size_t>(y) * H.gnx + x];
  }
  H.cell_off.assign(count.size() + 1, 0);
  std::uint64_t tot = 0;
  for (std::size_t c = 0; c < count.size(); ++c) {
    tot += count[c];
    if (tot > 0xFFFFFFFFull) throw std::bad_alloc();
    H.cell_off[c + 1] = static_cast<std::uint32_t>(tot);
  }
  H.cell_ids.resize(H.cell_off.back());
  std::vector<std::uint32_t> fill(H.cell_off.begin(), H.cell_off.end() - 1);
  for (std::uint64_t r = 0; r < n; ++r) {  // ascending ids per cell
    if (!span(r, &a0, &a1, &b0, &b1)) continue;
    for (long y = b0; y <= b1; ++y)
      for (long x = a0; x <= a1; ++x) H.cell_ids[fill[static_cast<std::size_t>(y) * H.gnx + x]++] = static_cast<std::uint32_t>(r);
  }
}

__device__ __forceinline__ double4 ld4(const double4* p) {  // 32 bytes as two 16-byte loads
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ int band_of(double v, double y0, double inv, int nb) {
  const double t = __dmul_rn(__dsub_rn(v, y0), inv);
  if (!(t > 0.0)) return 0;
  if (t >= static_cast<double>(nb)) return nb - 1;
  return min(static_cast<int>(t), nb - 1);
}

// points_in_polygon's parity for one region (geometry.hpp:184-210); `b` is
// the second half of the region record (band parameters).
__device__ __forceinline__ bool region_pip(const LevelDev& L, const double4& b, double px, double py) {
  const std::uint32_t base = __double2loint(b.z), nb = __double2hiint(b.z);
  const int q = band_of(py, b.x, b.y, static_cast<int>(nb));
  std::uint32_t par = 0;
  const std::uint32_t k1 = __ldg(L.band_off + base + q + 1);
  for (std::uint32_t k = __ldg(L.band_off + base + q); k < k1; ++k) {
    const double4 e = ld4(L.edges + k);
    if (e.y < py && py <= e.w && fm::ray_crosses(px, py, e.x, e.y, e.z, e.w)) par ^= 1u;
  }
  return par != 0;
}

#ifndef FM_SIMPLE_MINB
#define FM_SIMPLE_MINB 4
#endif
// E(p) over one level's polygons: the smallest region whose reference
// point_in_polygon holds p (geometry.hpp:214-225), -1 if none -- the exact
// query path (locate, then the slot's crossing tests from global memory).
__device__ __forceinline__ int level_lookup(const fm::KParams& Q, double px, double py) {
  const double2 pp[1] = {make_double2(px, py)};
  std::uint32_t e[1];
  fm::locate_n<1, true>(Q, pp, e);
  if (e[0] == fm::kEmpty) return -1;
  if (e[0] < fm::kRecordBit) return static_cast<int>(e[0]);
  fm::WorkCount wc;
  return fm::resolve_slot_global<false>(Q, e[0], px, py, wc);
}

template <bool kStrict, bool kCount>
__global__ void __launch_bounds__(256, FM_SIMPLE_MINB)
    simple_kernel(SimpleParams P, const double2* __restrict__ pts, std::uint64_t n,
                  std::int32_t* __restrict__ st, std::int32_t* __restrict__ co,
                  std::int32_t* __restrict__ bl, unsigned long long* __restrict__ evals) {
  unsigned long long ev = 0;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const double2 p = pts[i];
    int res[3] = {-1, -1, -1};
    std::uint32_t lo = 0, hi = static_cast<std::uint32_t>(P.L[0].n);
#pragma unroll 1
    for (int l = 0; l < 3 && lo < hi; ++l) {
      const LevelDev& L = P.L[l];
      // cells clamp; NaN maps to cell 0 and fails every strict bbox test
      const int cx = band_of(p.x, L.gx0, L.inv_w, L.gnx), cy = band_of(p.y, L.gy0, L.inv_h, L.gny);
      const std::uint64_t c = static_cast<std::uint64_t>(cy) * L.gnx + cx;
      const double4* R = reinterpret_cast<const double4*>(L.reg);
      // The reference takes the first candidate (ascending) whose polygon
      // holds p (relaxed: a unique candidate untested).  r = E(p) over the
      // whole level, from the level's exact index, is the smallest region
      // holding p: if r is a candidate (a child of this parent whose file
      // bbox strictly contains p) it is the answer in both modes -- the first
      // holding candidate, or the unique one -- and if no region holds p, no
      // candidate does (strict: unresolved; relaxed: the unique or highest
      // candidate).  Anything else -- r not a candidate, or p outside the
      // world box, where the index answers -1 by query_leaves' rule -- takes
      // the reference's own crossing tests.  Counting runs scan the
      // candidates either way: a pending point's evaluations are its
      // candidates up to the first holder (simple_mapper.hpp:84-101).
      int win = -1;
      bool known = false;  // index answer usable: `holder` is the first holder or -1
      int holder = -1;
      if (((P.use_index >> l) & 1) && p.x >= -180.0 && p.x <= 180.0 && p.y >= -90.0 && p.y <= 90.0) {
        const int r = level_lookup(P.Q[l], p.x, p.y);  // P.Q: global memory
        if (r < 0) {
          known = true;
        } else if (static_cast<std::uint32_t>(r) >= lo && static_cast<std::uint32_t>(r) < hi) {
          const double4 a = ld4(R + 2 * r);
          if (a.x < p.x && p.x < a.y && a.z < p.y && p.y < a.w) {
            known = true;
            holder = r;
          }
        }
      }
      bool decided = false;
      if (!kCount && known && (holder >= 0 || kStrict)) {  // no scan needed
        win = holder;
        decided = true;
      }
      int cnt = 0, last = -1;
      if (!decided) {
        const std::uint32_t k0 = __ldg(L.cell_off + c), k1 = __ldg(L.cell_off + c + 1);
        for (std::uint32_t k = k0; k < k1; ++k) {
          const std::uint32_t r = __ldg(L.cell_ids + k);
          if (r >= lo && r < hi) {
            const double4 a = ld4(R + 2 * r);
            if (a.x < p.x && p.x < a.y && a.z < p.y && p.y < a.w) {
              ++cnt;
              last = static_cast<int>(r);
            }
          }
        }
        if (cnt == 0) break;
        if (cnt >= (kStrict ? 1 : 2)) {  // the polygon-tested ("pending") points
          if (known) {
            win = holder;
            if (kCount) {  // the candidates the reference evaluates: up to the holder
              for (std::uint32_t k = k0; k < k1; ++k) {
                const std::uint32_t r = __ldg(L.cell_ids + k);
                if (r < lo || r >= hi || (holder >= 0 && r > static_cast<std::uint32_t>(holder))) continue;
                const double4 a = ld4(R + 2 * r);
                if (!(a.x < p.x && p.x < a.y && a.z < p.y && p.y < a.w)) continue;
                ++ev;
                if (!L.tested[r]) L.tested[r] = 1;  // most flags are set early: skip the store
              }
            }
          } else {
            for (std::uint32_t k = k0; k < k1; ++k) {
              const std::uint32_t r = __ldg(L.cell_ids + k);
              if (r < lo || r >= hi) continue;
              const double4 a = ld4(R + 2 * r);
              if (!(a.x < p.x && p.x < a.y && a.z < p.y && p.y < a.w)) continue;
              if (kCount) {
                ++ev;
                if (!L.tested[r]) L.tested[r] = 1;  // most flags are set early: skip the store
              }
              if (region_pip(L, ld4(R + 2 * r + 1), p.x, p.y)) {
                win = static_cast<int>(r);
                break;  // first hit wins (simple_mapper.hpp:98-101)
              }
            }
          }
        }
      }
      if (win < 0 && !kStrict && !decided) win = last;  // unique or highest-indexed candidate
      if (win < 0) break;
      res[l] = win - static_cast<int>(lo);
      if (l < 2) {
        const double4 b = ld4(R + 2 * win + 1);
        const unsigned long long ch = static_cast<unsigned long long>(__double_as_longlong(b.w));
        lo = static_cast<std::uint32_t>(ch);
        hi = static_cast<std::uint32_t>(ch >> 32);
      }
    }
    st[i] = res[0];
    co[i] = res[1];
    bl[i] = res[2];
  }
  if (kCount) {
    for (int o = 16; o > 0; o >>= 1) ev += __shfl_xor_sync(0xFFFFFFFFu, ev, o);
    if ((threadIdx.x & 31) == 0 && ev) atomicAdd(evals, ev);
  }
}

template <typename T>
bool upload(const std::vector<T>& v, T** d) {
  const std::size_t bytes = std::max<std::size_t>(1, v.size()) * sizeof(T);
  if (cudaMalloc(d, bytes) != cudaSuccess) return false;
  return v.empty() || cudaMemcpy(*d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess;
}

}  // namespace

struct fm_simple {
  int device = -1;
  SimpleParams P;
  fm_index* lidx[3] = {nullptr, nullptr, nullptr};
  std::vector<void*> allocs;
  std::uint64_t n_regions[3] = {0, 0, 0};
  unsigned long long* d_evals = nullptr;
};

namespace {

void release(fm_simple* s) {
  for (fm_index*& ix : s->lidx) {
    if (ix) fm_index_destroy(ix);
    ix = nullptr;
  }
  if (s->device >= 0) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(s->device);
    for (void* p : s->allocs) cudaFree(p);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete s;
}

template <typename T>
bool add(fm_simple* s, const std::vector<T>& v, const T** out) {
  T* d = nullptr;
  if (!upload(v, &d)) return false;
  s->allocs.push_back(d);
  *out = d;
  return true;
}

fm_status launch_simple(const fm_simple* s, int mode, const double* d_lonlat, std::uint64_t n,
                        std::int32_t* st, std::int32_t* co, std::int32_t* bl, bool count,
                        cudaStream_t stream) {
  if (n == 0) return FM_OK;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
  const std::uint64_t want = (n + 255) / 256;
  // persistent grid: exactly the resident CTAs (a grid-stride loop over the
  // points), so no partial last wave idles SMs on this divergent kernel
  // (c3s relaxed, crossing tests only, same box: 27.8-28.2 -> 27.25 ms per
  // 100M points against 16 CTAs per SM)
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, simple_kernel<false, false>, 256, 0);
  const int grid = static_cast<int>(std::min<std::uint64_t>(
      want, static_cast<std::uint64_t>(std::max(1, sms)) * std::max(1, per_sm)));
  const double2* p = reinterpret_cast<const double2*>(d_lonlat);
  const bool strict = mode == FM_ASSIGN_STRICT;
  if (strict && count) simple_kernel<true, true><<<grid, 256, 0, stream>>>(s->P, p, n, st, co, bl, s->d_evals);
  else if (strict) simple_kernel<true, false><<<grid, 256, 0, stream>>>(s->P, p, n, st, co, bl, s->d_evals);
  else if (count) simple_kernel<false, true><<<grid, 256, 0, stream>>>(s->P, p, n, st, co, bl, s->d_evals);
  else simple_kernel<false, false><<<grid, 256, 0, stream>>>(s->P, p, n, st, co, bl, s->d_evals);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fm_set_error(FM_ERR_CUDA, (std::string("simple_kernel: ") + cudaGetErrorString(e)).c_str());
  return FM_OK;
}

// pip_calls: regions that received at least one polygon test (one batch
// per region per resolve_level call in the reference; every region has a
// single parent, so that is one call per tested region)
fm_status collect_counters(const fm_simple* s, fm_assign_counters* out) {
  unsigned long long ev = 0;
  if (cudaMemcpy(&ev, s->d_evals, 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    return fm_set_error(FM_ERR_CUDA, "counter readback failed");
  }
  std::uint64_t calls = 0;
  for (int l = 0; l < 3; ++l) {
    std::vector<unsigned char> t(s->n_regions[l]);
    if (!t.empty() && cudaMemcpy(t.data(), s->P.L[l].tested, t.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      return fm_set_error(FM_ERR_CUDA, "counter readback failed");
    }
    for (unsigned char x : t) calls += x;
  }
  out->pip_point_evaluations += ev;
  out->pip_calls += calls;
  return FM_OK;
}

// On the query's stream: the counters are reset in order with this call's
// kernel and after any earlier call's kernel on the same stream.  Counting
// calls on one engine must not run concurrently on different streams.
fm_status reset_counters(const fm_simple* s, cudaStream_t stream) {
  if (cudaMemsetAsync(s->d_evals, 0, 8, stream) != cudaSuccess) return fm_set_error(FM_ERR_CUDA, "counter reset failed");
  for (int l = 0; l < 3; ++l) {
    if (s->n_regions[l] && cudaMemsetAsync(s->P.L[l].tested, 0, s->n_regions[l], stream) != cudaSuccess) {
      return fm_set_error(FM_ERR_CUDA, "counter reset failed");
    }
  }
  return FM_OK;
}

}  // namespace

extern "C" {

fm_status fm_simple_build(const fm_hierarchy* h, int device, fm_simple** out) {
  if (!h || !out) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    return fm_set_error(FM_ERR_NO_DEVICE, "no CUDA device available; the simple engine has no CPU fallback");
  }
  if (device < 0 || device >= count) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "CUDA device ordinal out of range");
  fm_simple* s = new (std::nothrow) fm_simple();
  if (!s) return fm_set_error(FM_ERR_OOM, "host allocation failed");
  s->device = device;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  bool ok = true;
  fm_status build_status = FM_OK;
  std::string build_msg;
  try {
    for (int l = 0; l < 3 && ok; ++l) {
      const fm::HierLevel& L = h->level[l];
      HostLevel H;
      build_level(L, H);
      LevelDev& D = s->P.L[l];
      D.n = static_cast<int>(L.n_regions());
      s->n_regions[l] = L.n_regions();
      D.gx0 = H.gx0;
      D.gy0 = H.gy0;
      D.inv_w = H.inv_w;
      D.inv_h = H.inv_h;
      D.gnx = H.gnx;
      D.gny = H.gny;
      ok = add(s, H.reg, &D.reg) && add(s, H.band_off, &D.band_off) && add(s, H.edges, &D.edges) &&
           add(s, H.cell_off, &D.cell_off) && add(s, H.cell_ids, &D.cell_ids);
      if (ok) {
        unsigned char* t = nullptr;
        ok = cudaMalloc(&t, std::max<std::uint64_t>(1, L.n_regions())) == cudaSuccess;
        if (ok) {
          s->allocs.push_back(t);
          D.tested = t;
        }
      }
    }
    if (ok) {
      ok = cudaMalloc(&s->d_evals, 8) == cudaSuccess;
      if (ok) s->allocs.push_back(s->d_evals);
    }
    // the per-level exact indexes (FASTMAP_B200_SIMPLE_INDEX=0: none).  A
    // level whose index cannot be built (inputs the index builder rejects
    // but load_hierarchy and assign() accept: non-finite vertices, the
    // candidate or slot limits) keeps the crossing-test path for that level.
    const char* off = std::getenv("FASTMAP_B200_SIMPLE_INDEX");
    const bool want_index = !(off && off[0] == '0');
    s->P.use_index = 0;
    std::vector<fm::KParams> q(3);
    for (int l = 0; l < 3 && ok && want_index; ++l) {
      const fm::HierLevel& L = h->level[l];
      fm_build_params bp{};
      bp.device = device;
      bp.build_on_gpu = 1;
      // the upper levels have few, large regions: their indexes get about
      // as many cells as the leaf level's 48 per polygon side would, up to
      // 64M, so boundary cells stay simple (c3s: relaxed 6.68 -> 6.18 ms,
      // strict 6.54 -> 6.06 ms per 100M points, same box)
      if (l < 2 && L.n_regions() > 0) {
        const double leaf_cells = 2304.0 * static_cast<double>(h->level[2].n_regions());
        bp.cells_per_polygon =
            std::max(48.0, std::sqrt(std::min(64.0e6, leaf_cells) / static_cast<double>(L.n_regions())));
      }
      const fm_status bs = fm_index_build(L.vxy.data(), L.ring_off.data(), L.ring_off.size() - 1,
                                          L.poly_ring.data(), L.n_regions(), &bp, &s->lidx[l]);
      if (bs == FM_OK && fm_index_kparams(s->lidx[l], &q[l])) {
        s->P.use_index |= 1 << l;
      } else if (bs == FM_ERR_CUDA || bs == FM_ERR_NO_DEVICE) {
        build_status = bs;  // a device failure is not an input limit: report it
        build_msg = fm_last_error();
        ok = false;
      } else {
        if (s->lidx[l]) fm_index_destroy(s->lidx[l]);
        s->lidx[l] = nullptr;
      }
    }
    s->P.Q = nullptr;
    if (ok && s->P.use_index) ok = add(s, q, &s->P.Q);
  } catch (const std::bad_alloc&) {
    ok = false;
  }
  if (prev >= 0) cudaSetDevice(prev);
  if (!ok) {
    release(s);
    if (build_status != FM_OK) return fm_set_error(build_status, build_msg.c_str());
    return fm_set_error(FM_ERR_OOM, "simple-engine build: allocation failed");
  }
  *out = s;
  return FM_OK;
}

void fm_simple_destroy(fm_simple* s) {
  if (s) release(s);
}

fm_status fm_simple_assign(const fm_simple* s, int mode, const double* d_lonlat, uint64_t n,
                           int32_t* d_state, int32_t* d_county, int32_t* d_block,
                           fm_assign_counters* counters, void* stream) {
  if (!s) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null engine");
  if (mode != FM_ASSIGN_RELAXED && mode != FM_ASSIGN_STRICT) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "unknown assign mode");
  if (n && (!d_lonlat || !d_state || !d_county || !d_block)) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null buffer");
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(s->device);
  fm_status st = FM_OK;
  if (counters) st = reset_counters(s, static_cast<cudaStream_t>(stream));
  if (st == FM_OK) {
    st = launch_simple(s, mode, d_lonlat, n, d_state, d_county, d_block, counters != nullptr,
                       static_cast<cudaStream_t>(stream));
  }
  if (st == FM_OK && counters) {  // counters make the call synchronous
    if (cudaStreamSynchronize(static_cast<cudaStream_t>(stream)) != cudaSuccess) st = fm_set_error(FM_ERR_CUDA, "simple_kernel failed");
    else st = collect_counters(s, counters);
  }
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

fm_status fm_simple_assign_host(const fm_simple* s, int mode, const double* lonlat, uint64_t n,
                                int32_t* state, int32_t* county, int32_t* block,
                                fm_assign_counters* counters) {
  if (!s) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null engine");
  if (mode != FM_ASSIGN_RELAXED && mode != FM_ASSIGN_STRICT) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "unknown assign mode");
  if (n == 0) return FM_OK;
  if (!lonlat || !state || !county || !block) return fm_set_error(FM_ERR_INVALID_ARGUMENT, "null buffer");
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(s->device);
  const std::uint64_t chunk = std::uint64_t{1} << 23;
  void* buf = nullptr;
  fm_status st = FM_OK;
  if (cudaMalloc(&buf, std::min(chunk, n) * 28) != cudaSuccess) st = fm_set_error(FM_ERR_OOM, "device buffer");
  if (st == FM_OK && counters) st = reset_counters(s, nullptr);  // one batch: regions counted once
  for (std::uint64_t off = 0; off < n && st == FM_OK; off += chunk) {
    const std::uint64_t m = std::min(chunk, n - off);
    double* d_p = static_cast<double*>(buf);
    std::int32_t* d_s = reinterpret_cast<std::int32_t*>(d_p + 2 * m);
    std::int32_t* d_c = d_s + m;
    std::int32_t* d_b = d_c + m;
    if (cudaMemcpy(d_p, lonlat + 2 * off, m * 16, cudaMemcpyHostToDevice) != cudaSuccess) {
      st = fm_set_error(FM_ERR_CUDA, "copy failed");
      break;
    }
    st = launch_simple(s, mode, d_p, m, d_s, d_c, d_b, counters != nullptr, nullptr);
    if (st == FM_OK &&
        (cudaMemcpy(state + off, d_s, m * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
         cudaMemcpy(county + off, d_c, m * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
         cudaMemcpy(block + off, d_b, m * 4, cudaMemcpyDeviceToHost) != cudaSuccess)) {
      st = fm_set_error(FM_ERR_CUDA, "copy failed");
    }
  }
  if (buf) cudaFree(buf);
  if (st == FM_OK && counters) st = collect_counters(s, counters);
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

}  // extern "C"
