// synth.cpp -- deterministic workload generators for the BASELINE configs.
//
// Not on the hot path: these build the polygon soups and the fp64 point
// streams that the projection is benchmarked and parity-tested on.  The
// reference's own generator (include/fastmap/synthetic.hpp:60-146) makes
// 4-vertex quads in a fixed box and does not implement the BASELINE recipes
// (SURVEY.md sec. 2, row 8), so the recipes are implemented here; every
// ambiguity the survey lists (sec. 8d) is resolved in DESIGN.md sec. 3.
//
// Randomness is counter based (splitmix64 of (seed, stream, index)) so any
// shard of any stream can be regenerated independently on any rank, and the
// mapping from 64 random bits to [0,1) is the reference's own
// (synthetic.hpp:32-34: (x >> 11) * 2^-53).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "synth_rng.h"

namespace {

inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

inline std::uint64_t draw(std::uint64_t seed, std::uint64_t stream,
                          std::uint64_t idx) {
  return mix64(mix64(seed * 0x2545F4914F6CDD1Dull + stream) ^ idx);
}

inline double unit(std::uint64_t bits) {
  return static_cast<double>(bits >> 11) * 0x1.0p-53;
}

// Box-Muller, first variate (synthetic.hpp:176-180 uses the same form)
inline double gauss(std::uint64_t b1, std::uint64_t b2) {
  const double u1 = 1.0 - unit(b1);  // (0, 1]
  const double u2 = unit(b2);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
}
inline void gauss2(std::uint64_t b1, std::uint64_t b2, double* a, double* b) {
  const double u1 = 1.0 - unit(b1);
  const double u2 = unit(b2);
  const double r = std::sqrt(-2.0 * std::log(u1));
  *a = r * std::cos(6.283185307179586 * u2);
  *b = r * std::sin(6.283185307179586 * u2);
}

enum : std::uint64_t {
  kStreamJitter = 1,
  kStreamHEdge = 2,
  kStreamVEdge = 3,
  kStreamPoints = 16,
  kStreamCentres = 17,
};

template <typename Fn>
void parallel_for(std::uint64_t n, int threads, Fn fn) {
  if (threads < 1) threads = 1;
  if (n < 4096 || threads == 1) {
    fn(std::uint64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const std::uint64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const std::uint64_t b = std::min(n, per * t), e = std::min(n, per * (t + 1));
    if (b < e) pool.emplace_back(fn, b, e);
  }
  for (auto& th : pool) th.join();
}

// The conformal nested lattice of synth_nested: node positions and the
// shared edge subdivision points, in lon/lat.  Regions spanning lattice
// cells [i0, i1) x [j0, j1) (a block, a county or a state) take their ring
// from the same shared points, so every level tiles its parent exactly.
struct NestedLattice {
  std::uint64_t NX = 0, NY = 0, S = 0;
  std::vector<double> gx, gy, hxy, vxy_e;
  // ring of the region [i0, i1) x [j0, j1), counter-clockwise from (i0, j0)
  std::uint64_t ring(std::uint64_t i0, std::uint64_t i1, std::uint64_t j0, std::uint64_t j1,
                     double* out) const {
    std::uint64_t w = 0;
    auto put = [&](double x, double y) {
      out[2 * w] = x;
      out[2 * w + 1] = y;
      ++w;
    };
    auto node = [&](std::uint64_t i, std::uint64_t j) {
      const std::uint64_t k = j * (NX + 1) + i;
      put(gx[k], gy[k]);
    };
    for (std::uint64_t i = i0; i < i1; ++i) {  // bottom, left to right
      node(i, j0);
      const double* h = hxy.data() + 2 * (j0 * NX + i) * (S - 1);
      for (std::uint64_t k = 0; k + 1 < S; ++k) put(h[2 * k], h[2 * k + 1]);
    }
    for (std::uint64_t j = j0; j < j1; ++j) {  // right, bottom to top
      node(i1, j);
      const double* v = vxy_e.data() + 2 * (j * (NX + 1) + i1) * (S - 1);
      for (std::uint64_t k = 0; k + 1 < S; ++k) put(v[2 * k], v[2 * k + 1]);
    }
    for (std::uint64_t i = i1; i-- > i0;) {  // top, right to left
      node(i + 1, j1);
      const double* h = hxy.data() + 2 * (j1 * NX + i) * (S - 1);
      for (std::uint64_t k = S - 1; k-- > 0;) put(h[2 * k], h[2 * k + 1]);
    }
    for (std::uint64_t j = j1; j-- > j0;) {  // left, top to bottom
      node(i0, j + 1);
      const double* v = vxy_e.data() + 2 * (j * (NX + 1) + i0) * (S - 1);
      for (std::uint64_t k = S - 1; k-- > 0;) put(v[2 * k], v[2 * k + 1]);
    }
    return w;
  }
};

bool build_nested(std::uint32_t sx, std::uint32_t sy, std::uint32_t cx, std::uint32_t cy,
                  std::uint32_t bx, std::uint32_t by, std::uint32_t segs, double jitter,
                  double sigma, double x0, double x1, double y0, double y1, std::uint64_t seed,
                  int threads, NestedLattice& LAT) {
  if (!sx || !sy || !cx || !cy || !bx || !by || !segs) return false;
  const std::uint64_t NX = std::uint64_t{sx} * cx * bx, NY = std::uint64_t{sy} * cy * by;
  const std::uint64_t S = segs;
  const std::uint64_t CX = std::uint64_t{cx} * bx, CY = std::uint64_t{cy} * by;  // blocks per state
  const double cw = (x1 - x0) / static_cast<double>(NX);
  const double ch = (y1 - y0) / static_cast<double>(NY);
  auto map_x = [&](double u) { return x0 + u * cw; };
  auto map_y = [&](double v) { return y0 + v * ch; };
  // state corners (lattice units of blocks)
  std::vector<double> su((sx + 1) * (sy + 1)), sv((sx + 1) * (sy + 1));
  for (std::uint32_t j = 0; j <= sy; ++j)
    for (std::uint32_t i = 0; i <= sx; ++i) {
      const std::uint64_t k = std::uint64_t{j} * (sx + 1) + i;
      double u = static_cast<double>(i * CX), v = static_cast<double>(j * CY);
      if (i > 0 && i < sx && j > 0 && j < sy && jitter > 0) {
        u += jitter * CX * (2.0 * unit(draw(seed, 31, 2 * k)) - 1.0);
        v += jitter * CY * (2.0 * unit(draw(seed, 31, 2 * k + 1)) - 1.0);
      }
      su[k] = u;
      sv[k] = v;
    }
  // county corners: global county lattice (sx*cx + 1) x (sy*cy + 1)
  const std::uint64_t KX = std::uint64_t{sx} * cx, KY = std::uint64_t{sy} * cy;
  std::vector<double> ku((KX + 1) * (KY + 1)), kv((KX + 1) * (KY + 1));
  auto bilerp = [](const double* q, double a, double b) {  // q: 00, 10, 01, 11
    return (1 - a) * (1 - b) * q[0] + a * (1 - b) * q[1] + (1 - a) * b * q[2] + a * b * q[3];
  };
  parallel_for(KY + 1, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t J = jb; J < je; ++J)
      for (std::uint64_t I = 0; I <= KX; ++I) {
        const std::uint64_t si = std::min<std::uint64_t>(I / cx, sx - 1), sj = std::min<std::uint64_t>(J / cy, sy - 1);
        const double a = static_cast<double>(I - si * cx) / cx, b = static_cast<double>(J - sj * cy) / cy;
        const std::uint64_t c00 = sj * (sx + 1) + si;
        const double qu[4] = {su[c00], su[c00 + 1], su[c00 + sx + 1], su[c00 + sx + 2]};
        const double qv[4] = {sv[c00], sv[c00 + 1], sv[c00 + sx + 1], sv[c00 + sx + 2]};
        double u = bilerp(qu, a, b), v = bilerp(qv, a, b);
        const bool on_state_edge = (I % cx == 0) || (J % cy == 0);
        if (!on_state_edge && jitter > 0) {
          const std::uint64_t k = J * (KX + 1) + I;
          u += jitter * bx * (2.0 * unit(draw(seed, 32, 2 * k)) - 1.0);
          v += jitter * by * (2.0 * unit(draw(seed, 32, 2 * k + 1)) - 1.0);
        }
        ku[J * (KX + 1) + I] = u;
        kv[J * (KX + 1) + I] = v;
      }
  });
  // block lattice nodes (global), lattice units
  std::vector<double> lu((NX + 1) * (NY + 1)), lv((NX + 1) * (NY + 1));
  parallel_for(NY + 1, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t J = jb; J < je; ++J)
      for (std::uint64_t I = 0; I <= NX; ++I) {
        const std::uint64_t ki = std::min<std::uint64_t>(I / bx, KX - 1), kj = std::min<std::uint64_t>(J / by, KY - 1);
        const double a = static_cast<double>(I - ki * bx) / bx, b = static_cast<double>(J - kj * by) / by;
        const std::uint64_t c00 = kj * (KX + 1) + ki;
        const double qu[4] = {ku[c00], ku[c00 + 1], ku[c00 + KX + 1], ku[c00 + KX + 2]};
        const double qv[4] = {kv[c00], kv[c00 + 1], kv[c00 + KX + 1], kv[c00 + KX + 2]};
        double u = bilerp(qu, a, b), v = bilerp(qv, a, b);
        const bool on_county_edge = (I % bx == 0) || (J % by == 0);
        if (!on_county_edge && jitter > 0) {
          const std::uint64_t k = J * (NX + 1) + I;
          u += jitter * (2.0 * unit(draw(seed, kStreamJitter, 2 * k)) - 1.0);
          v += jitter * (2.0 * unit(draw(seed, kStreamJitter, 2 * k + 1)) - 1.0);
        }
        lu[J * (NX + 1) + I] = u;
        lv[J * (NX + 1) + I] = v;
      }
  });
  // edge subdivision points (lon/lat), shared by both neighbours
  const std::uint64_t nh = NX * (NY + 1), nv = (NX + 1) * NY;
  std::vector<double>& hxy = LAT.hxy;
  std::vector<double>& vxy_e = LAT.vxy_e;
  hxy.assign(2 * nh * (S - 1) + 2, 0.0);
  vxy_e.assign(2 * nv * (S - 1) + 2, 0.0);
  auto subdivide = [&](double au, double av, double bu, double bv, bool border,
                       std::uint64_t stream, std::uint64_t e, double* dst) {
    const double du = bu - au, dv = bv - av;
    const double len = std::sqrt(du * du + dv * dv);
    const double nu = len > 0 ? -dv / len : 0.0, nvv = len > 0 ? du / len : 0.0;
    for (std::uint64_t k = 1; k < S; ++k) {
      const double t = static_cast<double>(k) / static_cast<double>(S);
      double u = au + du * t, v = av + dv * t;
      if (!border && sigma > 0.0) {
        const std::uint64_t idx = 2 * (e * S + k);
        const double d = sigma * gauss(draw(seed, stream, idx), draw(seed, stream, idx + 1));
        u += d * nu;
        v += d * nvv;
      }
      dst[2 * (k - 1)] = map_x(u);
      dst[2 * (k - 1) + 1] = map_y(v);
    }
  };
  parallel_for(NY + 1, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t j = jb; j < je; ++j)
      for (std::uint64_t i = 0; i < NX; ++i) {
        const std::uint64_t e = j * NX + i, a = j * (NX + 1) + i;
        subdivide(lu[a], lv[a], lu[a + 1], lv[a + 1], j == 0 || j == NY, kStreamHEdge, e,
                  hxy.data() + 2 * e * (S - 1));
      }
  });
  parallel_for(NY, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t j = jb; j < je; ++j)
      for (std::uint64_t i = 0; i <= NX; ++i) {
        const std::uint64_t e = j * (NX + 1) + i, a = e;
        subdivide(lu[a], lv[a], lu[a + NX + 1], lv[a + NX + 1], i == 0 || i == NX, kStreamVEdge, e,
                  vxy_e.data() + 2 * e * (S - 1));
      }
  });
  std::vector<double>& gx = LAT.gx;
  std::vector<double>& gy = LAT.gy;
  gx.assign((NX + 1) * (NY + 1), 0.0);
  gy.assign((NX + 1) * (NY + 1), 0.0);
  for (std::uint64_t j = 0; j <= NY; ++j)
    for (std::uint64_t i = 0; i <= NX; ++i) {
      const std::uint64_t k = j * (NX + 1) + i;
      gx[k] = (i == 0) ? x0 : (i == NX) ? x1 : map_x(lu[k]);
      gy[k] = (j == 0) ? y0 : (j == NY) ? y1 : map_y(lv[k]);
    }
  std::vector<double>().swap(lu);
  std::vector<double>().swap(lv);
  LAT.NX = NX;
  LAT.NY = NY;
  LAT.S = S;
  return true;
}

}  // namespace

extern "C" {

// Jittered-grid tiling (BASELINE configs 1, 2, 4).  Geometry is generated in
// lattice units (one tile = 1 x 1) and mapped affinely onto [x0,x1]x[y0,y1]:
//   * lattice nodes (i, j), 0<=i<=nx, 0<=j<=ny; interior nodes move by
//     U(-jitter, +jitter) per axis; border nodes stay on the domain box;
//   * every lattice edge is split into `segs` segments; the segs-1 interior
//     points are displaced perpendicular to the (jittered) edge by
//     N(0, sigma) lattice units; outer-border edges are not displaced, so the
//     union of the tiles is exactly the domain box;
//   * tile (i, j) has id j*nx + i (row-major) and one CCW ring: bottom edge
//     forward, right edge up, top edge backward, left edge down; shared
//     points are computed once and copied, so neighbours share them bitwise.
// Outputs: vxy[2 * 4*segs*nx*ny], ring_off[nx*ny + 1], poly_ring[nx*ny + 1].
int synth_tiling(std::uint32_t nx, std::uint32_t ny, std::uint32_t segs,
                 double jitter, double sigma, double x0, double x1, double y0,
                 double y1, std::uint64_t seed, int threads, double* vxy,
                 std::uint64_t* ring_off, std::uint64_t* poly_ring) {
  if (nx == 0 || ny == 0 || segs == 0) return 1;
  const std::uint64_t NX = nx, NY = ny, S = segs;
  const double cw = (x1 - x0) / static_cast<double>(nx);
  const double ch = (y1 - y0) / static_cast<double>(ny);
  auto map_x = [&](double u) { return x0 + u * cw; };
  auto map_y = [&](double v) { return y0 + v * ch; };

  // lattice nodes, lattice units
  std::vector<double> lu((NX + 1) * (NY + 1)), lv((NX + 1) * (NY + 1));
  parallel_for(NY + 1, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t j = jb; j < je; ++j) {
      for (std::uint64_t i = 0; i <= NX; ++i) {
        const std::uint64_t k = j * (NX + 1) + i;
        double u = static_cast<double>(i), v = static_cast<double>(j);
        if (i > 0 && i < NX && j > 0 && j < NY && jitter > 0.0) {
          u += jitter * (2.0 * unit(draw(seed, kStreamJitter, 2 * k)) - 1.0);
          v += jitter * (2.0 * unit(draw(seed, kStreamJitter, 2 * k + 1)) - 1.0);
        }
        lu[k] = u;
        lv[k] = v;
      }
    }
  });
  // interior points of horizontal edges (i,j)->(i+1,j): NX*(NY+1) edges,
  // vertical edges (i,j)->(i,j+1): (NX+1)*NY edges; S-1 points each, lon/lat
  const std::uint64_t nh = NX * (NY + 1), nv = (NX + 1) * NY;
  std::vector<double> hxy(2 * nh * (S - 1) + 2), vxy_e(2 * nv * (S - 1) + 2);
  auto subdivide = [&](double au, double av, double bu, double bv, bool border,
                       std::uint64_t stream, std::uint64_t e, double* dst) {
    const double du = bu - au, dv = bv - av;
    const double len = std::sqrt(du * du + dv * dv);
    const double nu = len > 0 ? -dv / len : 0.0, nvv = len > 0 ? du / len : 0.0;
    for (std::uint64_t k = 1; k < S; ++k) {
      const double t = static_cast<double>(k) / static_cast<double>(S);
      double u = au + du * t, v = av + dv * t;
      if (!border && sigma > 0.0) {
        const std::uint64_t idx = 2 * (e * S + k);
        const double d = sigma * gauss(draw(seed, stream, idx), draw(seed, stream, idx + 1));
        u += d * nu;
        v += d * nvv;
      }
      dst[2 * (k - 1)] = map_x(u);
      dst[2 * (k - 1) + 1] = map_y(v);
    }
  };
  parallel_for(NY + 1, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t j = jb; j < je; ++j)
      for (std::uint64_t i = 0; i < NX; ++i) {
        const std::uint64_t e = j * NX + i;
        const std::uint64_t a = j * (NX + 1) + i, b = a + 1;
        subdivide(lu[a], lv[a], lu[b], lv[b], j == 0 || j == NY, kStreamHEdge, e,
                  hxy.data() + 2 * e * (S - 1));
      }
  });
  parallel_for(NY, threads, [&](std::uint64_t jb, std::uint64_t je) {
    for (std::uint64_t j = jb; j < je; ++j)
      for (std::uint64_t i = 0; i <= NX; ++i) {
        const std::uint64_t e = j * (NX + 1) + i;
        const std::uint64_t a = j * (NX + 1) + i, b = a + (NX + 1);
        subdivide(lu[a], lv[a], lu[b], lv[b], i == 0 || i == NX, kStreamVEdge, e,
                  vxy_e.data() + 2 * e * (S - 1));
      }
  });
  // corner nodes in lon/lat (border nodes land exactly on x0/x1/y0/y1)
  std::vector<double> cx((NX + 1) * (NY + 1)), cy((NX + 1) * (NY + 1));
  for (std::uint64_t j = 0; j <= NY; ++j)
    for (std::uint64_t i = 0; i <= NX; ++i) {
      const std::uint64_t k = j * (NX + 1) + i;
      cx[k] = (i == 0) ? x0 : (i == NX) ? x1 : map_x(lu[k]);
      cy[k] = (j == 0) ? y0 : (j == NY) ? y1 : map_y(lv[k]);
    }
  const std::uint64_t per_poly = 4 * S;
  parallel_for(NX * NY, threads, [&](std::uint64_t pb, std::uint64_t pe) {
    for (std::uint64_t p = pb; p < pe; ++p) {
      const std::uint64_t i = p % NX, j = p / NX;
      double* out = vxy + 2 * p * per_poly;
      std::uint64_t w = 0;
      auto put = [&](double x, double y) {
        out[2 * w] = x;
        out[2 * w + 1] = y;
        ++w;
      };
      const std::uint64_t c00 = j * (NX + 1) + i, c10 = c00 + 1,
                          c01 = c00 + (NX + 1), c11 = c01 + 1;
      const double* hb = hxy.data() + 2 * (j * NX + i) * (S - 1);        // bottom
      const double* ht = hxy.data() + 2 * ((j + 1) * NX + i) * (S - 1);  // top
      const double* vl = vxy_e.data() + 2 * (j * (NX + 1) + i) * (S - 1);
      const double* vr = vxy_e.data() + 2 * (j * (NX + 1) + i + 1) * (S - 1);
      put(cx[c00], cy[c00]);
      for (std::uint64_t k = 0; k + 1 < S; ++k) put(hb[2 * k], hb[2 * k + 1]);
      put(cx[c10], cy[c10]);
      for (std::uint64_t k = 0; k + 1 < S; ++k) put(vr[2 * k], vr[2 * k + 1]);
      put(cx[c11], cy[c11]);
      for (std::uint64_t k = S - 1; k-- > 0;) put(ht[2 * k], ht[2 * k + 1]);
      put(cx[c01], cy[c01]);
      for (std::uint64_t k = S - 1; k-- > 0;) put(vl[2 * k], vl[2 * k + 1]);
      ring_off[p] = p * per_poly;
      poly_ring[p] = p;
    }
  });
  ring_off[NX * NY] = NX * NY * per_poly;
  poly_ring[NX * NY] = NX * NY;
  return 0;
}

// Three-level nested tiling (BASELINE config 3): sx x sy states, each split
// into cx x cy counties, each split into bx x by blocks (the leaves).  One
// global block lattice of (sx*cx*bx + 1) x (sy*cy*by + 1) nodes is placed
// hierarchically, in lattice units:
//   * state corners are jittered by U(+-jitter) state cells (interior only);
//   * county corners are bilinear in their state's four corners, then
//     jittered by U(+-jitter) county cells unless they lie on a state edge,
//     where they stay on that (straight) edge;
//   * block corners likewise inside their county, jittered by U(+-jitter)
//     block cells unless on a county edge.
// So every level is a jittered tiling conformal to (clipped exactly to) its
// parent.  Block edges are split into `segs` segments whose interior points
// are displaced perpendicular by N(0, sigma) block cells (not on the outer
// border), shared bitwise by the two blocks of an edge.  Leaves are written
// in collect_leaves order (hierarchy.hpp:76-91): state (row-major), county
// within state (row-major), block within county (row-major); scb receives
// (state, county, block) per leaf.
int synth_nested(std::uint32_t sx, std::uint32_t sy, std::uint32_t cx, std::uint32_t cy,
                 std::uint32_t bx, std::uint32_t by, std::uint32_t segs, double jitter,
                 double sigma, double x0, double x1, double y0, double y1, std::uint64_t seed,
                 int threads, double* vxy, std::uint64_t* ring_off, std::uint64_t* poly_ring,
                 std::uint32_t* scb) {
  NestedLattice LAT;
  if (!build_nested(sx, sy, cx, cy, bx, by, segs, jitter, sigma, x0, x1, y0, y1, seed, threads, LAT)) return 1;
  const std::uint64_t NX = LAT.NX, NY = LAT.NY, S = LAT.S;
  const std::uint64_t CX = std::uint64_t{cx} * bx, CY = std::uint64_t{cy} * by;  // blocks per state
  const std::vector<double>& gx = LAT.gx;
  const std::vector<double>& gy = LAT.gy;
  const std::vector<double>& hxy = LAT.hxy;
  const std::vector<double>& vxy_e = LAT.vxy_e;
  const std::uint64_t per_poly = 4 * S;
  const std::uint64_t P = NX * NY;
  const std::uint64_t per_state = CX * CY, per_county = std::uint64_t{bx} * by;
  parallel_for(P, threads, [&](std::uint64_t pb, std::uint64_t pe) {
    for (std::uint64_t p = pb; p < pe; ++p) {
      // leaf p in collect_leaves order -> (state, county, block) -> lattice cell (i, j)
      const std::uint64_t s = p / per_state, rem = p % per_state;
      const std::uint64_t c = rem / per_county, b = rem % per_county;
      const std::uint64_t si = s % sx, sj = s / sx, ci = c % cx, cj = c / cx, bi = b % bx, bj = b / bx;
      const std::uint64_t i = (si * cx + ci) * bx + bi, j = (sj * cy + cj) * by + bj;
      double* out = vxy + 2 * p * per_poly;
      std::uint64_t w = 0;
      auto put = [&](double x, double y) {
        out[2 * w] = x;
        out[2 * w + 1] = y;
        ++w;
      };
      const std::uint64_t c00 = j * (NX + 1) + i, c10 = c00 + 1, c01 = c00 + (NX + 1), c11 = c01 + 1;
      const double* hb = hxy.data() + 2 * (j * NX + i) * (S - 1);
      const double* ht = hxy.data() + 2 * ((j + 1) * NX + i) * (S - 1);
      const double* vl = vxy_e.data() + 2 * (j * (NX + 1) + i) * (S - 1);
      const double* vr = vxy_e.data() + 2 * (j * (NX + 1) + i + 1) * (S - 1);
      put(gx[c00], gy[c00]);
      for (std::uint64_t k = 0; k + 1 < S; ++k) put(hb[2 * k], hb[2 * k + 1]);
      put(gx[c10], gy[c10]);
      for (std::uint64_t k = 0; k + 1 < S; ++k) put(vr[2 * k], vr[2 * k + 1]);
      put(gx[c11], gy[c11]);
      for (std::uint64_t k = S - 1; k-- > 0;) put(ht[2 * k], ht[2 * k + 1]);
      put(gx[c01], gy[c01]);
      for (std::uint64_t k = S - 1; k-- > 0;) put(vl[2 * k], vl[2 * k + 1]);
      ring_off[p] = p * per_poly;
      poly_ring[p] = p;
      if (scb) {
        scb[3 * p] = static_cast<std::uint32_t>(s);
        scb[3 * p + 1] = static_cast<std::uint32_t>(c);
        scb[3 * p + 2] = static_cast<std::uint32_t>(b);
      }
    }
  });
  ring_off[P] = P * per_poly;
  poly_ring[P] = P;
  return 0;
}

// Uniform points over box4 = {x0, x1, y0, y1}; point k of the stream is
// global index offset + k.
// The nested config as a full three-level FMCB hierarchy (the format of
// save_hierarchy, hierarchy.hpp:102-202): state and county polygons are the
// outlines of their lattice cells on the same shared points as the blocks,
// bboxes are the polygon bboxes, FIPS = state+1, county+1, block/10,
// block%10.  For the simple engine (simple_mapper.hpp), which needs every
// level's geometry.  Returns 0, or 1 on bad arguments / IO failure.
int synth_nested_fmcb(std::uint32_t sx, std::uint32_t sy, std::uint32_t cx, std::uint32_t cy,
                      std::uint32_t bx, std::uint32_t by, std::uint32_t segs, double jitter,
                      double sigma, double x0, double x1, double y0, double y1, std::uint64_t seed,
                      int threads, const char* path) {
  NestedLattice LAT;
  if (!build_nested(sx, sy, cx, cy, bx, by, segs, jitter, sigma, x0, x1, y0, y1, seed, threads, LAT)) return 1;
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return 1;
  bool ok = true;
  auto put = [&](const void* p, std::size_t n) { ok = ok && std::fwrite(p, 1, n, f) == n; };
  auto u16 = [&](std::uint16_t v) { put(&v, 2); };
  auto u32 = [&](std::uint32_t v) { put(&v, 4); };
  auto u64 = [&](std::uint64_t v) { put(&v, 8); };
  std::vector<double> ring;
  auto region = [&](std::int64_t fp, const char* fips, std::uint64_t i0, std::uint64_t i1,
                    std::uint64_t j0, std::uint64_t j1) {
    ring.resize(2 * 2 * ((i1 - i0) + (j1 - j0)) * LAT.S);
    const std::uint64_t nv = LAT.ring(i0, i1, j0, j1, ring.data());
    double bx0 = ring[0], bx1 = ring[0], by0 = ring[1], by1 = ring[1];
    for (std::uint64_t k = 0; k < nv; ++k) {
      bx0 = std::min(bx0, ring[2 * k]);
      bx1 = std::max(bx1, ring[2 * k]);
      by0 = std::min(by0, ring[2 * k + 1]);
      by1 = std::max(by1, ring[2 * k + 1]);
    }
    put(&fp, 8);
    if (fips) put(fips, 12);
    const double bb[4] = {bx0, bx1, by0, by1};
    put(bb, 32);
    u32(static_cast<std::uint32_t>(nv));
    put(ring.data(), 16 * nv);
    u32(1);
    u32(0);
  };
  put("FMCB", 4);
  u16(1);
  u64(std::uint64_t{sx} * sy);
  u64(std::uint64_t{sx} * sy * cx * cy);
  u64(std::uint64_t{sx} * sy * cx * cy * bx * by);
  char fips[16];
  for (std::uint32_t s = 0; s < sx * sy && ok; ++s) {
    const std::uint64_t si = s % sx, sj = s / sx;
    const std::uint64_t CX = std::uint64_t{cx} * bx, CY = std::uint64_t{cy} * by;
    region(s + 1, nullptr, si * CX, (si + 1) * CX, sj * CY, (sj + 1) * CY);
    u32(cx * cy);
    for (std::uint32_t c = 0; c < cx * cy; ++c) {
      const std::uint64_t ci = c % cx, cj = c / cx;
      const std::uint64_t i0 = (si * cx + ci) * bx, j0 = (sj * cy + cj) * by;
      region(c + 1, nullptr, i0, i0 + bx, j0, j0 + by);
      u32(bx * by);
      for (std::uint32_t b = 0; b < bx * by; ++b) {
        const std::uint64_t bi = b % bx, bj = b / bx;
        std::snprintf(fips, sizeof(fips), "%02u%03u%06u%01u", (s + 1) % 100u, (c + 1) % 1000u,
                      (b / 10u) % 1000000u, b % 10u);
        region(b + 1, fips, i0 + bi, i0 + bi + 1, j0 + bj, j0 + bj + 1);
      }
    }
  }
  ok = (std::fclose(f) == 0) && ok;
  return ok ? 0 : 1;
}

int synth_points_uniform(const double* box4, std::uint64_t n, std::uint64_t offset,
                         std::uint64_t seed, int threads, double* out) {
  parallel_for(n, threads, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t k = b; k < e; ++k) synth::uniform_point(seed, offset + k, box4, out + 2 * k);
  });
  return 0;
}

// The clustered mixture's centre table: centres uniform over domain4, in
// generation order k = Zipf rank; cdf[k] = sum_{j<=k} (j+1)^-zipf_s.
// Returns the total weight.  The device generator (synth_gpu.cu) takes the
// same table.
double synth_centre_table(const double* domain4, std::uint64_t seed, std::uint32_t n_centres,
                          double zipf_s, double* cxy, double* cdf) {
  double acc = 0.0;
  for (std::uint32_t k = 0; k < n_centres; ++k) {
    cxy[2 * k] = domain4[0] + (domain4[1] - domain4[0]) * unit(draw(seed, kStreamCentres, 2 * k));
    cxy[2 * k + 1] = domain4[2] + (domain4[3] - domain4[2]) * unit(draw(seed, kStreamCentres, 2 * k + 1));
    acc += std::pow(static_cast<double>(k + 1), -zipf_s);
    cdf[k] = acc;
  }
  return acc;
}

// Clustered mixture (BASELINE configs 2, 3, 5): with probability
// frac_clustered a point is centre_k + N(0, sigma^2 I) degrees, k drawn with
// weight (k+1)^-zipf_s (k = generation order of the centres, which are
// uniform over `domain4`); otherwise uniform over `box4`.  Points that fall
// outside the box are kept (they project to -1), not clamped.
int synth_points_clustered(const double* domain4, const double* box4,
                           std::uint64_t n, std::uint64_t offset,
                           std::uint64_t seed, std::uint32_t n_centres,
                           double sigma, double zipf_s, double frac_clustered,
                           int threads, double* out) {
  if (n_centres == 0) return 1;
  std::vector<double> cxy(2 * n_centres), cdf(n_centres);
  const double acc = synth_centre_table(domain4, seed, n_centres, zipf_s, cxy.data(), cdf.data());
  parallel_for(n, threads, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t k = b; k < e; ++k) {
      synth::clustered_point(seed, offset + k, cxy.data(), cdf.data(), n_centres, acc, sigma,
                             frac_clustered, box4, out + 2 * k);
    }
  });
  return 0;
}

// Near-edge mixture (BASELINE config 4): with probability frac_near a point
// lies on a uniformly chosen edge of a uniformly chosen polygon, displaced
// perpendicular to it (in lattice units of cell size cw x ch) by
// U(-eps_cells, +eps_cells); otherwise uniform over box4.
int synth_points_near_edge(const double* vxy, const std::uint64_t* ring_off,
                           const std::uint64_t* poly_ring, std::uint64_t n_polys,
                           double cw, double ch, double eps_cells,
                           double frac_near, const double* box4,
                           std::uint64_t n, std::uint64_t offset,
                           std::uint64_t seed, int threads, double* out) {
  if (n_polys == 0) return 1;
  parallel_for(n, threads, [&](std::uint64_t b, std::uint64_t e) {
    for (std::uint64_t k = b; k < e; ++k) {
      synth::near_edge_point(seed, offset + k, vxy, ring_off, poly_ring, n_polys, cw, ch, eps_cells,
                             frac_near, box4, out + 2 * k);
    }
  });
  return 0;
}

}  // extern "C"
