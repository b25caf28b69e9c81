// index_gpu.cu -- the GPU index builder (north star (1)).
//
// Produces exactly the arrays the host builder (index_host.cpp) produces --
// same classification arithmetic (sweep.h, __host__ __device__), same
// dedupe / chaining / slot encoding, same slot order -- so tests can compare
// the two byte for byte.  Pipeline:
//   1. spans_kernel       per leaf: bbox and the grid span it touches
//   2. count/fill kernels per-cell candidate-leaf lists (CSR), then each
//                         cell's list sorted ascending (leaf order matters:
//                         the first containing leaf wins)
//   3. contrib_kernel     one warp per (grid row, leaf): the leaf's edges are
//                         clipped to the row slab once, then for every cell
//                         of the leaf's span the near edges, the constant
//                         parity c0 of the edges right of it and the
//                         breakpoints are written as a fixed 64-byte record
//   4. finalize_kernel    one thread per cell: dedupe edges across leaves,
//                         terminal / hit / empty detection, vertex chains,
//                         slot encoding (run twice: classify, then write)
//   5. cells that need a split or overflow record (beyond one slot) are
//      handed to the host's phase 2 with their candidate lists.
#include <cuda_runtime.h>

#include <chrono>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "index_build.h"
#include "index_format.h"
#include "sweep.h"

namespace fm {
namespace {


struct Contrib {  // 64 bytes
  double br[kBreakCap];                     // breakpoints, ascending
  std::uint32_t pid;
  std::uint8_t c0, n_near, n_breaks, flag;  // flag: does not fit -> host
  std::uint32_t a[kNearCap], c[kNearCap];   // near edges as soup vertex pairs (ring order)
};
static_assert(sizeof(Contrib) == 64, "contribution record is 64 bytes");

struct DevSoup {
  const double* vxy;
  const std::uint64_t* ring_off;
  const std::uint64_t* poly_ring;
  std::uint64_t n_polys;
};

__global__ void spans_kernel(DevSoup s, GridGeom g, PolySpan* spans,
                             unsigned long long* cells_per_poly, unsigned long long* rows_per_poly) {
  const std::uint64_t p = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (p >= s.n_polys) return;
  PolySpan sp{};
  sp.active = 0;
  const std::uint64_t v0 = s.ring_off[s.poly_ring[p]], v1 = s.ring_off[s.poly_ring[p + 1]];
  if (s.poly_ring[p + 1] > s.poly_ring[p]) {
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (std::uint64_t v = v0; v < v1; ++v) {
      const double x = s.vxy[2 * v], y = s.vxy[2 * v + 1];
      x0 = fmin(x0, x);
      x1 = fmax(x1, x);
      y0 = fmin(y0, y);
      y1 = fmax(y1, y);
    }
    polygon_span(g, x0, x1, y0, y1, &sp);
  }
  spans[p] = sp;
  cells_per_poly[p] = sp.active ? static_cast<unsigned long long>((sp.c1 - sp.c0 + 1) * (sp.r1 - sp.r0 + 1)) : 0ull;
  rows_per_poly[p] = sp.active ? static_cast<unsigned long long>(sp.r1 - sp.r0 + 1) : 0ull;
}

__global__ void count_kernel(const PolySpan* spans, std::uint64_t n, std::int64_t nx,
                             unsigned int* cnt) {
  const std::uint64_t p = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (p >= n || !spans[p].active) return;
  const PolySpan sp = spans[p];
  for (std::int64_t r = sp.r0; r <= sp.r1; ++r)
    for (std::int64_t c = sp.c0; c <= sp.c1; ++c) atomicAdd(cnt + r * nx + c, 1u);
}

__global__ void fill_kernel(const PolySpan* spans, std::uint64_t n, std::int64_t nx,
                            const unsigned long long* off, unsigned int* fill, std::uint32_t* cand,
                            const unsigned long long* pair_off, std::uint32_t* pair_pid,
                            std::int32_t* pair_row) {
  const std::uint64_t p = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (p >= n || !spans[p].active) return;
  const PolySpan sp = spans[p];
  for (std::int64_t r = sp.r0; r <= sp.r1; ++r) {
    pair_pid[pair_off[p] + (r - sp.r0)] = static_cast<std::uint32_t>(p);
    pair_row[pair_off[p] + (r - sp.r0)] = static_cast<std::int32_t>(r);
    for (std::int64_t c = sp.c0; c <= sp.c1; ++c) {
      const std::int64_t cell = r * nx + c;
      cand[off[cell] + atomicAdd(fill + cell, 1u)] = static_cast<std::uint32_t>(p);
    }
  }
}

__global__ void sort_cells_kernel(const unsigned long long* off, std::uint64_t n_cells,
                                  std::uint32_t* cand) {
  const std::uint64_t cell = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (cell >= n_cells) return;
  std::uint32_t* a = cand + off[cell];
  const std::uint64_t m = off[cell + 1] - off[cell];
  for (std::uint64_t i = 1; i < m; ++i) {  // insertion sort: lists are short
    const std::uint32_t v = a[i];
    std::uint64_t j = i;
    while (j > 0 && a[j - 1] > v) {
      a[j] = a[j - 1];
      --j;
    }
    a[j] = v;
  }
}

// One warp per (row, leaf) pair.
__global__ void __launch_bounds__(256) contrib_kernel(DevSoup s, GridGeom g, double tol,
                                                      const PolySpan* spans, const std::uint32_t* pair_pid,
                                                      const std::int32_t* pair_row, std::uint64_t n_pairs,
                                                      const unsigned long long* off, const std::uint32_t* cand,
                                                      Contrib* out) {
  __shared__ SlabEdge rel_s[8][kRelCap];
  __shared__ std::uint32_t rel_a[8][kRelCap], rel_c[8][kRelCap];
  __shared__ double brk[8][kBreakRawCap];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const std::uint64_t pair = blockIdx.x * 8ull + wid;
  if (pair >= n_pairs) return;
  const std::uint32_t pid = pair_pid[pair];
  const std::int64_t iy = pair_row[pair];
  const PolySpan sp = spans[pid];
  const double ys0 = cell_y0(g, iy) - g.margin, ys1 = cell_y0(g, iy + 1) + g.margin;
  // slab-relevant edges, in ring order
  int n_rel = 0;
  bool rel_overflow = false;
  for (std::uint64_t r = s.poly_ring[pid]; r < s.poly_ring[pid + 1]; ++r) {
    const std::uint64_t b = s.ring_off[r], e = s.ring_off[r + 1], n = e - b;
    for (std::uint64_t i0 = 0; i0 < n; i0 += 32) {
      const std::uint64_t i = i0 + lane;
      SlabEdge se{};
      bool ok = false;
      std::uint64_t a = 0, c = 0;
      if (i < n) {
        a = b + i;
        c = (i + 1 < n) ? a + 1 : b;
        ok = slab_edge(g, tol, ys0, ys1, s.vxy[2 * a], s.vxy[2 * a + 1], s.vxy[2 * c],
                       s.vxy[2 * c + 1], &se);
      }
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, ok);
      if (ok) {
        const int pos = n_rel + __popc(bal & ((1u << lane) - 1u));
        if (pos < kRelCap) {
          rel_s[wid][pos] = se;
          rel_a[wid][pos] = static_cast<std::uint32_t>(a);
          rel_c[wid][pos] = static_cast<std::uint32_t>(c);
        }
      }
      n_rel += __popc(bal);
    }
  }
  if (n_rel > kRelCap) rel_overflow = true;
  __syncwarp();
  for (std::int64_t ix = sp.c0; ix <= sp.c1; ++ix) {
    const std::int64_t cell = iy * g.nx + ix;
    // rank of pid in the cell's (sorted) candidate list
    const std::uint32_t* cl = cand + off[cell];
    const std::uint64_t cm = off[cell + 1] - off[cell];
    std::uint64_t rank = 0;
    for (std::uint64_t k = lane; k < cm; k += 32) {
      if (cl[k] == pid) rank = k;
    }
    for (int o = 16; o > 0; o >>= 1) rank = max(rank, __shfl_xor_sync(0xFFFFFFFFu, rank, o));
    Contrib* rec = out + off[cell] + rank;
    std::uint32_t c0 = 0;
    int n_near = 0, n_br = 0;
    bool flag = rel_overflow;
    for (int k0 = 0; k0 < min(n_rel, kRelCap); k0 += 32) {
      const int k = k0 + lane;
      bool near = false, right = false;
      SlabEdge se{};
      if (k < min(n_rel, kRelCap)) {
        se = rel_s[wid][k];
        right = se.tlo > ix;
        near = !right && se.thi >= ix;
      }
      // right edges: endpoints below the slab flip c0, inside become breakpoints
      std::uint32_t mybit = 0;
      bool b_lo = false, b_hi = false;
      if (right) {
        if (se.ly < ys0) mybit ^= 1u; else if (se.ly < ys1) b_lo = true;
        if (se.hy < ys0) mybit ^= 1u; else if (se.hy < ys1) b_hi = true;
      }
      c0 ^= __popc(__ballot_sync(0xFFFFFFFFu, mybit != 0u)) & 1u;
      const unsigned blo = __ballot_sync(0xFFFFFFFFu, b_lo), bhi = __ballot_sync(0xFFFFFFFFu, b_hi);
      if (b_lo) {
        const int pos = n_br + __popc(blo & ((1u << lane) - 1u));
        if (pos < kBreakRawCap) brk[wid][pos] = se.ly;
      }
      const int nlo = __popc(blo);
      if (b_hi) {
        const int pos = n_br + nlo + __popc(bhi & ((1u << lane) - 1u));
        if (pos < kBreakRawCap) brk[wid][pos] = se.hy;
      }
      n_br += nlo + __popc(bhi);
      const unsigned bn = __ballot_sync(0xFFFFFFFFu, near);
      if (near) {
        const int pos = n_near + __popc(bn & ((1u << lane) - 1u));
        if (pos < kNearCap) {
          rec->a[pos] = rel_a[wid][k];
          rec->c[pos] = rel_c[wid][k];
        }
      }
      n_near += __popc(bn);
    }
    __syncwarp();
    if (lane == 0) {
      // breakpoints: values of odd multiplicity, ascending (host: toggle set)
      int m = min(n_br, kBreakRawCap);
      if (n_br > kBreakRawCap) flag = true;
      double* v = brk[wid];
      for (int i = 1; i < m; ++i) {
        const double x = v[i];
        int j = i;
        while (j > 0 && v[j - 1] > x) {
          v[j] = v[j - 1];
          --j;
        }
        v[j] = x;
      }
      int nb = 0;
      double keep[kBreakCap] = {0.0, 0.0};
      for (int i = 0; i < m;) {
        int j = i;
        while (j < m && v[j] == v[i]) ++j;
        if ((j - i) & 1) {
          if (nb < kBreakCap) keep[nb] = v[i];
          ++nb;
        }
        i = j;
      }
      if (nb > kBreakCap || n_near > kNearCap) flag = true;
      rec->pid = pid;
      rec->c0 = static_cast<std::uint8_t>(c0);
      rec->n_near = static_cast<std::uint8_t>(min(n_near, kNearCap));
      rec->n_breaks = static_cast<std::uint8_t>(min(nb, kBreakCap));
      rec->flag = flag ? 1 : 0;
      rec->br[0] = keep[0];
      rec->br[1] = keep[1];
    }
    __syncwarp();
  }
}

struct E4 {
  double lx, ly, hx, hy;
};
__device__ __forceinline__ bool same_e4(const E4& a, const E4& b) {
  return __double_as_longlong(a.lx) == __double_as_longlong(b.lx) &&
         __double_as_longlong(a.ly) == __double_as_longlong(b.ly) &&
         __double_as_longlong(a.hx) == __double_as_longlong(b.hx) &&
         __double_as_longlong(a.hy) == __double_as_longlong(b.hy);
}
__device__ __forceinline__ bool same_pt(double ax, double ay, double bx, double by) {
  return __double_as_longlong(ax) == __double_as_longlong(bx) &&
         __double_as_longlong(ay) == __double_as_longlong(by);
}

enum : int { kCellEmpty = 0, kCellHit = 1, kCellSlot = 2, kCellDefer = 3, kCellDouble = 4 };

// Device port of RowWorker::finalize + encode_slot / encode_double_slot
// (phase 1 only).  Returns the cell kind; for kCellHit sets *hit, for
// kCellSlot writes slot[128] and for kCellDouble slot[256] when non-null.
__device__ int finalize_cell(const DevSoup& s, const Contrib* recs, std::uint64_t m,
                             std::uint32_t* hit, std::uint8_t* slot) {
  E4 U[kCellEdges];
  int nU = 0;
  std::uint32_t cid[kCellCands], cc0[kCellCands];
  std::uint8_t ced[kCellCands][kCellEdges];
  int nced[kCellCands];
  double cbr[kCellCands][kBreakCap];
  int cnb[kCellCands];
  int nc = 0;
  for (std::uint64_t q = 0; q < m; ++q) {
    const Contrib& r = recs[q];
    if (r.flag) return kCellDefer;
    int ne = 0;
    std::uint8_t eds[kCellEdges];
    for (int t = 0; t < r.n_near; ++t) {
      const double ax = s.vxy[2ull * r.a[t]], ay = s.vxy[2ull * r.a[t] + 1];
      const double bx = s.vxy[2ull * r.c[t]], by = s.vxy[2ull * r.c[t] + 1];
      E4 E = ay > by ? E4{bx, by, ax, ay} : E4{ax, ay, bx, by};
      int idx = 0;
      while (idx < nU && !same_e4(U[idx], E)) ++idx;
      if (idx == nU) {
        if (nU == kCellEdges) return kCellDefer;
        U[nU++] = E;
      }
      int f = -1;
      for (int k = 0; k < ne; ++k) {
        if (eds[k] == idx) f = k;
      }
      if (f >= 0) {  // even multiplicity cancels (order kept like vector::erase)
        for (int k = f; k + 1 < ne; ++k) eds[k] = eds[k + 1];
        --ne;
      } else {
        eds[ne++] = static_cast<std::uint8_t>(idx);
      }
    }
    if (ne == 0 && r.n_breaks == 0) {
      if (r.c0) {  // terminal
        if (nc == kCellCands) return kCellDefer;
        cid[nc] = r.pid;
        cc0[nc] = 1;
        nced[nc] = 0;
        cnb[nc] = 0;
        ++nc;
        break;
      }
      continue;
    }
    if (nc == kCellCands) return kCellDefer;
    cid[nc] = r.pid;
    cc0[nc] = r.c0;
    nced[nc] = ne;
    for (int k = 0; k < ne; ++k) ced[nc][k] = eds[k];
    cnb[nc] = r.n_breaks;
    cbr[nc][0] = r.br[0];
    cbr[nc][1] = r.br[1];
    ++nc;
  }
  if (nc == 0) return kCellEmpty;
  if (nced[0] == 0 && cnb[0] == 0) {
    *hit = cid[0];
    return kCellHit;
  }
  // remap referenced edges in candidate order
  int remap[kCellEdges];
  for (int k = 0; k < nU; ++k) remap[k] = -1;
  E4 used[kCellEdges];
  int nused = 0;
  for (int c = 0; c < nc; ++c) {
    for (int k = 0; k < nced[c]; ++k) {
      const int e = ced[c][k];
      if (remap[e] < 0) {
        remap[e] = nused;
        used[nused++] = U[e];
      }
      ced[c][k] = static_cast<std::uint8_t>(remap[e]);
    }
  }
  // encode_slot, else encode_double_slot: the same distinct breakpoints and
  // chains, wider capacities
  if (nc > static_cast<int>(kDblMaxCands)) return kCellDefer;
  double ub[kCellCands * kBreakCap];
  int nub = 0;
  for (int c = 0; c < nc; ++c) {
    for (int k = 0; k < cnb[c]; ++k) {
      bool found = false;
      for (int j = 0; j < nub; ++j) found |= ub[j] == cbr[c][k];
      if (!found) ub[nub++] = cbr[c][k];
    }
  }
  if (nub > static_cast<int>(kDblMaxBreaks)) return kCellDefer;
  for (int a = 1; a < nub; ++a) {  // ascending (std::sort)
    const double t = ub[a];
    int b = a - 1;
    while (b >= 0 && ub[b] > t) {
      ub[b + 1] = ub[b];
      --b;
    }
    ub[b + 1] = t;
  }
  // chain_edges (record_encode.h), literal port
  double vx[kDblMaxVerts], vy[kDblMaxVerts];
  int nv = 0;
  std::uint32_t chain_mask = 0;
  int bit_of[kCellEdges];
  bool usedf[kCellEdges];
  for (int k = 0; k < nused; ++k) usedf[k] = false;
  for (int st = 0; st < nused; ++st) {
    if (usedf[st]) continue;
    usedf[st] = true;
    double cx[kCellEdges + 1], cy[kCellEdges + 1];
    int ce[kCellEdges];
    int len = 2, nce = 1;
    cx[0] = used[st].lx;
    cy[0] = used[st].ly;
    cx[1] = used[st].hx;
    cy[1] = used[st].hy;
    ce[0] = st;
    for (bool grew = true; grew;) {
      grew = false;
      for (int k = 0; k < nused; ++k) {
        if (usedf[k]) continue;
        const E4& e = used[k];
        const double tx = cx[len - 1], ty = cy[len - 1], hx0 = cx[0], hy0 = cy[0];
        if (same_pt(e.lx, e.ly, tx, ty)) {
          cx[len] = e.hx;
          cy[len] = e.hy;
          ++len;
          ce[nce++] = k;
        } else if (same_pt(e.hx, e.hy, tx, ty)) {
          cx[len] = e.lx;
          cy[len] = e.ly;
          ++len;
          ce[nce++] = k;
        } else if (same_pt(e.hx, e.hy, hx0, hy0)) {
          for (int j = len; j > 0; --j) {
            cx[j] = cx[j - 1];
            cy[j] = cy[j - 1];
          }
          cx[0] = e.lx;
          cy[0] = e.ly;
          ++len;
          for (int j = nce; j > 0; --j) ce[j] = ce[j - 1];
          ce[0] = k;
          ++nce;
        } else if (same_pt(e.lx, e.ly, hx0, hy0)) {
          for (int j = len; j > 0; --j) {
            cx[j] = cx[j - 1];
            cy[j] = cy[j - 1];
          }
          cx[0] = e.hx;
          cy[0] = e.hy;
          ++len;
          for (int j = nce; j > 0; --j) ce[j] = ce[j - 1];
          ce[0] = k;
          ++nce;
        } else {
          continue;
        }
        usedf[k] = true;
        grew = true;
      }
    }
    if (nv + len > static_cast<int>(kDblMaxVerts)) return kCellDefer;
    chain_mask |= 1u << nv;
    for (int q = 0; q < nce; ++q) bit_of[ce[q]] = nv + q;
    for (int q = 0; q < len; ++q) {
      vx[nv + q] = cx[q];
      vy[nv + q] = cy[q];
    }
    nv += len;
  }
  const bool leaf = nc <= static_cast<int>(kSlotMaxCands) && nub <= static_cast<int>(kSlotMaxBreaks) &&
                    nv <= static_cast<int>(kSlotMaxVerts);
  if (!leaf) {  // double leaf slot (index_format.h, kind 4)
    if (slot) {
      std::uint32_t w[64];
      for (int k = 0; k < 64; ++k) w[k] = 0;
      w[0] = kSlotDouble | (static_cast<std::uint32_t>(nv) << 8) | (static_cast<std::uint32_t>(nc) << 16) |
             (static_cast<std::uint32_t>(nub) << 24);
      w[1] = chain_mask;
      for (int c = 0; c < nc; ++c) {
        w[2 + c] = cid[c];
        std::uint32_t mask = 0;
        for (int k = 0; k < nced[c]; ++k) mask |= 1u << bit_of[ced[c][k]];
        std::uint32_t info = (cc0[c] & 1u) << 7;
        for (int k = 0; k < cnb[c]; ++k) {
          for (int j = 0; j < nub; ++j) info |= cbr[c][k] == ub[j] ? (1u << j) : 0u;
        }
        w[10 + c / 2] |= (mask & 0xFFFFu) << (16 * (c & 1));
        w[14 + c / 4] |= (info & 0xFFu) << (8 * (c & 3));
      }
      for (int j = 0; j < nub; ++j) {
        const unsigned long long b = __double_as_longlong(ub[j]);
        w[16 + 2 * j] = static_cast<std::uint32_t>(b);
        w[17 + 2 * j] = static_cast<std::uint32_t>(b >> 32);
      }
      for (int k = 0; k < nv; ++k) {
        const unsigned long long x = __double_as_longlong(vx[k]), y = __double_as_longlong(vy[k]);
        w[24 + 4 * k] = static_cast<std::uint32_t>(x);
        w[25 + 4 * k] = static_cast<std::uint32_t>(x >> 32);
        w[26 + 4 * k] = static_cast<std::uint32_t>(y);
        w[27 + 4 * k] = static_cast<std::uint32_t>(y >> 32);
      }
      uint4* dst = reinterpret_cast<uint4*>(slot);
      for (int k = 0; k < 16; ++k) dst[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
    }
    return kCellDouble;
  }
  if (slot) {
    std::uint32_t w[32];
    for (int k = 0; k < 32; ++k) w[k] = 0;
    w[0] = kSlotLeaf | (static_cast<std::uint32_t>(nv) << 8) | (static_cast<std::uint32_t>(nc) << 16) |
           (static_cast<std::uint32_t>(nub) << 24);
    w[16] = nv > 3 ? chain_mask : 0u;  // <= 3 vertices: one chain, implied
    for (int c = 0; c < nc; ++c) {
      const int hi = c < 2 ? 0 : 16, j = c & 1;
      w[hi + 2 + j] = cid[c];
      std::uint32_t mask = 0;
      for (int k = 0; k < nced[c]; ++k) mask |= 1u << bit_of[ced[c][k]];
      std::uint32_t info = (cc0[c] & 1u) << 7;
      for (int k = 0; k < cnb[c]; ++k) info |= (cbr[c][k] == ub[0]) ? 1u : 2u;
      w[hi + 1] |= ((mask & 0xFFu) << (8 * j)) | ((info & 0xFFu) << (16 + 8 * j));
    }
    for (int j = 0; j < nub; ++j) {
      const unsigned long long b = __double_as_longlong(ub[j]);
      const int o = nv >= 3 ? 20 + 2 * j : (j == 0 ? 12 : 20);
      w[o] = static_cast<std::uint32_t>(b);
      w[o + 1] = static_cast<std::uint32_t>(b >> 32);
    }
    for (int k = 0; k < nv; ++k) {
      const unsigned long long x = __double_as_longlong(vx[k]), y = __double_as_longlong(vy[k]);
      const int o = k < 3 ? 4 + 4 * k : 24 + 4 * (k - 3);
      w[o] = static_cast<std::uint32_t>(x);
      w[o + 1] = static_cast<std::uint32_t>(x >> 32);
      w[o + 2] = static_cast<std::uint32_t>(y);
      w[o + 3] = static_cast<std::uint32_t>(y >> 32);
    }
    uint4* dst = reinterpret_cast<uint4*>(slot);
    for (int k = 0; k < 8; ++k) dst[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
  }
  return kCellSlot;
}

__global__ void classify_cells_kernel(DevSoup s, const unsigned long long* off, const Contrib* recs,
                                      std::uint64_t n_cells, std::uint32_t* grid,
                                      std::uint8_t* kind) {
  const std::uint64_t cell = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (cell >= n_cells) return;
  std::uint32_t hit = 0;
  const int k = finalize_cell(s, recs + off[cell], off[cell + 1] - off[cell], &hit, nullptr);
  kind[cell] = static_cast<std::uint8_t>(k);
  grid[cell] = k == kCellHit ? hit : kEmpty;
}

__global__ void write_slots_kernel(DevSoup s, const unsigned long long* off, const Contrib* recs,
                                   std::uint64_t n_cells, const std::uint8_t* kind,
                                   const unsigned long long* slot_idx, std::uint32_t* grid,
                                   std::uint8_t* slots) {
  const std::uint64_t cell = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (cell >= n_cells || (kind[cell] != kCellSlot && kind[cell] != kCellDouble)) return;
  std::uint32_t hit = 0;
  const unsigned long long k = slot_idx[cell];
  std::uint8_t* slot = slots + k * kSlotBytes;
  finalize_cell(s, recs + off[cell], off[cell + 1] - off[cell], &hit, slot);
  grid[cell] = slot_entry_hdr(k, *reinterpret_cast<const std::uint32_t*>(slot));
}

__global__ void flag_kernel(const std::uint8_t* kind, std::uint64_t n, int want,
                            unsigned long long* flags) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) flags[i] = kind[i] == want ? 1ull : 0ull;
}

// phase-1 slot positions: a leaf slot takes one slot index, a double two
__global__ void slot_flag_kernel(const std::uint8_t* kind, std::uint64_t n, unsigned long long* flags) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) flags[i] = kind[i] == kCellSlot ? 1ull : (kind[i] == kCellDouble ? 2ull : 0ull);
}

__global__ void compact_kernel(const std::uint8_t* kind, std::uint64_t n, int want,
                               const unsigned long long* pos, long long* out) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n && kind[i] == want) out[pos[i]] = static_cast<long long>(i);
}

// candidate lists of the deferred cells, packed (cand_off = exclusive scan of their lengths)
__global__ void gather_cands_kernel(const long long* cells, std::uint64_t n,
                                    const unsigned long long* off, const std::uint32_t* cand,
                                    const unsigned long long* cand_off, std::uint32_t* out) {
  const std::uint64_t k = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const unsigned long long b = off[cells[k]], e = off[cells[k] + 1];
  for (unsigned long long q = b; q < e; ++q) out[cand_off[k] + (q - b)] = cand[q];
}

__global__ void deferred_len_kernel(const long long* cells, std::uint64_t n,
                                    const unsigned long long* off, unsigned long long* len) {
  const std::uint64_t k = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (k < n) len[k] = off[cells[k] + 1] - off[cells[k]];
  if (k == n) len[k] = 0;
}

__global__ void scatter_kernel(const long long* cells, const std::uint32_t* vals, std::uint64_t n,
                               std::uint32_t* grid) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) grid[cells[i]] = vals[i];
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw RuntimeError(std::string("GPU index build: ") + what + ": " + cudaGetErrorString(e));
}

template <typename T>
void dalloc(DevBuf& b, std::uint64_t n, const char* what) {
  ck(cudaMalloc(&b.p, std::max<std::uint64_t>(n, 1) * sizeof(T)), what);
}

void exclusive_scan_u64(const unsigned long long* in, unsigned long long* out, std::uint64_t n) {
  std::size_t tmp_bytes = 0;
  ck(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, in, out, static_cast<int64_t>(n)), "scan size");
  DevBuf tmp;
  ck(cudaMalloc(&tmp.p, tmp_bytes + 16), "scan tmp");
  ck(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, in, out, static_cast<int64_t>(n)), "scan");
}

__global__ void widen_kernel(const unsigned int* in, unsigned long long* out, std::uint64_t n) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = in[i];
}

inline unsigned grid1d(std::uint64_t n, unsigned b = 256) {
  return static_cast<unsigned>((n + b - 1) / b);
}

}  // namespace

// Builds the index on `device`.  Returns device arrays in `dev_*` (owned by
// the caller) and fills `out` with the geometry, stats and -- when
// keep_host -- host copies for comparison tests.
// cell kinds counted on the device: counts[kind] += cells of that kind
__global__ void kind_count_kernel(const std::uint8_t* kind, std::uint64_t n, unsigned long long* counts) {
  __shared__ unsigned int s[4];
  if (threadIdx.x < 4) s[threadIdx.x] = 0u;
  __syncthreads();
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  unsigned int c[4] = {0u, 0u, 0u, 0u};  // empty, hit, other (boundary), -
  for (std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const std::uint8_t k = kind[i];
    c[k < 2 ? k : 2]++;
  }
  for (int k = 0; k < 4; ++k) {
    if (c[k]) atomicAdd(s + k, c[k]);
  }
  __syncthreads();
  if (threadIdx.x < 4 && s[threadIdx.x]) atomicAdd(counts + threadIdx.x, static_cast<unsigned long long>(s[threadIdx.x]));
}

void build_index_gpu(const Soup& s, const BuildOptions& o, int device, HostIndex& out,
                     std::uint32_t** dev_grid, std::uint8_t** dev_slots, std::uint64_t* slots_len,
                     std::uint8_t** dev_overflow, std::uint64_t* overflow_len) {
  ck(cudaSetDevice(device), "cudaSetDevice");
  double phase_s[6] = {0, 0, 0, 0, 0, 0};
  auto t_mark = std::chrono::steady_clock::now();
  auto lap = [&](int k) {  // wall time of phase k (device work included)
    ck(cudaDeviceSynchronize(), "phase sync");
    const auto now = std::chrono::steady_clock::now();
    phase_s[k] += std::chrono::duration<double>(now - t_mark).count();
    t_mark = now;
  };
  out = HostIndex{};
  out.g = plan_grid(s, o, &out.stats);
  const GridGeom g = out.g;
  const std::uint64_t n_cells = static_cast<std::uint64_t>(g.nx * g.ny);
  const std::uint64_t P = s.n_polys;
  const std::uint64_t V = s.n_rings ? s.ring_off[s.n_rings] : 0;
  // soup on the device
  DevBuf d_vxy, d_ro, d_pr;
  dalloc<double>(d_vxy, 2 * V, "vxy");
  dalloc<std::uint64_t>(d_ro, s.n_rings + 1, "ring_off");
  dalloc<std::uint64_t>(d_pr, P + 1, "poly_ring");
  if (V) ck(cudaMemcpy(d_vxy.p, s.vxy, 16 * V, cudaMemcpyHostToDevice), "upload vxy");
  ck(cudaMemcpy(d_ro.p, s.ring_off, 8 * (s.n_rings + 1), cudaMemcpyHostToDevice), "upload ring_off");
  if (P) ck(cudaMemcpy(d_pr.p, s.poly_ring, 8 * (P + 1), cudaMemcpyHostToDevice), "upload poly_ring");
  DevSoup ds{d_vxy.as<double>(), d_ro.as<std::uint64_t>(), d_pr.as<std::uint64_t>(), P};
  lap(0);
  // 1. spans
  DevBuf d_spans, d_cpp, d_rpp;
  dalloc<PolySpan>(d_spans, P, "spans");
  dalloc<unsigned long long>(d_cpp, P, "cells_per_poly");
  dalloc<unsigned long long>(d_rpp, P + 1, "rows_per_poly");
  if (P) {
    spans_kernel<<<grid1d(P), 256>>>(ds, g, d_spans.as<PolySpan>(), d_cpp.as<unsigned long long>(),
                                      d_rpp.as<unsigned long long>());
    ck(cudaGetLastError(), "spans_kernel");
  }
  // 2. per-cell candidate CSR
  DevBuf d_cnt, d_off, d_fill;
  dalloc<unsigned int>(d_cnt, n_cells, "cnt");
  dalloc<unsigned long long>(d_off, n_cells + 1, "off");
  dalloc<unsigned int>(d_fill, n_cells, "fill");
  ck(cudaMemset(d_cnt.p, 0, 4 * n_cells), "memset cnt");
  ck(cudaMemset(d_fill.p, 0, 4 * n_cells), "memset fill");
  if (P) count_kernel<<<grid1d(P), 256>>>(d_spans.as<PolySpan>(), P, g.nx, d_cnt.as<unsigned int>());
  {
    DevBuf wide;
    dalloc<unsigned long long>(wide, n_cells + 1, "cnt64");
    ck(cudaMemset(wide.p, 0, 8 * (n_cells + 1)), "memset cnt64");
    widen_kernel<<<grid1d(n_cells), 256>>>(d_cnt.as<unsigned int>(), wide.as<unsigned long long>(), n_cells);
    exclusive_scan_u64(wide.as<unsigned long long>(), d_off.as<unsigned long long>(), n_cells + 1);
  }
  unsigned long long n_pairs_cells = 0;
  ck(cudaMemcpy(&n_pairs_cells, d_off.as<unsigned long long>() + n_cells, 8, cudaMemcpyDeviceToHost),
     "read total");
  DevBuf d_pair_off, d_cand;
  dalloc<unsigned long long>(d_pair_off, P + 1, "pair_off");
  if (P) {
    // rows_per_poly has P+1 entries (last = 0) -> exclusive scan gives the total at [P]
    ck(cudaMemset(d_rpp.as<unsigned long long>() + P, 0, 8), "memset rpp tail");
    exclusive_scan_u64(d_rpp.as<unsigned long long>(), d_pair_off.as<unsigned long long>(), P + 1);
  }
  unsigned long long n_pairs = 0;
  if (P) ck(cudaMemcpy(&n_pairs, d_pair_off.as<unsigned long long>() + P, 8, cudaMemcpyDeviceToHost), "pairs");
  dalloc<std::uint32_t>(d_cand, n_pairs_cells, "cand");
  DevBuf d_ppid, d_prow;
  dalloc<std::uint32_t>(d_ppid, n_pairs, "pair_pid");
  dalloc<std::int32_t>(d_prow, n_pairs, "pair_row");
  if (P) {
    fill_kernel<<<grid1d(P), 256>>>(d_spans.as<PolySpan>(), P, g.nx, d_off.as<unsigned long long>(),
                                     d_fill.as<unsigned int>(), d_cand.as<std::uint32_t>(),
                                     d_pair_off.as<unsigned long long>(), d_ppid.as<std::uint32_t>(),
                                     d_prow.as<std::int32_t>());
    ck(cudaGetLastError(), "fill_kernel");
  }
  sort_cells_kernel<<<grid1d(n_cells), 256>>>(d_off.as<unsigned long long>(), n_cells,
                                               d_cand.as<std::uint32_t>());
  ck(cudaGetLastError(), "sort_cells_kernel");
  lap(1);
  // 3. contributions
  DevBuf d_rec;
  dalloc<Contrib>(d_rec, n_pairs_cells, "contributions");
  if (n_pairs) {
    contrib_kernel<<<static_cast<unsigned>((n_pairs + 7) / 8), 256>>>(
        ds, g, classify_tol(g), d_spans.as<PolySpan>(), d_ppid.as<std::uint32_t>(),
        d_prow.as<std::int32_t>(), n_pairs, d_off.as<unsigned long long>(),
        d_cand.as<std::uint32_t>(), d_rec.as<Contrib>());
    ck(cudaGetLastError(), "contrib_kernel");
  }
  lap(2);
  // 4. classify cells, allocate phase-1 slots (row-major), write them
  DevBuf d_grid, d_kind, d_flags, d_pos;
  dalloc<std::uint32_t>(d_grid, n_cells, "grid");
  dalloc<std::uint8_t>(d_kind, n_cells, "kind");
  dalloc<unsigned long long>(d_flags, n_cells + 1, "flags");
  dalloc<unsigned long long>(d_pos, n_cells + 1, "pos");
  classify_cells_kernel<<<grid1d(n_cells, 128), 128>>>(ds, d_off.as<unsigned long long>(), d_rec.as<Contrib>(),
                                                  n_cells, d_grid.as<std::uint32_t>(), d_kind.as<std::uint8_t>());
  ck(cudaGetLastError(), "classify_cells_kernel");
  auto count_kind = [&](int want) {  // want < 0: phase-1 slot indices (slot 1, double 2)
    ck(cudaMemset(d_flags.p, 0, 8 * (n_cells + 1)), "memset flags");
    if (want < 0) {
      slot_flag_kernel<<<grid1d(n_cells), 256>>>(d_kind.as<std::uint8_t>(), n_cells,
                                                 d_flags.as<unsigned long long>());
    } else {
      flag_kernel<<<grid1d(n_cells), 256>>>(d_kind.as<std::uint8_t>(), n_cells, want,
                                            d_flags.as<unsigned long long>());
    }
    exclusive_scan_u64(d_flags.as<unsigned long long>(), d_pos.as<unsigned long long>(), n_cells + 1);
    unsigned long long total = 0;
    ck(cudaMemcpy(&total, d_pos.as<unsigned long long>() + n_cells, 8, cudaMemcpyDeviceToHost), "count");
    return total;
  };
  const unsigned long long n1 = count_kind(-1);
  if (n1 > kMaxSlots) throw RuntimeError("index needs more than 2^29 slots");
  DevBuf d_slots1;
  dalloc<std::uint8_t>(d_slots1, std::max<unsigned long long>(n1, 1) * kSlotBytes, "slots");
  write_slots_kernel<<<grid1d(n_cells, 128), 128>>>(ds, d_off.as<unsigned long long>(), d_rec.as<Contrib>(),
                                               n_cells, d_kind.as<std::uint8_t>(),
                                               d_pos.as<unsigned long long>(), d_grid.as<std::uint32_t>(),
                                               d_slots1.as<std::uint8_t>());
  ck(cudaGetLastError(), "write_slots_kernel");
  // 5. deferred cells -> host phase 2
  const unsigned long long nd = count_kind(kCellDefer);
  std::vector<std::int64_t> cells(nd);
  std::vector<std::uint64_t> cand_off(nd + 1, 0);
  std::vector<std::uint32_t> cand_ids;
  if (nd) {
    DevBuf d_cells;
    dalloc<long long>(d_cells, nd, "deferred cells");
    compact_kernel<<<grid1d(n_cells), 256>>>(d_kind.as<std::uint8_t>(), n_cells, kCellDefer,
                                             d_pos.as<unsigned long long>(), d_cells.as<long long>());
    ck(cudaMemcpy(cells.data(), d_cells.p, 8 * nd, cudaMemcpyDeviceToHost), "deferred cells");
    DevBuf d_len, d_coff, d_cids;
    dalloc<unsigned long long>(d_len, nd + 1, "deferred lens");
    dalloc<unsigned long long>(d_coff, nd + 1, "deferred cand_off");
    deferred_len_kernel<<<grid1d(nd + 1), 256>>>(d_cells.as<long long>(), nd,
                                                 d_off.as<unsigned long long>(),
                                                 d_len.as<unsigned long long>());
    exclusive_scan_u64(d_len.as<unsigned long long>(), d_coff.as<unsigned long long>(), nd + 1);
    ck(cudaMemcpy(cand_off.data(), d_coff.p, 8 * (nd + 1), cudaMemcpyDeviceToHost), "cand_off");
    cand_ids.resize(cand_off[nd]);
    dalloc<std::uint32_t>(d_cids, cand_off[nd], "deferred cands");
    gather_cands_kernel<<<grid1d(nd), 256>>>(d_cells.as<long long>(), nd,
                                             d_off.as<unsigned long long>(), d_cand.as<std::uint32_t>(),
                                             d_coff.as<unsigned long long>(), d_cids.as<std::uint32_t>());
    ck(cudaGetLastError(), "gather_cands_kernel");
    if (cand_off[nd]) {
      ck(cudaMemcpy(cand_ids.data(), d_cids.p, 4 * cand_off[nd], cudaMemcpyDeviceToHost), "cands");
    }
  }
  // stats of the GPU phase (cell kinds), counted on the device
  {
    DevBuf d_kc;
    dalloc<unsigned long long>(d_kc, 4, "kind counts");
    ck(cudaMemset(d_kc.p, 0, 32), "memset kind counts");
    kind_count_kernel<<<1184, 256>>>(d_kind.as<std::uint8_t>(), n_cells, d_kc.as<unsigned long long>());
    ck(cudaGetLastError(), "kind_count_kernel");
    unsigned long long kc[4];
    ck(cudaMemcpy(kc, d_kc.p, 32, cudaMemcpyDeviceToHost), "kind counts");
    out.stats.cells_empty += kc[kCellEmpty];
    out.stats.cells_hit += kc[kCellHit];
    out.stats.cells_boundary += n_cells - kc[kCellEmpty] - kc[kCellHit];
    const unsigned long long n_dbl = count_kind(kCellDouble);
    out.stats.slots_double += n_dbl;
    out.stats.records += n1 - n_dbl;  // a double slot is one record in two slot indices
    out.stats.records_compact += n1 - n_dbl;
  }
  lap(3);
  std::vector<std::uint32_t> grid_h;  // only entries of deferred cells are used
  std::vector<std::uint8_t> slots2, ovf2;
  if (nd) {
    grid_h.assign(n_cells, kEmpty);
    BuildStats st2;
    finish_deferred_cells(s, g, o, cells, cand_off, cand_ids, n1, grid_h, slots2, ovf2, st2);
    out.stats.records += st2.records;
    out.stats.records_overflow += st2.records_overflow;
    out.stats.cells_split += st2.cells_split;
    out.stats.slots_double += st2.slots_double;
    out.stats.records_compact += st2.records_compact;
    out.stats.records_wide += st2.records_wide;
    std::vector<std::uint32_t> vals(nd);
    for (std::uint64_t k = 0; k < nd; ++k) vals[k] = grid_h[static_cast<std::size_t>(cells[k])];
    DevBuf d_c, d_v;
    dalloc<long long>(d_c, nd, "scatter cells");
    dalloc<std::uint32_t>(d_v, nd, "scatter vals");
    ck(cudaMemcpy(d_c.p, cells.data(), 8 * nd, cudaMemcpyHostToDevice), "scatter cells");
    ck(cudaMemcpy(d_v.p, vals.data(), 4 * nd, cudaMemcpyHostToDevice), "scatter vals");
    scatter_kernel<<<grid1d(nd), 256>>>(d_c.as<long long>(), d_v.as<std::uint32_t>(), nd,
                                        d_grid.as<std::uint32_t>());
    ck(cudaGetLastError(), "scatter_kernel");
  }
  lap(4);
  // final device arrays: slots = phase 1 ++ phase 2, overflow (+ zero tail)
  const std::uint64_t n_slots = n1 + slots2.size() / kSlotBytes;
  std::uint8_t* slots = nullptr;
  ck(cudaMalloc(&slots, std::max<std::uint64_t>(n_slots, 1) * kSlotBytes), "slots");
  if (n1) ck(cudaMemcpy(slots, d_slots1.p, n1 * kSlotBytes, cudaMemcpyDeviceToDevice), "slots copy");
  if (!slots2.empty()) {
    ck(cudaMemcpy(slots + n1 * kSlotBytes, slots2.data(), slots2.size(), cudaMemcpyHostToDevice), "slots2");
  }
  if (n_slots == 0) ck(cudaMemset(slots, 0, kSlotBytes), "slots zero");
  ovf2.resize(ovf2.size() + 512, 0);
  std::uint8_t* ovf = nullptr;
  ck(cudaMalloc(&ovf, ovf2.size()), "overflow");
  ck(cudaMemcpy(ovf, ovf2.data(), ovf2.size(), cudaMemcpyHostToDevice), "overflow copy");
  ck(cudaDeviceSynchronize(), "build sync");
  *dev_grid = static_cast<std::uint32_t*>(d_grid.p);
  d_grid.p = nullptr;  // ownership to the caller
  *dev_slots = slots;
  *slots_len = std::max<std::uint64_t>(n_slots, 1) * kSlotBytes;
  *dev_overflow = ovf;
  *overflow_len = ovf2.size();
  out.n_slots = n_slots;
  out.n_phase1_slots = n1;
  lap(5);
  for (int k = 0; k < 6; ++k) out.stats.phase_s[k] = phase_s[k];
}

}  // namespace fm
