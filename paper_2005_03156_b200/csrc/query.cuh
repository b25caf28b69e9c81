// query.cuh -- device side of the projection: point location and the exact
// fp64 crossing-number evaluation of boundary records.
//
// Parity with the reference rests on ray_crosses below evaluating
//   (hi.lon - lo.lon) * (p.lat - lo.lat) - (hi.lat - lo.lat) * (p.lon - lo.lon) > 0
// (geometry.hpp:170-174) as three rounded subtractions, two rounded
// products and one rounded subtraction -- never a fused multiply-add.  The
// __dsub_rn/__dmul_rn intrinsics are never contracted by nvcc, and the
// library is additionally compiled with --fmad=false; tests/test_sass.py
// checks the SASS of every kernel for DFMA.
#pragma once

#include <cstdint>

#include "index_format.h"

namespace fm {

struct KParams {
  const std::uint32_t* __restrict__ grid;
  const std::uint8_t* __restrict__ arena;
  double gx0, gy0, inv_w, inv_h;
  double ax0, ax1, ay0, ay1;  // acceptance box = padded domain intersect world box
  int nx, ny;
};

__device__ __forceinline__ bool ray_crosses(double px, double py, double lx,
                                            double ly, double hx, double hy) {
  const double a = __dmul_rn(__dsub_rn(hx, lx), __dsub_rn(py, ly));
  const double b = __dmul_rn(__dsub_rn(hy, ly), __dsub_rn(px, lx));
  return __dsub_rn(a, b) > 0.0;
}

// Grid entry for p, or kEmpty when p is outside the acceptance box (which
// also rejects NaN: every comparison with NaN is false).
__device__ __forceinline__ std::uint32_t locate(const KParams& P, double px, double py) {
  if (!(px >= P.ax0 && px <= P.ax1 && py >= P.ay0 && py <= P.ay1)) return kEmpty;
  int ix = static_cast<int>(__dmul_rn(__dsub_rn(px, P.gx0), P.inv_w));
  int iy = static_cast<int>(__dmul_rn(__dsub_rn(py, P.gy0), P.inv_h));
  ix = min(max(ix, 0), P.nx - 1);
  iy = min(max(iy, 0), P.ny - 1);
  return __ldg(P.grid + static_cast<std::size_t>(iy) * static_cast<std::size_t>(P.nx) + ix);
}

struct WorkCount {
  unsigned long long boundary = 0, cands = 0, edges = 0;
};

// Resolve a point inside a boundary cell (format: index_format.h).
template <bool kCount>
__device__ __noinline__ int resolve_record(const std::uint8_t* __restrict__ arena,
                                           std::uint32_t entry, double px, double py,
                                           WorkCount& wc) {
  const std::uint8_t* rec = arena + static_cast<std::size_t>(entry & ~kRecordBit) * kRecordAlign;
  const uint4 h = __ldg(reinterpret_cast<const uint4*>(rec));
  const std::uint32_t n_edges = h.x & 0xFFFFu, n_cands = h.x >> 16, n_words = h.y & 0xFFFFu;
  const double2* E = reinterpret_cast<const double2*>(rec + 16);
  const int2* C = reinterpret_cast<const int2*>(rec + record_cands_offset(n_edges));
  const std::uint32_t* Mk =
      reinterpret_cast<const std::uint32_t*>(rec + record_masks_offset(n_edges, n_cands));
  const double* B =
      reinterpret_cast<const double*>(rec + record_breaks_offset(n_edges, n_cands, n_words));
  if (kCount) wc.boundary++;
  if (n_words <= 1) {
    std::uint32_t m = 0;
    for (std::uint32_t k = 0; k < n_edges; ++k) {
      const double2 lo = __ldg(E + 2 * k);
      const double2 hi = __ldg(E + 2 * k + 1);
      if (lo.y < py && py <= hi.y) {
        if (kCount) wc.edges++;
        if (ray_crosses(px, py, lo.x, lo.y, hi.x, hi.y)) m |= 1u << k;
      }
    }
    std::uint32_t boff = 0;
    for (std::uint32_t c = 0; c < n_cands; ++c) {
      const int2 cd = __ldg(C + c);
      const std::uint32_t info = static_cast<std::uint32_t>(cd.y);
      const std::uint32_t nb = info >> 1;
      const std::uint32_t mk = n_words ? __ldg(Mk + c) : 0u;
      std::uint32_t par = (info & 1u) ^ static_cast<std::uint32_t>(__popc(m & mk));
      for (std::uint32_t b = 0; b < nb; ++b) par ^= (py > __ldg(B + boff + b)) ? 1u : 0u;
      boff += nb;
      if (kCount) wc.cands++;
      if (par & 1u) return cd.x;
    }
    return -1;
  }
  // wide record (> 32 edges): evaluate each candidate's edges directly
  std::uint32_t boff = 0;
  for (std::uint32_t c = 0; c < n_cands; ++c) {
    const int2 cd = __ldg(C + c);
    const std::uint32_t info = static_cast<std::uint32_t>(cd.y);
    const std::uint32_t nb = info >> 1;
    std::uint32_t par = info & 1u;
    for (std::uint32_t w = 0; w < n_words; ++w) {
      std::uint32_t bits = __ldg(Mk + static_cast<std::size_t>(c) * n_words + w);
      while (bits) {
        const std::uint32_t k = w * 32 + (__ffs(bits) - 1);
        bits &= bits - 1;
        const double2 lo = __ldg(E + 2 * k);
        const double2 hi = __ldg(E + 2 * k + 1);
        if (lo.y < py && py <= hi.y) {
          if (kCount) wc.edges++;
          if (ray_crosses(px, py, lo.x, lo.y, hi.x, hi.y)) par ^= 1u;
        }
      }
    }
    for (std::uint32_t b = 0; b < nb; ++b) par ^= (py > __ldg(B + boff + b)) ? 1u : 0u;
    boff += nb;
    if (kCount) wc.cands++;
    if (par & 1u) return cd.x;
  }
  return -1;
}

}  // namespace fm
