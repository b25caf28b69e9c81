// quick.h -- 32-byte quantised boundary records ("quick records").
//
// A quick record is a lossy, self-certifying copy of one phase-1 leaf slot
// (index_format.h, kind 1): the same candidates, edge masks, c0 bits and
// breakpoint masks, with the chain vertices and breakpoints quantised to
// int16 in the slot's own cell frame.  The stream kernel evaluates it
// inline (one 32-byte gather instead of a queue round trip and a 64-128
// byte slot fetch); every bit it derives carries a rigorous error bound,
// and a point whose answer depends on a bit inside that bound is handed to
// the exact fp64 path (resolve_kernel), which reads slot k itself.  So the
// answer is always the reference's: the quick path only answers when the
// exact predicate's result is provably the one it computed.
//
// Frame.  Local coordinates in quanta: U(x) = ((x - gx0) * inv_w - ix) * 2^13
// for the slot's cell column ix (same for y).  The kernel computes
// (p - gx0) * inv_w in locate anyway; subtracting the integer part is exact,
// so points and vertices go through one monotone map whose real-arithmetic
// counterpart is affine (error ~1e-8 quanta).  Vertices and breakpoints must
// lie within [-4, 4) cells of the cell's corner (int16 range) or the record
// is not emitted (`valid` clear) and the cell goes the exact way.
//
// Error bounds (quanta; derivation in DESIGN.md sec. 5, quick records):
//  * vertex / breakpoint quantisation: |q - X| <= 0.5 (+1e-8);
//    rounding is monotone, so the quantised order of two latitudes never
//    contradicts the true order;
//  * point: fp64 -> fp32 conversion of a value < 2^16: <= 2^-9;
//  * range and breakpoint tests are certain when the point is more than
//    kQuickDelta = 0.6 quanta from the quantised latitude;
//  * crossing: with D = hi - lo (exact), E = p - lo (fp32),
//      |cr_fp32 - cross_true| <= (|Ex|+|Ey|) + 0.51 (|Dx|+|Dy|) + 1.02
//                               + 2^-23 (|Dx Ey| + |Dy Ex|),
//    and the reference's own fp64 evaluation of the sign is exact whenever
//    |cross_true| > 0.01 quanta^2; the kernel uses a bound at least 1.001x
//    this plus 2, so cr > T / cr < -T certify the reference's bit.
//
// Layout (eight u32 words w0..w7, little endian):
//   w0  header: bits 0-2 n_verts (0..5), 3-4 n_cands (1..2), 5-6 n_breaks
//       (0..2), 7-10 chain bits (bit 7+i set: vertex i+1 starts a new
//       chain, so edge i is absent), 11-14 edge mask of candidate 0, 15-18
//       of candidate 1, 19 c0 of cand 0, 20 c0 of cand 1, 21-22 break mask
//       of cand 0, 23-24 of cand 1, 31 valid
//   w1  i32 leaf id of candidate 0 (the smaller id)
//   w2..w6  vertex j: int16 U | int16 V << 16
//   w7  n_cands == 2: i32 leaf id of candidate 1;  else breaks (int16 V each)
//   n_cands == 2 with breakpoints: breaks live in w6 (then n_verts <= 4).
#pragma once

#include <cmath>
#include <cstdint>

#include "index_format.h"

namespace fm {

constexpr std::uint64_t kQuickBytes = 32;
constexpr double kQuickScale = 8192.0;  // quanta per cell (2^13)
constexpr float kQuickDelta = 0.6f;     // range / breakpoint certainty margin (quanta)
constexpr int kQuickUnsure = -3;        // quick_eval: hand the point to the exact path

FM_HD bool quick_quantise(double local_cells, std::int32_t* q) {
  const double s = local_cells * kQuickScale;
  if (!(s > -32768.0 && s < 32767.0)) return false;  // also rejects NaN
  *q = static_cast<std::int32_t>(std::nearbyint(s));
  return true;
}

// Encode phase-1 slot `slot` (128 bytes) of cell (ix, iy) into w[8].  The
// record is marked invalid (w0 = 0) when the slot does not fit the format.
FM_HD void quick_encode(const std::uint8_t* slot, std::int64_t ix, std::int64_t iy, double gx0,
                        double gy0, double inv_w, double inv_h, std::uint32_t* w) {
  for (int k = 0; k < 8; ++k) w[k] = 0;
  const std::uint32_t h = *reinterpret_cast<const std::uint32_t*>(slot);
  const std::uint32_t kind = h & 0xFFu, nv = (h >> 8) & 0xFFu, nc = (h >> 16) & 0xFFu,
                      nb = h >> 24;
  if (kind != kSlotLeaf || nc < 1 || nc > 2 || nv > 5 || nb > 2) return;
  if (nc == 2 && nb > 0 && nv > 4) return;
  const double fx = static_cast<double>(ix), fy = static_cast<double>(iy);
  // vertex offsets in the slot (index_format.h): 16, 32, 48 | 96, 112
  const int voff[5] = {16, 32, 48, 96, 112};
  for (std::uint32_t j = 0; j < nv; ++j) {
    const double* v = reinterpret_cast<const double*>(slot + voff[j]);
    std::int32_t qu, qv;
    if (!quick_quantise((v[0] - gx0) * inv_w - fx, &qu) || !quick_quantise((v[1] - gy0) * inv_h - fy, &qv)) {
      return;
    }
    w[2 + j] = (static_cast<std::uint32_t>(qu) & 0xFFFFu) | (static_cast<std::uint32_t>(qv) << 16);
  }
  // breakpoints: +48 / +80 when n_verts < 3, else +80 / +88
  const int boff[2] = {nv >= 3 ? 80 : 48, nv >= 3 ? 88 : 80};
  std::uint32_t bw = 0;
  for (std::uint32_t j = 0; j < nb; ++j) {
    const double b = *reinterpret_cast<const double*>(slot + boff[j]);
    std::int32_t qb;
    if (!quick_quantise((b - gy0) * inv_h - fy, &qb)) return;
    bw |= (static_cast<std::uint32_t>(qb) & 0xFFFFu) << (16 * j);
  }
  const std::uint32_t chain = nv <= 3 ? 1u : *reinterpret_cast<const std::uint32_t*>(slot + 64);
  const std::uint8_t* mk = slot + 4;    // edge_mask[0..1], info[0..1]
  std::uint32_t hdr = nv | (nc << 3) | (nb << 5) | (((chain >> 1) & 0xFu) << 7);
  for (std::uint32_t c = 0; c < nc; ++c) {
    const std::uint32_t mask = mk[c], info = mk[2 + c];
    if (mask & ~0xFu) return;  // edges 0..3 only (<= 5 vertices)
    hdr |= mask << (11 + 4 * c);
    hdr |= ((info >> 7) & 1u) << (19 + c);
    hdr |= (info & 3u) << (21 + 2 * c);
  }
  w[0] = hdr | 0x80000000u;
  w[1] = *reinterpret_cast<const std::uint32_t*>(slot + 8);
  if (nc == 2) {
    w[7] = *reinterpret_cast<const std::uint32_t*>(slot + 12);
    if (nb > 0) w[6] = bw;
  } else {
    w[7] = bw;
  }
}

// fp32 helpers that are never contracted (device: explicit _rn intrinsics;
// host: built with -ffp-contract=off)
#ifdef __CUDA_ARCH__
#define FMQ_MUL(a, b) __fmul_rn(a, b)
#define FMQ_SUB(a, b) __fsub_rn(a, b)
#define FMQ_ADD(a, b) __fadd_rn(a, b)
#define FMQ_POPC(x) __popc(x)
#else
#define FMQ_POPC(x) __builtin_popcount(x)
#define FMQ_MUL(a, b) ((a) * (b))
#define FMQ_SUB(a, b) ((a) - (b))
#define FMQ_ADD(a, b) ((a) + (b))
#endif

FM_HD float quick_u(std::uint32_t v) { return static_cast<float>(static_cast<std::int16_t>(v & 0xFFFFu)); }
FM_HD float quick_v(std::uint32_t v) { return static_cast<float>(static_cast<std::int16_t>(v >> 16)); }

// Evaluate a quick record at a point with local coordinates (pu, pv) in
// quanta.  Returns the leaf id, -1, or kQuickUnsure.
FM_HD int quick_eval(const std::uint32_t (&w)[8], float pu, float pv) {
  const std::uint32_t h = w[0];
  // valid record, point within 2 cells of the corner (keeps every fp32
  // difference below 2^16 quanta, as the bound assumes)
  if (!(h >> 31) || !(fabsf(pu) < 16384.0f) || !(fabsf(pv) < 16384.0f)) return kQuickUnsure;
  const std::uint32_t nv = h & 7u, nc = (h >> 3) & 3u, nb = (h >> 5) & 3u;
  std::uint32_t m = 0, unsure = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const std::uint32_t a = w[2 + k], b = w[3 + k];
    const bool present = static_cast<std::uint32_t>(k + 1) < nv && !((h >> (7 + k)) & 1u);
    const float ay = quick_v(a), by = quick_v(b);
    const bool up = ay < by;
    const float lx = up ? quick_u(a) : quick_u(b), ly = up ? ay : by;
    const float hx = up ? quick_u(b) : quick_u(a), hy = up ? by : ay;
    const float dlo = FMQ_SUB(pv, ly), dhi = FMQ_SUB(hy, pv);
    const bool in_sure = dlo > kQuickDelta && dhi > kQuickDelta;
    const bool out_sure = dlo < -kQuickDelta || dhi < -kQuickDelta;
    const float dx = FMQ_SUB(hx, lx), dy = FMQ_SUB(hy, ly);  // exact
    const float ex = FMQ_SUB(pu, lx);
    const float t1 = FMQ_MUL(dx, dlo), t2 = FMQ_MUL(dy, ex);
    const float cr = FMQ_SUB(t1, t2);
    const float lin = FMQ_ADD(FMQ_ADD(fabsf(ex), fabsf(dlo)), FMQ_MUL(0.52f, FMQ_ADD(fabsf(dx), fabsf(dy))));
    const float quad = FMQ_MUL(2.384185791015625e-7f /* 2^-22 */, FMQ_ADD(fabsf(t1), fabsf(t2)));
    const float T = FMQ_ADD(FMQ_MUL(1.001f, FMQ_ADD(lin, quad)), 2.0f);
    const bool bit = in_sure && cr > T;
    const bool amb = !out_sure && (!in_sure || !(cr > T || cr < -T));
    if (present) {
      m |= (bit ? 1u : 0u) << k;
      unsure |= (amb ? 1u : 0u) << k;
    }
  }
  const std::uint32_t bw = nc == 2 ? w[6] : w[7];
  std::uint32_t bm = 0, bunsure = 0;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const float d = FMQ_SUB(pv, quick_v(bw << (16 - 16 * j)));
    if (static_cast<std::uint32_t>(j) < nb) {
      bm |= (d > kQuickDelta ? 1u : 0u) << j;
      bunsure |= (!(d > kQuickDelta) && !(d < -kQuickDelta) ? 1u : 0u) << j;
    }
  }
  // the first candidate (ascending id) with odd parity; every bit that
  // parity depends on must be certain
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if (static_cast<std::uint32_t>(c) < nc) {
      const std::uint32_t mask = (h >> (11 + 4 * c)) & 0xFu;
      const std::uint32_t c0 = (h >> (19 + c)) & 1u;
      const std::uint32_t bmask = (h >> (21 + 2 * c)) & 3u;
      if ((unsure & mask) | (bunsure & bmask)) return kQuickUnsure;
      const std::uint32_t par = c0 ^ FMQ_POPC(m & mask) ^ FMQ_POPC(bm & bmask);
      if (par & 1u) return static_cast<int>(c == 0 ? w[1] : w[7]);
    }
  }
  return -1;
}

}  // namespace fm
