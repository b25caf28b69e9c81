// synth_rng.h -- the counter-based random streams of the workload
// generators, shared by the host generator (synth.cpp) and the device one
// (synth_gpu.cu) so both produce the same bits for every point index.
//
// splitmix64 of (seed, stream, index) gives 64 random bits per draw; the
// mapping to [0, 1) is the reference's (synthetic.hpp:32-34:
// (x >> 11) * 2^-53).  The Gaussian variates of the clustered point streams
// use Box-Muller (synthetic.hpp:176-180 uses the same form) with log, sin
// and cos written out below in plain IEEE operations -- no libm, no FMA
// (both sides compile with contraction off) -- so host and device agree bit
// for bit.  They are accurate to a few ulps, far more than a generator
// needs.  Not on the product path.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define SR_HD __host__ __device__ __forceinline__
#else
#define SR_HD inline
#endif

namespace synth {

SR_HD std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

SR_HD std::uint64_t draw(std::uint64_t seed, std::uint64_t stream, std::uint64_t idx) {
  return mix64(mix64(seed * 0x2545F4914F6CDD1Dull + stream) ^ idx);
}

SR_HD double unit(std::uint64_t bits) { return static_cast<double>(bits >> 11) * 0x1.0p-53; }

SR_HD double bits_f64(std::uint64_t b) {
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
}
SR_HD std::uint64_t f64_bits(double d) {
  std::uint64_t b;
  __builtin_memcpy(&b, &d, 8);
  return b;
}

// log(x) for finite x > 0: x = m * 2^e with m in [sqrt(1/2), sqrt(2)),
// log(m) = 2 atanh(s), s = (m - 1) / (m + 1), |s| < 0.1716.
SR_HD double det_log(double x) {
  std::uint64_t b = f64_bits(x);
  int e = static_cast<int>((b >> 52) & 0x7FF);
  if (e == 0) {  // subnormal: scale into the normal range
    x *= 0x1.0p54;
    b = f64_bits(x);
    e = static_cast<int>((b >> 52) & 0x7FF) - 54;
  }
  e -= 1023;
  double m = bits_f64((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);  // [1, 2)
  if (m > 1.4142135623730951) {
    m *= 0.5;
    ++e;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  // 2 (s + s^3/3 + s^5/5 + ...), |s|^2 < 0.0295: 13 terms reach 2^-60
  double p = 1.0 / 27.0;
  p = p * s2 + 1.0 / 25.0;
  p = p * s2 + 1.0 / 23.0;
  p = p * s2 + 1.0 / 21.0;
  p = p * s2 + 1.0 / 19.0;
  p = p * s2 + 1.0 / 17.0;
  p = p * s2 + 1.0 / 15.0;
  p = p * s2 + 1.0 / 13.0;
  p = p * s2 + 1.0 / 11.0;
  p = p * s2 + 1.0 / 9.0;
  p = p * s2 + 1.0 / 7.0;
  p = p * s2 + 1.0 / 5.0;
  p = p * s2 + 1.0 / 3.0;
  p = p * s2 + 1.0;
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double de = static_cast<double>(e);
  return (de * ln2_hi) + ((2.0 * s * p) + de * ln2_lo);
}

// sin and cos of 2*pi*u for u in [0, 1): quadrant q = floor(4u), angle
// r*pi/2 with r = 4u - q in [0, 1) (both exact), Taylor series on [0, pi/2).
SR_HD void det_sincos2pi(double u, double* sn, double* cs) {
  const double f = 4.0 * u;
  const int q = static_cast<int>(f);
  const double t = (f - static_cast<double>(q)) * 1.5707963267948966;
  const double t2 = t * t;
  // sin t = t (1 - t^2/3! + t^4/5! - ...), cos t = 1 - t^2/2! + ...; t < 1.571
  // Horner in t2 for sin: coefficients (-1)^k / (2k+1)!, k = 0..10
  double s = -1.0 / 51090942171709440000.0;       // -1/21!
  s = s * t2 + 1.0 / 121645100408832000.0;        // 1/19!
  s = s * t2 - 1.0 / 355687428096000.0;           // -1/17!
  s = s * t2 + 1.0 / 1307674368000.0;             // 1/15!
  s = s * t2 - 1.0 / 6227020800.0;                // -1/13!
  s = s * t2 + 1.0 / 39916800.0;                  // 1/11!
  s = s * t2 - 1.0 / 362880.0;                    // -1/9!
  s = s * t2 + 1.0 / 5040.0;                      // 1/7!
  s = s * t2 - 1.0 / 120.0;                       // -1/5!
  s = s * t2 + 1.0 / 6.0;                         // 1/3!
  s = t - t * t2 * s;
  double c = 1.0 / 2432902008176640000.0;         // 1/20!
  c = c * t2 - 1.0 / 6402373705728000.0;          // -1/18!
  c = c * t2 + 1.0 / 20922789888000.0;            // 1/16!
  c = c * t2 - 1.0 / 87178291200.0;               // -1/14!
  c = c * t2 + 1.0 / 479001600.0;                 // 1/12!
  c = c * t2 - 1.0 / 3628800.0;                   // -1/10!
  c = c * t2 + 1.0 / 40320.0;                     // 1/8!
  c = c * t2 - 1.0 / 720.0;                       // -1/6!
  c = c * t2 + 1.0 / 24.0;                        // 1/4!
  c = c * t2 - 0.5;                               // -1/2!
  c = 1.0 + t2 * c;
  switch (q & 3) {
    case 0: *sn = s; *cs = c; break;
    case 1: *sn = c; *cs = -s; break;
    case 2: *sn = -s; *cs = -c; break;
    default: *sn = -c; *cs = s; break;
  }
}

// Box-Muller pair from two draws (deterministic form of synth.cpp's gauss2).
SR_HD void gauss2(std::uint64_t b1, std::uint64_t b2, double* a, double* b) {
  const double u1 = 1.0 - unit(b1);  // (0, 1]
  const double u2 = unit(b2);
  const double r2 = -2.0 * det_log(u1);
#ifdef __CUDA_ARCH__
  const double r = __dsqrt_rn(r2 > 0.0 ? r2 : 0.0);
#else
  const double r = __builtin_sqrt(r2 > 0.0 ? r2 : 0.0);
#endif
  double sn, cs;
  det_sincos2pi(u2, &sn, &cs);
  *a = r * cs;
  *b = r * sn;
}

enum : std::uint64_t {
  kStreamJitter = 1,
  kStreamHEdge = 2,
  kStreamVEdge = 3,
  kStreamPoints = 16,
  kStreamCentres = 17,
};

// Point i of the clustered mixture (BASELINE configs 2, 3, 5): with
// probability frac_clustered a Gaussian (sigma degrees) around a Zipf-chosen
// centre (cdf over n_centres, total `acc`), else uniform over box4.
SR_HD void clustered_point(std::uint64_t seed, std::uint64_t i, const double* cxy, const double* cdf,
                           std::uint32_t n_centres, double acc, double sigma, double frac_clustered,
                           const double* box4, double* out) {
  const double u0 = unit(draw(seed, kStreamPoints, 4 * i));
  if (u0 < frac_clustered) {
    const double t = unit(draw(seed, kStreamPoints, 4 * i + 1)) * acc;
    std::uint32_t lo = 0, hi = n_centres;  // upper_bound(cdf, t)
    while (lo < hi) {
      const std::uint32_t mid = lo + (hi - lo) / 2;
      if (cdf[mid] <= t) lo = mid + 1; else hi = mid;
    }
    const std::uint32_t c = lo >= n_centres ? n_centres - 1 : lo;
    double gx, gy;
    gauss2(draw(seed, kStreamPoints, 4 * i + 2), draw(seed, kStreamPoints, 4 * i + 3), &gx, &gy);
    out[0] = cxy[2 * c] + sigma * gx;
    out[1] = cxy[2 * c + 1] + sigma * gy;
  } else {
    out[0] = box4[0] + (box4[1] - box4[0]) * unit(draw(seed, kStreamPoints, 4 * i + 2));
    out[1] = box4[2] + (box4[3] - box4[2]) * unit(draw(seed, kStreamPoints, 4 * i + 3));
  }
}

// Point i of the uniform stream over box4 (config 1).
SR_HD void uniform_point(std::uint64_t seed, std::uint64_t i, const double* box4, double* out) {
  out[0] = box4[0] + (box4[1] - box4[0]) * unit(draw(seed, kStreamPoints, 4 * i + 2));
  out[1] = box4[2] + (box4[3] - box4[2]) * unit(draw(seed, kStreamPoints, 4 * i + 3));
}

// Point i of the near-edge mixture (config 4): with probability frac_near
// on a uniformly chosen edge of a uniformly chosen polygon (first ring),
// displaced perpendicular to it by U(-eps_cells, +eps_cells) cells of size
// cw x ch; otherwise uniform over box4.
SR_HD void near_edge_point(std::uint64_t seed, std::uint64_t i, const double* vxy,
                           const std::uint64_t* ring_off, const std::uint64_t* poly_ring,
                           std::uint64_t n_polys, double cw, double ch, double eps_cells,
                           double frac_near, const double* box4, double* out) {
  const double u0 = unit(draw(seed, kStreamPoints, 4 * i));
  if (u0 < frac_near) {
    const std::uint64_t r1 = draw(seed, kStreamPoints, 4 * i + 1);
    const std::uint64_t r2 = draw(seed, kStreamPoints, 4 * i + 2);
    const std::uint64_t r3 = draw(seed, kStreamPoints, 4 * i + 3);
    std::uint64_t p = static_cast<std::uint64_t>(unit(r1) * static_cast<double>(n_polys));
    if (p > n_polys - 1) p = n_polys - 1;
    const std::uint64_t r = poly_ring[p];
    const std::uint64_t vb = ring_off[r], nvert = ring_off[r + 1] - vb;
    const std::uint64_t ea = vb + (mix64(r1) % nvert);
    const std::uint64_t eb = (ea + 1 < vb + nvert) ? ea + 1 : vb;
    const double ax = vxy[2 * ea], ay = vxy[2 * ea + 1];
    const double bx = vxy[2 * eb], by = vxy[2 * eb + 1];
    const double t = unit(r2);
    const double du = (bx - ax) / cw, dv = (by - ay) / ch;
    const double l2 = du * du + dv * dv;
#ifdef __CUDA_ARCH__
    const double len = __dsqrt_rn(l2);
#else
    const double len = __builtin_sqrt(l2);
#endif
    const double d = eps_cells * (2.0 * unit(r3) - 1.0);
    const double nu = len > 0 ? -dv / len : 0.0, nv = len > 0 ? du / len : 0.0;
    out[0] = ax + (bx - ax) * t + d * nu * cw;
    out[1] = ay + (by - ay) * t + d * nv * ch;
  } else {
    out[0] = box4[0] + (box4[1] - box4[0]) * unit(draw(seed, kStreamPoints, 4 * i + 2));
    out[1] = box4[2] + (box4[3] - box4[2]) * unit(draw(seed, kStreamPoints, 4 * i + 3));
  }
}


}  // namespace synth
