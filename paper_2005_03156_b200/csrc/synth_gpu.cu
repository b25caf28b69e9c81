// synth_gpu.cu -- the workload point streams generated on the GPU.
//
// Not on the product path: the benchmark generates each rank's shard of a
// config's point stream in HBM (c3 is 16 GB of points per GPU, c5 8B
// points), instead of generating it on host cores and copying it over PCIe.
// Every point is synth_rng.h's function of (seed, index), the same code the
// host generator (synth.cpp) runs, compiled without FMA on both sides, so a
// shard generated here is bit-identical to the host's.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "synth_rng.h"

extern "C" double synth_centre_table(const double* domain4, std::uint64_t seed,
                                     std::uint32_t n_centres, double zipf_s, double* cxy,
                                     double* cdf);

namespace {

struct Box {
  double v[4];
};

__global__ void uniform_kernel(Box box, std::uint64_t n, std::uint64_t offset, std::uint64_t seed,
                               double2* __restrict__ out) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t k = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += stride) {
    double p[2];
    synth::uniform_point(seed, offset + k, box.v, p);
    out[k] = make_double2(p[0], p[1]);
  }
}

__global__ void clustered_kernel(Box box, std::uint64_t n, std::uint64_t offset, std::uint64_t seed,
                                 const double* __restrict__ cxy, const double* __restrict__ cdf,
                                 std::uint32_t n_centres, double acc, double sigma, double frac,
                                 double2* __restrict__ out) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t k = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += stride) {
    double p[2];
    synth::clustered_point(seed, offset + k, cxy, cdf, n_centres, acc, sigma, frac, box.v, p);
    out[k] = make_double2(p[0], p[1]);
  }
}

__global__ void near_edge_kernel(Box box, std::uint64_t n, std::uint64_t offset, std::uint64_t seed,
                                 const double* __restrict__ vxy, const std::uint64_t* __restrict__ ring_off,
                                 const std::uint64_t* __restrict__ poly_ring, std::uint64_t n_polys,
                                 double cw, double ch, double eps, double frac,
                                 double2* __restrict__ out) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t k = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += stride) {
    double p[2];
    synth::near_edge_point(seed, offset + k, vxy, ring_off, poly_ring, n_polys, cw, ch, eps, frac,
                           box.v, p);
    out[k] = make_double2(p[0], p[1]);
  }
}

unsigned grid_for(std::uint64_t n) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const std::uint64_t want = (n + 255) / 256;
  const std::uint64_t cap = static_cast<std::uint64_t>(sms) * 16;
  return static_cast<unsigned>(want < cap ? (want > 0 ? want : 1) : cap);
}

Box mkbox(const double* b) { return Box{{b[0], b[1], b[2], b[3]}}; }

}  // namespace

extern "C" {

// All take a DEVICE output (n interleaved lon/lat pairs) and a cudaStream_t
// (NULL = legacy default stream); asynchronous.  0 ok, 1 bad argument,
// 2 CUDA error.
int synth_points_uniform_dev(const double* box4, std::uint64_t n, std::uint64_t offset,
                             std::uint64_t seed, double* d_out, void* stream) {
  if (!box4 || (n && !d_out)) return 1;
  if (n == 0) return 0;
  uniform_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      mkbox(box4), n, offset, seed, reinterpret_cast<double2*>(d_out));
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int synth_points_clustered_dev(const double* domain4, const double* box4, std::uint64_t n,
                               std::uint64_t offset, std::uint64_t seed, std::uint32_t n_centres,
                               double sigma, double zipf_s, double frac_clustered, double* d_out,
                               void* stream) {
  if (!domain4 || !box4 || n_centres == 0 || (n && !d_out)) return 1;
  if (n == 0) return 0;
  std::vector<double> tab(3ull * n_centres);
  const double acc = synth_centre_table(domain4, seed, n_centres, zipf_s, tab.data(),
                                        tab.data() + 2ull * n_centres);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* d_tab = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&d_tab), tab.size() * 8, s) != cudaSuccess) return 2;
  if (cudaMemcpyAsync(d_tab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice, s) != cudaSuccess) return 2;
  clustered_kernel<<<grid_for(n), 256, 0, s>>>(mkbox(box4), n, offset, seed, d_tab,
                                                d_tab + 2ull * n_centres, n_centres, acc, sigma,
                                                frac_clustered, reinterpret_cast<double2*>(d_out));
  const bool ok = cudaGetLastError() == cudaSuccess;
  cudaFreeAsync(d_tab, s);
  // the host table must outlive the async copy
  if (cudaStreamSynchronize(s) != cudaSuccess) return 2;
  return ok ? 0 : 2;
}

// d_vxy / d_ring_off / d_poly_ring: the soup in DEVICE memory.
int synth_points_near_edge_dev(const double* d_vxy, const std::uint64_t* d_ring_off,
                               const std::uint64_t* d_poly_ring, std::uint64_t n_polys, double cw,
                               double ch, double eps_cells, double frac_near, const double* box4,
                               std::uint64_t n, std::uint64_t offset, std::uint64_t seed,
                               double* d_out, void* stream) {
  if (!box4 || n_polys == 0 || (n && (!d_out || !d_vxy || !d_ring_off || !d_poly_ring))) return 1;
  if (n == 0) return 0;
  near_edge_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      mkbox(box4), n, offset, seed, d_vxy, d_ring_off, d_poly_ring, n_polys, cw, ch, eps_cells,
      frac_near, reinterpret_cast<double2*>(d_out));
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
