// FP64 throughput microbenchmark on the B200 (SURVEY.md sec. 8d asks the
// builder to measure it): independent chains of unfused DADD / DMUL, and
// the exact crossing predicate (2 DADD + 2 DMUL + 1 DADD + DSETP per edge
// test, geometry.hpp:170-174, with dx, dy precomputed) -- the ceiling for
// resolve_kernel's fp64 work.  Build + run: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a --fmad=false tools/exp_fp64.cu -o x && ./x
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void add_mul(double* out, double a, double b) {
  double x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = __dmul_rn(__dadd_rn(x[c], a), b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void edge_tests(int* out, double px0, double py0) {
  // kChains independent (point, edge) tests per iteration, like eval_leaf_slot
  double lx[kChains], ly[kChains], dx[kChains], dy[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    lx[c] = 0.1 * c + threadIdx.x * 1e-7;
    ly[c] = 0.2 * c;
    dx[c] = 1.0 + 0.01 * c;
    dy[c] = 2.0 - 0.01 * c;
  }
  int cnt = 0;
  double px = px0, py = py0;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      const double a = __dmul_rn(dx[c], __dsub_rn(py, ly[c]));
      const double b = __dmul_rn(dy[c], __dsub_rn(px, lx[c]));
      cnt += __dsub_rn(a, b) > 0.0;
    }
    px = __dadd_rn(px, 1e-9);
  }
  if (cnt == -1) out[0] = cnt;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  int* di;
  cudaMalloc(&d, 8);
  cudaMalloc(&di, 4);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  add_mul<<<blocks, threads>>>(d, 1e-12, 1.0000001);
  edge_tests<<<blocks, threads>>>(di, 0.5, 0.5);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventRecord(e0);
  add_mul<<<blocks, threads>>>(d, 1e-12, 1.0000001);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * kChains * kIters * static_cast<double>(blocks) * threads;
  std::printf("{\"kernel\": \"dadd+dmul\", \"fp64_instr_per_s\": %.4g, \"ms\": %.3f}\n", ops / (ms * 1e-3), ms);
  cudaEventRecord(e0);
  edge_tests<<<blocks, threads>>>(di, 0.5, 0.5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double tests = static_cast<double>(kChains) * kIters * blocks * threads;
  std::printf("{\"kernel\": \"edge_test\", \"edge_tests_per_s\": %.4g, \"fp64_instr_per_s\": %.4g, \"ms\": %.3f}\n",
              tests / (ms * 1e-3), 5.0 * tests / (ms * 1e-3), ms);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
