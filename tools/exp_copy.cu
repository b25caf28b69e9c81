// Copy-pattern microbenchmark for the binning scatter: n double2 points read
// and written (16 B/pt each way) plus a 4-byte index stream, in the access
// patterns the scatter uses.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/exp_copy.cu -o /tmp/exp_copy
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kPer, int kStoreKind, bool kBlocks>
__global__ void __launch_bounds__(256) copy_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                   unsigned* __restrict__ pos, std::uint64_t n, std::uint64_t G) {
  const std::uint64_t step = static_cast<std::uint64_t>(kPer) * 256;
  std::uint64_t lo, hi, stride;
  if (kBlocks) {
    lo = n / G * blockIdx.x + (blockIdx.x < n % G ? (std::uint64_t)blockIdx.x : n % G);
    hi = n / G * (blockIdx.x + 1) + (blockIdx.x + 1 < n % G ? (std::uint64_t)blockIdx.x + 1 : n % G);
    stride = step;
  } else {
    lo = blockIdx.x * step;
    hi = n;
    stride = step * gridDim.x;
  }
  for (std::uint64_t i0 = lo + threadIdx.x; i0 < hi; i0 += stride) {
    double2 p[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const std::uint64_t i = i0 + j * 256ull;
      p[j] = i < hi ? __ldcs(in + i) : make_double2(0, 0);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const std::uint64_t i = i0 + j * 256ull;
      if (i < hi) {
        if (kStoreKind == 0) out[i] = p[j];
        if (kStoreKind == 1) __stcs(out + i, p[j]);
        if (kStoreKind == 2) __stcg(out + i, p[j]);
        __stcs(pos + i, static_cast<unsigned>(i));
      }
    }
  }
}

// points scattered into F fronts: point i goes to front i % F, at its rank
// i / F there -- every front advances sequentially, consecutive lanes write
// to different fronts (the binning scatter's pattern with uniform keys)
template <int kPer>
__global__ void __launch_bounds__(256) fronts_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                                     unsigned* __restrict__ pos, std::uint64_t n, unsigned F) {
  const std::uint64_t step = static_cast<std::uint64_t>(kPer) * 256;
  const std::uint64_t per = n / F;
  for (std::uint64_t i0 = blockIdx.x * step + threadIdx.x; i0 < n; i0 += step * gridDim.x) {
    double2 p[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const std::uint64_t i = i0 + j * 256ull;
      p[j] = i < n ? __ldcs(in + i) : make_double2(0, 0);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const std::uint64_t i = i0 + j * 256ull;
      if (i < n) {
        const std::uint64_t d = (i % F) * per + i / F;
        if (d < n) out[d] = p[j];
        __stcs(pos + i, static_cast<unsigned>(d));
      }
    }
  }
}

void run_fronts(unsigned F, const double2* in, double2* out, unsigned* pos, std::uint64_t n, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) fronts_kernel<16><<<grid, 256>>>(in, out, pos, n, F);
  cudaEventRecord(a);
  for (int w = 0; w < 5; ++w) fronts_kernel<16><<<grid, 256>>>(in, out, pos, n, F);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("{\"variant\": \"fronts\", \"F\": %u, \"ms\": %.3f, \"TBps\": %.2f}\n", F, ms, 36.0 * n / ms / 1e9);
}

template <int kPer, int kStoreKind, bool kBlocks>
void run(const char* name, const double2* in, double2* out, unsigned* pos, std::uint64_t n, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) copy_kernel<kPer, kStoreKind, kBlocks><<<grid, 256>>>(in, out, pos, n, grid);
  cudaEventRecord(a);
  for (int w = 0; w < 5; ++w) copy_kernel<kPer, kStoreKind, kBlocks><<<grid, 256>>>(in, out, pos, n, grid);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  printf("{\"variant\": \"%s\", \"grid\": %d, \"ms\": %.3f, \"TBps\": %.2f}\n", name, grid, ms, 36.0 * n / ms / 1e9);
}

int main() {
  const std::uint64_t n = 1000000000ull;
  double2 *in, *out;
  unsigned* pos;
  cudaMalloc(&in, n * 16);
  cudaMalloc(&out, n * 16);
  cudaMalloc(&pos, n * 4);
  cudaMemset(in, 0, n * 16);
  int sms = 148;
  run<16, 0, true>("blocks per16 default-store", in, out, pos, n, sms * 2);
  run<16, 1, true>("blocks per16 stcs", in, out, pos, n, sms * 2);
  run<16, 2, true>("blocks per16 stcg", in, out, pos, n, sms * 2);
  run<8, 0, true>("blocks per8 default-store", in, out, pos, n, sms * 4);
  run<4, 0, true>("blocks per4 default-store", in, out, pos, n, sms * 8);
  run<16, 0, false>("stride per16 default-store", in, out, pos, n, sms * 2);
  run<8, 0, false>("stride per8 default-store", in, out, pos, n, sms * 4);
  run<4, 0, false>("stride per4 default-store", in, out, pos, n, sms * 8);
  run<4, 1, false>("stride per4 stcs", in, out, pos, n, sms * 8);
  run<2, 0, false>("stride per2 default-store", in, out, pos, n, sms * 16);
  for (unsigned F : {1u, 4u, 16u, 64u, 162u, 256u, 630u, 1024u, 4096u}) run_fronts(F, in, out, pos, n, sms * 2);
  return 0;
}
