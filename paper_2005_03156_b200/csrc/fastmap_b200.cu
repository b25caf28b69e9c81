// fastmap_b200.cu -- the C-ABI (include/fastmap_b200.h) and the sm_100a
// projection kernel.
//
// Kernel shape: a persistent grid sized to the SM count
// times resident CTAs; each thread walks the point stream with stride
// gridDim*blockDim, U points at a time so U independent 16-byte point loads,
// U cell-entry gathers and U 4-byte id stores are in flight per thread.
// Points in true-hit / empty cells (the large majority) cost one coalesced
// read of the point, one L2-resident cell entry and one coalesced write.
// Points in boundary cells walk one contiguous record (resolve_record).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/fastmap_b200.h"
#include "index_build.h"
#include "index_format.h"
#include "query.cuh"

namespace {

thread_local std::string g_err;

fm_status set_err(fm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

constexpr int kBlock = 256;
constexpr int kStreams = 3;
constexpr std::uint64_t kChunkPoints = std::uint64_t{1} << 23;  // 8M points = 128 MiB

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

#define FM_CUDA(call)                                                        \
  do {                                                                       \
    const cudaError_t err_ = (call);                                         \
    if (err_ != cudaSuccess) {                                               \
      return set_err(FM_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(err_)); \
    }                                                                        \
  } while (0)

// Kernel configuration.  kWarps warps per CTA; each warp streams tiles of
// 32*kU points.  Points in boundary cells are parked in a per-warp
// shared-memory queue and resolved up to 32 at a time with all lanes busy:
// the batch's records (their sizes come from the grid entries) are copied
// into a per-warp shared pool by cooperative cp.async -- half a warp per
// record, so one instruction moves two records -- in a single round trip,
// then each lane evaluates its own record from shared memory.  A point in
// a split cell is re-queued with the child's entry.
constexpr int kWarps = 8;
constexpr int kU = 2;
constexpr int kQCap = 32 * kU + 32;
constexpr int kPool = 4096;  // bytes of record staging per warp

struct WarpSmem {
  double qx[kQCap];
  double qy[kQCap];
  unsigned long long qi[kQCap];
  std::uint32_t qe[kQCap];
  std::uint32_t bstart[32];  // pool offset (16-byte chunks) per batch slot
  std::uint32_t bsize[32];   // chunks per batch slot
  alignas(16) std::uint8_t pool[kPool];
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

template <bool kHist>
__device__ __forceinline__ void emit(int* __restrict__ out, unsigned long long* __restrict__ hist,
                                     std::uint64_t i, int id) {
  __stcs(out + i, id);
  if (kHist && id >= 0) atomicAdd(hist + id, 1ull);
}

constexpr int kRequeue = INT_MIN;

// Resolve the batch S.q*[k0 .. k0+cnt-1] (cnt <= 32; lane l owns item
// k0 + l).  Returns the leaf id, -1, or kRequeue with *next_e set.
template <bool kCount>
__device__ __forceinline__ int resolve_batch(const fm::KParams& P, WarpSmem& S, int lane,
                                             int k0, int cnt, std::uint32_t* next_e,
                                             fm::WorkCount& wc) {
  const bool mine = lane < cnt;
  const std::uint32_t e = mine ? S.qe[k0 + lane] : 0u;
  const std::uint32_t chunks = mine ? fm::entry_fetch_bytes(e) / 16 : 0u;
  // exclusive scan of chunk counts -> pool layout
  std::uint32_t incl = chunks;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  const std::uint32_t start = incl - chunks;
  S.bstart[lane] = start;
  S.bsize[lane] = chunks;
  __syncwarp();
  // cooperative copy: iteration m moves slots 2m (lanes 0-15) and 2m+1 (16-31)
  const int half = lane >> 4, c = lane & 15;
  for (int m = 0; 2 * m < cnt; ++m) {
    const int slot = 2 * m + half;
    if (slot < cnt && static_cast<std::uint32_t>(c) < S.bsize[slot]) {
      const std::uint8_t* rec = fm::record_ptr(P, S.qe[k0 + slot]);
      cp_async16(S.pool + 16 * (S.bstart[slot] + c), rec + 16 * c);
    }
  }
  cp_async_wait_all();
  __syncwarp();
  if (!mine) return -1;
  const double px = S.qx[k0 + lane], py = S.qy[k0 + lane];
  const fm::SmemReader W{S.pool + 16 * start};
  const std::uint32_t h = W.u32(0);
  const std::uint32_t kind = h & 0xFFu;
  if (kind == fm::kKindSplit) {
    const double x0 = W.f64(8), y0 = W.f64(16), ihw = W.f64(24), ihh = W.f64(32);
    int i = static_cast<int>(__dmul_rn(__dsub_rn(px, x0), ihw));
    int j = static_cast<int>(__dmul_rn(__dsub_rn(py, y0), ihh));
    i = min(max(i, 0), 1);
    j = min(max(j, 0), 1);
    const std::uint32_t ce = W.u32(40 + 4 * (2 * j + i));
    if (ce == fm::kEmpty) return -1;
    if (ce < fm::kRecordBit) return static_cast<int>(ce);
    *next_e = ce;
    return kRequeue;
  }
  if (kCount) wc.boundary++;
  if (kind == fm::kKindCompact) {
    const std::uint32_t nv = (h >> 8) & 0xFFu, nc = (h >> 16) & 0xFFu, nb = h >> 24;
    if (fm::compact_bytes(nv, nc, nb) <= 16u * chunks) {
      return fm::resolve_compact<kCount>(W, h, px, py, wc);
    }
    return fm::resolve_compact<kCount>(fm::GlobalReader{fm::record_ptr(P, e)}, h, px, py, wc);
  }
  return fm::resolve_wide<kCount>(fm::record_ptr(P, e), px, py, wc);
}

// Pop up to 32 items off the top of the queue (as many as the pool holds),
// resolve them, emit the finished ones and push split descents back.
template <bool kHist, bool kCount>
__device__ __forceinline__ void drain_once(const fm::KParams& P, WarpSmem& S, int lane, int& qn,
                                           int* __restrict__ out,
                                           unsigned long long* __restrict__ hist,
                                           fm::WorkCount& wc) {
  const int cnt = min(qn, 32);
  // the batch is the top `take` items, as many as fit the pool (items are at
  // most 256 bytes, so at least 16 always fit): scan sizes from the top
  const std::uint32_t bytes = lane < cnt ? fm::entry_fetch_bytes(S.qe[qn - 1 - lane]) : 0u;
  std::uint32_t incl = bytes;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const std::uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += v;
  }
  const int take = __popc(__ballot_sync(0xFFFFFFFFu, lane < cnt && incl <= kPool));
  const int b0 = qn - take;
  const double px = lane < take ? S.qx[b0 + lane] : 0.0;
  const double py = lane < take ? S.qy[b0 + lane] : 0.0;
  const std::uint64_t i = lane < take ? S.qi[b0 + lane] : 0ull;
  std::uint32_t ne = 0;
  const int id = resolve_batch<kCount>(P, S, lane, b0, take, &ne, wc);
  __syncwarp();
  qn = b0;
  const bool requeue = lane < take && id == kRequeue;
  if (lane < take && !requeue) emit<kHist>(out, hist, i, id);
  const std::uint32_t b = __ballot_sync(0xFFFFFFFFu, requeue);
  if (requeue) {
    const int pos = qn + __popc(b & ((1u << lane) - 1u));
    S.qx[pos] = px;
    S.qy[pos] = py;
    S.qi[pos] = i;
    S.qe[pos] = ne;
  }
  qn += __popc(b);
  __syncwarp();
}

template <bool kHist, bool kCount>
__global__ void __launch_bounds__(kWarps * 32)
    project_kernel(fm::KParams P, const double2* __restrict__ pts, std::uint64_t n,
                   int* __restrict__ out, unsigned long long* __restrict__ hist,
                   unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  WarpSmem* smem = reinterpret_cast<WarpSmem*>(dsmem);
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  WarpSmem& S = smem[wid];
  const std::uint32_t lt_mask = (1u << lane) - 1u;
  const std::uint64_t tile = 32ull * kU;
  const std::uint64_t n_tiles = (n + tile - 1) / tile;
  const std::uint64_t gwarp = static_cast<std::uint64_t>(blockIdx.x) * kWarps + wid;
  const std::uint64_t nwarps = static_cast<std::uint64_t>(gridDim.x) * kWarps;
  fm::WorkCount wc;
  unsigned long long n_done = 0;
  int qn = 0;
  double2 pn[kU];  // next tile's points, loaded one tile ahead
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    const std::uint64_t i = gwarp * tile + u * 32 + lane;
    pn[u] = (gwarp < n_tiles && i < n) ? __ldcs(pts + i) : make_double2(NAN, NAN);
  }
  for (std::uint64_t t = gwarp; t < n_tiles; t += nwarps) {
    const std::uint64_t base = t * tile;
    double2 p[kU];
    std::uint32_t e[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) p[u] = pn[u];
#pragma unroll
    for (int u = 0; u < kU; ++u) e[u] = fm::locate(P, p[u].x, p[u].y);
    const std::uint64_t tn = t + nwarps;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const std::uint64_t i = tn * tile + u * 32 + lane;
      pn[u] = (tn < n_tiles && i < n) ? __ldcs(pts + i) : make_double2(NAN, NAN);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const std::uint64_t i = base + u * 32 + lane;
      const bool valid = i < n;
      const bool is_rec = valid && e[u] >= fm::kRecordBit && e[u] != fm::kEmpty;
      if (valid && !is_rec) emit<kHist>(out, hist, i, e[u] < fm::kRecordBit ? static_cast<int>(e[u]) : -1);
      if (kCount && valid) ++n_done;
      const std::uint32_t b = __ballot_sync(0xFFFFFFFFu, is_rec);
      if (is_rec) {
        const int pos = qn + __popc(b & lt_mask);
        S.qx[pos] = p[u].x;
        S.qy[pos] = p[u].y;
        S.qi[pos] = i;
        S.qe[pos] = e[u];
      }
      qn += __popc(b);
    }
    __syncwarp();
    while (qn >= 32) drain_once<kHist, kCount>(P, S, lane, qn, out, hist, wc);
  }
  while (qn > 0) drain_once<kHist, kCount>(P, S, lane, qn, out, hist, wc);
  if (kCount) {
    unsigned long long v[4] = {n_done, wc.boundary, wc.cands, wc.edges};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xFFFFFFFFu, v[k], o);
    }
    if (lane == 0) {
      for (int k = 0; k < 4; ++k) atomicAdd(counters + k, v[k]);
    }
  }
}

constexpr int kSmemBytes = static_cast<int>(sizeof(WarpSmem)) * kWarps;

int grid_size_for(int device, std::uint64_t n, const void* kernel) {
  // resident CTAs per SM x SM count, cached per (device, kernel)
  struct Slot {
    int device;
    const void* kernel;
    int blocks;
  };
  static std::mutex mu;
  static std::vector<Slot> cache;
  int blocks = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const Slot& s : cache) {
      if (s.device == device && s.kernel == kernel) blocks = s.blocks;
    }
    if (blocks == 0) {
      int sms = 0, per_sm = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, kSmemBytes);
      blocks = std::max(1, sms) * std::max(1, per_sm);
      cache.push_back({device, kernel, blocks});
    }
  }
  const std::uint64_t per_cta = static_cast<std::uint64_t>(kBlock) * kU;
  const std::uint64_t need = (n + per_cta - 1) / per_cta;
  return static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(need, blocks)));
}

}  // namespace

struct fm_index {
  int device = -1;
  fm::GridGeom g{};
  double ax0 = 0, ax1 = 0, ay0 = 0, ay1 = 0;
  std::uint32_t* d_grid = nullptr;
  std::uint8_t* d_arena = nullptr;
  std::uint64_t grid_len = 0, arena_len = 0, granule = 16;
  fm::HostIndex host;  // retained only for host-only (device < 0) indexes
  fm_index_stats stats{};
  // fm_query_host staging
  std::mutex mu;
  bool staged = false;
  cudaStream_t streams[kStreams] = {};
  double* d_in[kStreams] = {};
  int* d_out[kStreams] = {};
  unsigned long long* d_hist = nullptr;
};

namespace {

fm::KParams kparams(const fm_index* ix) {
  fm::KParams P;
  P.grid = ix->d_grid;
  P.arena = ix->d_arena;
  P.gx0 = ix->g.gx0;
  P.gy0 = ix->g.gy0;
  P.inv_w = ix->g.inv_w;
  P.inv_h = ix->g.inv_h;
  P.ax0 = ix->ax0;
  P.ax1 = ix->ax1;
  P.ay0 = ix->ay0;
  P.ay1 = ix->ay1;
  P.nx = static_cast<int>(ix->g.nx);
  P.ny = static_cast<int>(ix->g.ny);
  P.granule = ix->granule;
  return P;
}

fm_status launch(const fm_index* ix, const double* d_pts, std::uint64_t n, int* d_out,
                 unsigned long long* d_hist, unsigned long long* d_counters,
                 cudaStream_t stream) {
  const fm::KParams P = kparams(ix);
  const double2* pts = reinterpret_cast<const double2*>(d_pts);
  if (d_hist && d_counters) {
    auto k = project_kernel<true, true>;
    k<<<grid_size_for(ix->device, n, (const void*)k), kBlock, kSmemBytes, stream>>>(P, pts, n, d_out, d_hist, d_counters);
  } else if (d_hist) {
    auto k = project_kernel<true, false>;
    k<<<grid_size_for(ix->device, n, (const void*)k), kBlock, kSmemBytes, stream>>>(P, pts, n, d_out, d_hist, d_counters);
  } else if (d_counters) {
    auto k = project_kernel<false, true>;
    k<<<grid_size_for(ix->device, n, (const void*)k), kBlock, kSmemBytes, stream>>>(P, pts, n, d_out, d_hist, d_counters);
  } else {
    auto k = project_kernel<false, false>;
    k<<<grid_size_for(ix->device, n, (const void*)k), kBlock, kSmemBytes, stream>>>(P, pts, n, d_out, d_hist, d_counters);
  }
  FM_CUDA(cudaGetLastError());
  return FM_OK;
}

fm_status check_device(int device) {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    return set_err(FM_ERR_NO_DEVICE, std::string("no CUDA device available (") +
                                         cudaGetErrorString(e) +
                                         "); the B200 path has no CPU fallback");
  }
  if (device < 0 || device >= count) {
    return set_err(FM_ERR_INVALID_ARGUMENT, "CUDA device ordinal out of range");
  }
  return FM_OK;
}

void free_device(fm_index* ix) {
  if (ix->device < 0) return;
  DeviceGuard guard(ix->device);
  for (int s = 0; s < kStreams; ++s) {
    if (ix->d_in[s]) cudaFree(ix->d_in[s]);
    if (ix->d_out[s]) cudaFree(ix->d_out[s]);
    if (ix->streams[s]) cudaStreamDestroy(ix->streams[s]);
  }
  if (ix->d_hist) cudaFree(ix->d_hist);
  if (ix->d_grid) cudaFree(ix->d_grid);
  if (ix->d_arena) cudaFree(ix->d_arena);
}

}  // namespace

extern "C" {

const char* fm_status_string(fm_status s) {
  switch (s) {
    case FM_OK: return "ok";
    case FM_ERR_INVALID_ARGUMENT: return "invalid argument";
    case FM_ERR_RUNTIME: return "runtime error";
    case FM_ERR_DOMAIN: return "domain error";
    case FM_ERR_CUDA: return "CUDA error";
    case FM_ERR_NO_DEVICE: return "no CUDA device";
    case FM_ERR_OOM: return "out of memory";
  }
  return "unknown status";
}

const char* fm_last_error(void) { return g_err.c_str(); }

const char* fm_version(void) { return "fastmap_b200 0.1 (sm_100a)"; }

fm_status fm_index_build(const double* vertex_lonlat, const std::uint64_t* ring_offsets,
                         std::uint64_t n_rings, const std::uint64_t* poly_ring_offsets,
                         std::uint64_t n_polys, const fm_build_params* params,
                         fm_index** out_index) {
  g_err.clear();
  if (out_index == nullptr) return set_err(FM_ERR_INVALID_ARGUMENT, "out_index is null");
  *out_index = nullptr;
  fm_build_params p{};
  if (params) p = *params;
  if (p.device >= 0) {
    const fm_status st = check_device(p.device);
    if (st != FM_OK) return st;
  }
  fm::Soup soup;
  soup.vxy = vertex_lonlat;
  soup.ring_off = ring_offsets;
  soup.n_rings = n_rings;
  soup.poly_ring = poly_ring_offsets;
  soup.n_polys = n_polys;
  fm::BuildOptions opt;
  opt.cells_per_polygon = p.cells_per_polygon;
  opt.nx = p.nx;
  opt.ny = p.ny;
  opt.margin = p.margin;
  opt.threads = p.threads;

  fm_index* ix = new (std::nothrow) fm_index();
  if (!ix) return set_err(FM_ERR_OOM, "host allocation failed");
  const auto t0 = std::chrono::steady_clock::now();
  try {
    ix->host = fm::build_index_host(soup, opt);
  } catch (const fm::InvalidArgument& e) {
    delete ix;
    return set_err(FM_ERR_INVALID_ARGUMENT, e.what());
  } catch (const fm::RuntimeError& e) {
    delete ix;
    return set_err(FM_ERR_RUNTIME, e.what());
  } catch (const std::bad_alloc&) {
    delete ix;
    return set_err(FM_ERR_OOM, "host allocation failed during index build");
  } catch (const std::exception& e) {
    delete ix;
    return set_err(FM_ERR_RUNTIME, e.what());
  }
  ix->device = p.device;
  ix->g = ix->host.g;
  ix->ax0 = std::max(ix->g.gx0, -180.0);
  ix->ax1 = std::min(ix->g.gx1, 180.0);
  ix->ay0 = std::max(ix->g.gy0, -90.0);
  ix->ay1 = std::min(ix->g.gy1, 90.0);
  ix->grid_len = ix->host.grid.size();
  ix->arena_len = ix->host.arena.size();
  ix->granule = ix->host.granule;

  fm_index_stats& s = ix->stats;
  s.n_polys = n_polys;
  s.n_rings = n_rings;
  s.n_vertices = n_rings ? ring_offsets[n_rings] - ring_offsets[0] : 0;
  s.n_edges = ix->host.stats.n_edges;
  s.nx = ix->g.nx;
  s.ny = ix->g.ny;
  s.cells_empty = ix->host.stats.cells_empty;
  s.cells_hit = ix->host.stats.cells_hit;
  s.cells_boundary = ix->host.stats.cells_boundary;
  s.grid_bytes = ix->grid_len * 4;
  s.arena_bytes = ix->host.arena_used;
  s.geometry_bytes = s.n_vertices * 16;
  s.record_edges = ix->host.stats.record_edges;
  s.record_cands = ix->host.stats.record_cands;
  s.record_breaks = ix->host.stats.record_breaks;
  s.max_record_edges = ix->host.stats.max_record_edges;
  s.max_record_cands = ix->host.stats.max_record_cands;
  s.gx0 = ix->g.gx0;
  s.gx1 = ix->g.gx1;
  s.gy0 = ix->g.gy0;
  s.gy1 = ix->g.gy1;
  s.cell_w = ix->g.w;
  s.cell_h = ix->g.h;
  s.margin = ix->g.margin;

  if (ix->device >= 0) {
    DeviceGuard guard(ix->device);
    if (!guard.ok) {
      delete ix;
      return set_err(FM_ERR_CUDA, "cudaSetDevice failed");
    }
    cudaError_t e1 = cudaMalloc(&ix->d_grid, ix->grid_len * 4);
    cudaError_t e2 = cudaMalloc(&ix->d_arena, ix->arena_len);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      free_device(ix);
      delete ix;
      return set_err(FM_ERR_OOM, "device allocation of the index failed");
    }
    e1 = cudaMemcpy(ix->d_grid, ix->host.grid.data(), ix->grid_len * 4, cudaMemcpyHostToDevice);
    e2 = cudaMemcpy(ix->d_arena, ix->host.arena.data(), ix->arena_len, cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      free_device(ix);
      delete ix;
      return set_err(FM_ERR_CUDA, "index upload failed");
    }
    // the device copy is authoritative; drop the host arrays
    std::vector<std::uint32_t>().swap(ix->host.grid);
    std::vector<std::uint8_t>().swap(ix->host.arena);
  }
  s.build_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out_index = ix;
  return FM_OK;
}

void fm_index_destroy(fm_index* index) {
  if (!index) return;
  free_device(index);
  delete index;
}

fm_status fm_index_stats_get(const fm_index* index, fm_index_stats* out) {
  if (!index || !out) return set_err(FM_ERR_INVALID_ARGUMENT, "null argument");
  *out = index->stats;
  return FM_OK;
}

int fm_index_device(const fm_index* index) { return index ? index->device : -1; }

fm_status fm_query(const fm_index* index, const double* d_lonlat, std::uint64_t n,
                   std::int32_t* d_out, std::int64_t* d_hist, fm_query_counters* d_counters,
                   void* stream) {
  g_err.clear();
  if (!index) return set_err(FM_ERR_INVALID_ARGUMENT, "index is null");
  if (index->device < 0) {
    return set_err(FM_ERR_NO_DEVICE, "index was built host-only (device < 0); no CPU query path exists");
  }
  if (n == 0) return FM_OK;
  if (!d_lonlat || !d_out) return set_err(FM_ERR_INVALID_ARGUMENT, "null point or output buffer");
  DeviceGuard guard(index->device);
  if (!guard.ok) return set_err(FM_ERR_CUDA, "cudaSetDevice failed");
  return launch(index, d_lonlat, n, reinterpret_cast<int*>(d_out),
                reinterpret_cast<unsigned long long*>(d_hist),
                reinterpret_cast<unsigned long long*>(d_counters),
                static_cast<cudaStream_t>(stream));
}

fm_status fm_query_host(const fm_index* cindex, const double* h_lonlat, std::uint64_t n,
                        std::int32_t* h_out, std::int64_t* h_hist) {
  g_err.clear();
  if (!cindex) return set_err(FM_ERR_INVALID_ARGUMENT, "index is null");
  fm_index* index = const_cast<fm_index*>(cindex);  // staging buffers are mutable state
  if (index->device < 0) {
    return set_err(FM_ERR_NO_DEVICE, "index was built host-only (device < 0); no CPU query path exists");
  }
  if (n == 0) return FM_OK;
  if (!h_lonlat || !h_out) return set_err(FM_ERR_INVALID_ARGUMENT, "null point or output buffer");
  std::lock_guard<std::mutex> lk(index->mu);
  DeviceGuard guard(index->device);
  if (!guard.ok) return set_err(FM_ERR_CUDA, "cudaSetDevice failed");
  if (!index->staged) {
    for (int s = 0; s < kStreams; ++s) {
      FM_CUDA(cudaStreamCreateWithFlags(&index->streams[s], cudaStreamNonBlocking));
      FM_CUDA(cudaMalloc(&index->d_in[s], kChunkPoints * 16));
      FM_CUDA(cudaMalloc(&index->d_out[s], kChunkPoints * 4));
    }
    index->staged = true;
  }
  unsigned long long* dh = nullptr;
  if (h_hist) {
    if (!index->d_hist) FM_CUDA(cudaMalloc(&index->d_hist, std::max<std::uint64_t>(1, index->stats.n_polys) * 8));
    dh = index->d_hist;
    FM_CUDA(cudaMemsetAsync(dh, 0, std::max<std::uint64_t>(1, index->stats.n_polys) * 8, index->streams[0]));
    FM_CUDA(cudaStreamSynchronize(index->streams[0]));
  }
  const std::uint64_t n_chunks = (n + kChunkPoints - 1) / kChunkPoints;
  for (std::uint64_t c = 0; c < n_chunks; ++c) {
    const int s = static_cast<int>(c % kStreams);
    const std::uint64_t off = c * kChunkPoints;
    const std::uint64_t m = std::min(kChunkPoints, n - off);
    FM_CUDA(cudaMemcpyAsync(index->d_in[s], h_lonlat + 2 * off, m * 16, cudaMemcpyHostToDevice,
                            index->streams[s]));
    const fm_status st = launch(index, index->d_in[s], m, index->d_out[s], dh, nullptr, index->streams[s]);
    if (st != FM_OK) return st;
    FM_CUDA(cudaMemcpyAsync(h_out + off, index->d_out[s], m * 4, cudaMemcpyDeviceToHost,
                            index->streams[s]));
  }
  for (int s = 0; s < kStreams; ++s) FM_CUDA(cudaStreamSynchronize(index->streams[s]));
  if (h_hist) {
    std::vector<std::int64_t> tmp(index->stats.n_polys);
    FM_CUDA(cudaMemcpy(tmp.data(), dh, index->stats.n_polys * 8, cudaMemcpyDeviceToHost));
    for (std::uint64_t k = 0; k < index->stats.n_polys; ++k) h_hist[k] += tmp[k];
  }
  return FM_OK;
}

fm_status fm_index_export(const fm_index* index, std::uint32_t* grid, std::uint64_t* grid_len,
                          std::uint8_t* arena, std::uint64_t* arena_len, double* geometry16) {
  if (!index || !grid_len || !arena_len) return set_err(FM_ERR_INVALID_ARGUMENT, "null argument");
  *grid_len = index->grid_len;
  *arena_len = index->arena_len;
  if (geometry16) {
    const fm::GridGeom& g = index->g;
    const double v[16] = {g.gx0, g.gx1, g.gy0, g.gy1, g.w, g.h, g.inv_w, g.inv_h,
                          static_cast<double>(g.nx), static_cast<double>(g.ny), g.margin,
                          static_cast<double>(index->stats.n_polys),
                          static_cast<double>(index->granule), 0.0, 0.0, 0.0};
    std::memcpy(geometry16, v, sizeof(v));
  }
  if (!grid && !arena) return FM_OK;
  if (index->device < 0) {
    if (grid) std::memcpy(grid, index->host.grid.data(), index->grid_len * 4);
    if (arena) std::memcpy(arena, index->host.arena.data(), index->arena_len);
    return FM_OK;
  }
  DeviceGuard guard(index->device);
  if (grid) FM_CUDA(cudaMemcpy(grid, index->d_grid, index->grid_len * 4, cudaMemcpyDeviceToHost));
  if (arena) FM_CUDA(cudaMemcpy(arena, index->d_arena, index->arena_len, cudaMemcpyDeviceToHost));
  return FM_OK;
}

}  // extern "C"
