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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/fastmap_b200.h"
#include "index_build.h"
#include "index_format.h"
#include "query.cuh"

#include <cub/cub.cuh>

namespace {

thread_local std::string g_err;

fm_status set_err(fm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

}  // namespace

// For io.cpp (not part of the C-ABI).
__attribute__((visibility("hidden"))) fm_status fm_set_error(fm_status s, const char* msg) {
  return set_err(s, msg);
}

namespace {

#ifndef FM_KU
#define FM_KU 2
#endif
#ifndef FM_AMINB
#define FM_AMINB 6
#endif
#ifndef FM_BWARPS
#define FM_BWARPS 8
#endif

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

// Two kernels per query:
//  stream_kernel  -- the HBM stream.  Each warp walks tiles of 32*kU points
//    (next tile loaded one tile ahead), locates each point's cell, answers
//    true-hit / empty cells at once, and appends boundary points (24-byte
//    items) to its own private region of a global queue: no atomics, fully
//    coalesced appends.  Small shared/register footprint -> high occupancy.
//  resolve_kernel -- one warp per queue region.  Items are taken 32 at a
//    time; the records of batch k+1 (sizes come from the grid entries) are
//    copied into a double-buffered shared pool by cooperative cp.async while
//    batch k is evaluated, so record latency overlaps compute.  Evaluation
//    spreads the (item, edge) crossing tests over all 32 lanes.
constexpr int kU = FM_KU;
constexpr int kAWarps = 8;
constexpr int kBWarps = FM_BWARPS;

struct QItem {  // 24 bytes
  double px, py;
  std::uint32_t i;  // point index within the launch
  std::uint32_t e;  // grid entry of the boundary cell
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait0() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Per-launch histogram counters are u32: half the footprint of the int64
// result, so more of them stay in L2 (c5, 12.5M leaves: 59.5 -> 55.5 ms per
// 1B points).  fm_query adds them into the caller's int64 histogram after
// every slice of <= 2^28 points, so they cannot overflow.
using HistT = unsigned int;

// The per-block histogram sink of one CTA (stream path).  Clustered
// streams put most of their points into a few hundred leaves (the top Zipf
// clusters), and same-address atomics serialise, so equal ids of a warp are
// first aggregated (__match_any_sync) and a CTA counts into a small
// shared-memory cache of hot leaves: a slot is claimed by the first leaf
// that hashes to it (atomicCAS) and counted with shared-memory atomics;
// a leaf whose slot is taken goes straight to the global counter.  The
// cache is flushed into the global counters when the CTA exits.  (The
// binned path counts its histogram afterwards, binned_hist_kernel.)
// 3 (default): equal ids of the active lanes aggregated with
// __match_any_sync, then the hot-leaf cache (c2 with histogram: 1.61 ms per
// 100M points against 1.83 for the cache alone, 2.73 for plain global
// atomics; profiles/r2y, r2w)
#ifndef FM_HIST_MODE
#define FM_HIST_MODE 3
#endif
constexpr int kHotSlots = 1024;
struct HistSink {
  HistT* g = nullptr;         // global per-launch counters
  unsigned int* tag = nullptr;  // shared: kHotSlots leaf ids (kEmpty = free)
  unsigned int* cnt = nullptr;  // shared: their counts
  __device__ __forceinline__ void add(int id) const {
    const unsigned int u = static_cast<unsigned int>(id);
#if FM_HIST_MODE == 1  // experiment: straight to the global counters
    atomicAdd(g + u, 1u);
    return;
#elif FM_HIST_MODE == 2  // experiment: aggregated over equal ids of the active lanes
    const unsigned int peers = __match_any_sync(__activemask(), u);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(g + u, static_cast<unsigned int>(__popc(peers)));
    return;
#elif FM_HIST_MODE == 3  // experiment: aggregated, then the hot-leaf cache
    const unsigned int peers = __match_any_sync(__activemask(), u);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) add_n(u, static_cast<unsigned int>(__popc(peers)));
    return;
#endif
    add_n(u, 1u);
  }
  __device__ __forceinline__ void add_n(unsigned int u, unsigned int k) const {
    const unsigned int s = (u * 2654435761u) >> 22;  // 10-bit multiplicative hash
    unsigned int t = tag[s];
    if (t == fm::kEmpty) {
      t = atomicCAS(tag + s, fm::kEmpty, u);
      if (t == fm::kEmpty) t = u;
    }
    if (t == u) {
      atomicAdd(cnt + s, k);
    } else {
      atomicAdd(g + u, k);
    }
  }
};
static_assert(kHotSlots == 1024, "hash is 10 bits");

// Shared-memory backing of a HistSink (kHist instantiations only).
template <bool kHist>
struct HotSmem {
  unsigned int tag[kHist ? kHotSlots : 1];
  unsigned int cnt[kHist ? kHotSlots : 1];
};

template <bool kHist>
__device__ __forceinline__ HistSink hist_open(HistT* g, HotSmem<kHist>& h) {
  HistSink hs;
  hs.g = g;
  if (kHist) {
    for (int k = threadIdx.x; k < kHotSlots; k += blockDim.x) {
      h.tag[k] = fm::kEmpty;
      h.cnt[k] = 0u;
    }
    hs.tag = h.tag;
    hs.cnt = h.cnt;
    __syncthreads();
  }
  return hs;
}

template <bool kHist>
__device__ __forceinline__ void hist_close(const HistSink& hs) {
  if (kHist) {
    __syncthreads();
    for (int k = threadIdx.x; k < kHotSlots; k += blockDim.x) {
      const unsigned int c = hs.cnt[k];
      if (c) atomicAdd(hs.g + hs.tag[k], c);
    }
  }
}

template <bool kHist>
__device__ __forceinline__ void emit(int* __restrict__ out, const HistSink& hs, std::uint64_t i,
                                     int id) {
  __stcs(out + i, id);
  if (kHist && id >= 0) hs.add(id);
}
template <bool kHist>
__device__ __forceinline__ void emit(int* __restrict__ out, unsigned long long* __restrict__ hist,
                                     std::uint64_t i, int id) {
  __stcs(out + i, id);
  if (kHist && id >= 0) atomicAdd(hist + id, 1ull);
}


template <bool kHist, bool kCount, int kLs>
__global__ void __launch_bounds__(kAWarps * 32, FM_AMINB)
    stream_kernel(fm::KParams P, const double2* __restrict__ pts, std::uint64_t n,
                  int* __restrict__ out, HistT* __restrict__ hist,
                  QItem* __restrict__ q, std::uint32_t* __restrict__ qcount,
                  std::uint64_t region_cap, unsigned long long* __restrict__ counters) {
  __shared__ HotSmem<kHist> hot;
  const HistSink hs = hist_open<kHist>(hist, hot);
  const int lane = threadIdx.x & 31;
  const std::uint64_t tile = 32ull * kU;
  const std::uint64_t n_tiles = (n + tile - 1) / tile;
  const std::uint64_t gwarp = static_cast<std::uint64_t>(blockIdx.x) * kAWarps + (threadIdx.x >> 5);
  const std::uint64_t nwarps = static_cast<std::uint64_t>(gridDim.x) * kAWarps;
  QItem* __restrict__ my = q + gwarp * region_cap;
  std::uint32_t cnt = 0;
  const std::uint32_t lt_mask = (1u << lane) - 1u;
  double2 pn[kU];
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
    fm::locate_n<kU, true, kLs>(P, p, e);
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
      // every lane stores (boundary lanes a placeholder the resolve pass
      // overwrites), so output sectors are written whole, not masked
      if (valid) {
        const int id = is_rec ? -2 : (e[u] < fm::kRecordBit ? static_cast<int>(e[u]) : -1);
        __stcs(out + i, id);
        if (kHist && id >= 0) hs.add(id);
      }
      const std::uint32_t b = __ballot_sync(0xFFFFFFFFu, is_rec);
      if (is_rec) {  // streaming stores: the resolve pass reads these much later
        double* d = reinterpret_cast<double*>(my + cnt + __popc(b & lt_mask));
        __stcs(d, p[u].x);
        __stcs(d + 1, p[u].y);
        __stcs(reinterpret_cast<uint2*>(d + 2), make_uint2(static_cast<std::uint32_t>(i), e[u]));
      }
      cnt += __popc(b);
    }
  }
  if (gwarp < nwarps && lane == 0) qcount[gwarp] = cnt;
  hist_close<kHist>(hs);
  if (kCount) {
    unsigned long long v = 0;
    for (std::uint64_t t = gwarp; t < n_tiles; t += nwarps) {
      const std::uint64_t base = t * tile;
      v += min(tile, n - base);
    }
    if (lane == 0) atomicAdd(counters + 0, v);
  }
}

// resolve_kernel: one warp per queue region (pulled from an atomic counter).
// Items are taken 32 at a time; the 128-byte slots of batch k+1 are copied
// by cp.async into a double-buffered shared pool (8 lanes x 16 B per slot,
// chunk c of slot r stored at chunk c ^ (r & 7) so the owner lanes' 16-byte
// reads are bank-conflict free) while batch k is evaluated -- straight-line,
// predicated code over registers (eval_leaf_slot).
struct WarpSmemB {
  alignas(16) std::uint8_t pool[2][32 * fm::kSlotBytes];
};

__device__ __forceinline__ QItem load_item(const QItem* __restrict__ items, std::uint32_t k,
                                           std::uint32_t cnt) {
  QItem it;
  if (k < cnt) {  // 24-byte items are only 8-byte aligned
    const double* d = reinterpret_cast<const double*>(items + k);
    it.px = __ldcs(d);
    it.py = __ldcs(d + 1);
    const uint2 ie = __ldcs(reinterpret_cast<const uint2*>(d + 2));
    it.i = ie.x;
    it.e = ie.y;
  } else {
    it.px = it.py = 0.0;
    it.i = 0;
    it.e = fm::kEmpty;
  }
  return it;
}

// Start copying the slots of the items held by lanes [0, n) into `buf`: 8
// lanes per slot, 16 bytes each, so every cp.async instruction requests 4
// whole slots (lines) -- per-lane copies of its own slot measured far slower
// on the stream path (c3: 47 -> 111 ms; each line requested in 8 pieces at
// different times).  Chunk c of slot r is stored at chunk c ^ (r & 7) so
// the owner lane's reads in eval_staged are bank-conflict free.  The second
// half of a double slot (kDoubleBit) is prefetched into L2, where its
// evaluation one batch later finds it.  (Precomputing the swizzled shared
// addresses and folding validity and the half flag into one compare cut
// the instructions per copy from ~14 to 6 but measured slower on c3, 31.94
// vs 31.43 ms, through register pressure: profiles/r2ak.)
__device__ __forceinline__ void stage_slots(const fm::KParams& P, std::uint8_t* buf,
                                            std::uint32_t e, int n, int lane) {
  if (lane < n && (e & fm::kDoubleBit) && !(e & fm::kHalfBit)) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(fm::slot_ptr(P, e) + fm::kSlotBytes));
  }
  // source: slots + 16 * (8 * index + chunk) (the entry shifted left by 3
  // drops its flag bits); destination: a per-lane constant + 512 bytes per
  // instruction (r & 7 = 4 (q & 1) + j for r = 4 q + j)
  const int c = lane & 7, j = lane >> 3;
  const std::uint8_t* slots = P.slots;
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(buf)) + j * 128;
  const unsigned d0 = b + 16 * (c ^ j), d1 = b + (16 * (c ^ j) ^ 64);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int r = 4 * q + j;
    const std::uint32_t er = __shfl_sync(0xFFFFFFFFu, e, r);
    if (r < n && (c < 4 || !(er & fm::kHalfBit))) {  // half slots: first 64 bytes only
      const unsigned dst = ((q & 1) ? d1 : d0) + q * 512;
      const std::uint8_t* src = slots + static_cast<std::size_t>(er * 8u + static_cast<std::uint32_t>(c)) * 16u;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
    }
  }
  cp_async_commit();
}

// Evaluate the staged batch.  Returns, per lane, the child entry a split
// cell descends to (to be re-queued) or 0 when the item is finished.
template <bool kHist, bool kCount>
__device__ __forceinline__ std::uint32_t eval_staged(const fm::KParams& P, const std::uint8_t* buf,
                                                     const QItem& it, int n, int lane,
                                                     int* __restrict__ out,
                                                     const HistSink& hist,
                                                     fm::WorkCount& wc) {
  std::uint32_t requeue = 0;
  if (lane < n) {
    const std::uint8_t* base = buf + lane * fm::kSlotBytes;
    const int s = lane & 7;
    uint4 c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = *reinterpret_cast<const uint4*>(base + 16 * (k ^ s));
    const std::uint32_t kind = c[0].x & 0xFFu;
    int id = -1;
    bool done = true;
    if (kind == fm::kSlotLeaf) {
      if (kCount) wc.boundary++;
      id = fm::eval_leaf_slot<kCount>(c, it.px, it.py, wc);
    } else if (kind == fm::kSlotDouble) {  // second half from global memory (prefetched to L2)
      if (kCount) wc.boundary++;
      uint4 b[8];
      fm::load_double_tail(P, it.e, b);
      id = fm::eval_double_slot<kCount>(c, b, it.px, it.py, wc);
    } else if (kind == fm::kSlotSplit) {
      const double x0 = fm::as_f64(c[0].z, c[0].w), y0 = fm::as_f64(c[1].x, c[1].y);
      const double ihw = fm::as_f64(c[1].z, c[1].w), ihh = fm::as_f64(c[2].x, c[2].y);
      int ci = static_cast<int>(__dmul_rn(__dsub_rn(it.px, x0), ihw));
      int cj = static_cast<int>(__dmul_rn(__dsub_rn(it.py, y0), ihh));
      ci = min(max(ci, 0), 1);
      cj = min(max(cj, 0), 1);
      const std::uint32_t k2 = 2 * cj + ci;
      const std::uint32_t ce = k2 == 0 ? c[2].z : k2 == 1 ? c[2].w : k2 == 2 ? c[3].x : c[3].y;
      if (ce == fm::kEmpty) {
        id = -1;
      } else if (ce < fm::kRecordBit) {
        id = static_cast<int>(ce);
      } else {
        requeue = ce;
        done = false;
      }
    } else {  // overflow record: its offset is in the staged slot, the record in global memory
      if (kCount) wc.boundary++;
      id = fm::resolve_overflow<kCount>(P, (static_cast<std::uint64_t>(c[0].w) << 32) | c[0].z, it.px,
                                        it.py, wc);
    }
    if (done) emit<kHist>(out, hist, it.i, id);
  }
  return requeue;
}

#ifndef FM_BMINB
#define FM_BMINB 2
#endif
template <bool kHist, bool kCount>
__global__ void __launch_bounds__(kBWarps * 32, FM_BMINB)
    resolve_kernel(fm::KParams P, const QItem* __restrict__ q,
                   const std::uint32_t* __restrict__ qcount, std::uint64_t n_regions,
                   std::uint64_t region_cap, unsigned long long* __restrict__ next_region,
                   int* __restrict__ out, HistT* __restrict__ hist,
                   unsigned long long* __restrict__ counters) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  __shared__ HotSmem<kHist> hot;
  const HistSink hs = hist_open<kHist>(hist, hot);
  const int lane = threadIdx.x & 31;
  WarpSmemB& S = reinterpret_cast<WarpSmemB*>(dsmem)[threadIdx.x >> 5];
  fm::WorkCount wc;
  for (;;) {
    unsigned long long region = 0;
    if (lane == 0) region = atomicAdd(next_region, 1ull);
    region = __shfl_sync(0xFFFFFFFFu, region, 0);
    if (region >= n_regions) break;
    QItem* items = const_cast<QItem*>(q) + region * region_cap;
    std::uint32_t cnt = qcount[region];
    // passes: split-cell descents are written back in place (the write
    // cursor never passes the read cursor) and resolved by the next pass
    while (cnt > 0) {
      std::uint32_t wr = 0;
      QItem cur = load_item(items, lane, cnt);
      QItem nxt = load_item(items, 32 + lane, cnt);
      int ncur = static_cast<int>(min(cnt, 32u));
      stage_slots(P, S.pool[0], cur.e, ncur, lane);
      int buf = 0;
      for (std::uint32_t b = 0; b < cnt; b += 32) {
        const int nnext = b + 32 < cnt ? static_cast<int>(min(cnt - b - 32, 32u)) : 0;
        QItem nn{};
        if (nnext > 0) {
          stage_slots(P, S.pool[buf ^ 1], nxt.e, nnext, lane);
          nn = load_item(items, b + 64 + lane, cnt);
          cp_async_wait1();
        } else {
          cp_async_wait0();
        }
        __syncwarp();
        const std::uint32_t ce = eval_staged<kHist, kCount>(P, S.pool[buf], cur, ncur, lane, out,
                                                            hs, wc);
        const std::uint32_t rq = __ballot_sync(0xFFFFFFFFu, ce != 0u);
        if (ce != 0u) {
          QItem it = cur;
          it.e = ce;
          items[wr + __popc(rq & ((1u << lane) - 1u))] = it;
        }
        wr += __popc(rq);
        __syncwarp();
        cur = nxt;
        nxt = nn;
        ncur = nnext;
        buf ^= 1;
      }
      cnt = wr;
      __syncwarp();
    }
  }
  hist_close<kHist>(hs);
  if (kCount) {
    unsigned long long v[3] = {wc.boundary, wc.cands, wc.edges};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xFFFFFFFFu, v[k], o);
    }
    if (lane == 0) {
      for (int k = 0; k < 3; ++k) atomicAdd(counters + 1 + k, v[k]);
    }
  }
}

constexpr int kSmemB = static_cast<int>(sizeof(WarpSmemB)) * kBWarps;

#include "binned.cuh"

// ---------------------------------------------------------------------------
// Fast-approx mode (CoverMode::approx, cell_index.hpp:558-560).  The approx
// cover assigns every cell of an epsilon-fine grid one answer: hits and
// empties as in the exact grid, boundary cells their deemed leaf.  It is
// stored two-level so the first level stays L2-resident: blocks of S x S
// fine cells (S a power of two) hold either their common answer or, when
// the block is not uniform, kRecordBit | k -> sub-block k (S*S u32, row-
// major).  A query is one 16-byte point read, one or two 4-byte gathers and
// one 4-byte write -- no queue, no crossing tests.
constexpr int kXThreads = 256;
#ifndef FM_XU
#define FM_XU 4
#endif
constexpr int kXU = FM_XU;

template <bool kHist, bool kCount>
__global__ void __launch_bounds__(kXThreads)
    approx_kernel(fm::KParams A, const double2* __restrict__ pts, std::uint64_t n,
                  int* __restrict__ out, unsigned long long* __restrict__ hist,
                  unsigned long long* __restrict__ counters) {
  const std::uint64_t chunk = static_cast<std::uint64_t>(kXThreads) * kXU;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * chunk;
  unsigned long long done = 0;
  // the next chunk's points are loaded while this chunk's gathers run
  double2 pn[kXU];
  const std::uint64_t b0 = blockIdx.x * chunk + threadIdx.x;
#pragma unroll
  for (int u = 0; u < kXU; ++u) {
    const std::uint64_t i = b0 + static_cast<std::uint64_t>(u) * kXThreads;
    pn[u] = i < n ? __ldcs(pts + i) : make_double2(NAN, NAN);
  }
  for (std::uint64_t b = b0; b < n + threadIdx.x; b += stride) {
    double2 p[kXU];
#pragma unroll
    for (int u = 0; u < kXU; ++u) {
      p[u] = pn[u];
      const std::uint64_t i = b + stride + static_cast<std::uint64_t>(u) * kXThreads;
      pn[u] = i < n ? __ldcs(pts + i) : make_double2(NAN, NAN);
    }
    std::uint32_t e[kXU];
    fm::locate_n<kXU, false>(A, p, e);
#pragma unroll
    for (int u = 0; u < kXU; ++u) {
      const std::uint64_t i = b + static_cast<std::uint64_t>(u) * kXThreads;
      if (i < n) {
        emit<kHist>(out, hist, i, static_cast<int>(e[u]));
        if (kCount) ++done;
      }
    }
  }
  if (kCount) {
    for (int o = 16; o > 0; o >>= 1) done += __shfl_xor_sync(0xFFFFFFFFu, done, o);
    if ((threadIdx.x & 31) == 0 && done) atomicAdd(counters + 0, done);
  }
}

// Per block of S x S fine cells: 0 when its entries are all equal, the
// number of compact units (low word) when a compact sub-block holds it,
// 1 << 32 when a full sub-block does.  The exclusive scan of these u64 flags
// numbers both kinds at once.  Compact kinds (`mode`): 1 = approx palette
// (<= 3 distinct answers, ls <= 3; one unit = one palette); 2 = exact, in
// 16-byte units (ls <= 2, phase-1 slot references with consecutive indices
// -- see renumber_slots): a "small" sub-block (one unit) when the hit
// entries take <= 2 distinct values besides empty, else a compact one (two
// units: <= 3 distinct hit/empty entries, <= 12 slot references).
__global__ void __launch_bounds__(256)
    block_flag_kernel(const std::uint32_t* __restrict__ fine, int nx, int ny, int bnx, int bny,
                      int ls, int mode, std::uint64_t n1, unsigned long long* __restrict__ flag) {
  const std::uint64_t b = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= static_cast<std::uint64_t>(bnx) * bny) return;
  const int by = static_cast<int>(b / bnx), bx = static_cast<int>(b - static_cast<std::uint64_t>(by) * bnx);
  const int S = 1 << ls;
  const int x0 = bx << ls, y0 = by << ls;
  std::uint32_t v[3];
  int nd = 0, nrec = 0;
  bool far_rec = false, has_empty = false;
  std::uint32_t kmin = 0xFFFFFFFFu, kmax = 0;
  for (int j = 0; j < S; ++j) {
    for (int i = 0; i < S; ++i) {
      const bool in = y0 + j < ny && x0 + i < nx;
      if (!in && j + i > 0) continue;  // outside cells never take part
      const std::uint32_t x = fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i];
      if (x != fm::kEmpty && x >= fm::kRecordBit) {  // slot reference
        const std::uint32_t k = x & fm::kSlotIndexMask;
        ++nrec;
        far_rec |= k >= n1;
        kmin = min(kmin, k);
        kmax = max(kmax, k);
        continue;
      }
      has_empty |= x == fm::kEmpty;
      bool seen = false;
      for (int q = 0; q < nd && q < 3; ++q) seen |= v[q] == x;
      if (!seen) {
        if (nd < 3) v[nd] = x;
        ++nd;
      }
    }
  }
  unsigned long long f;
  if (nrec == 0 && nd == 1) {
    f = 0ull;
  } else if (mode == 1 && nrec == 0 && nd <= 3 && ls <= 3) {
    f = 1ull;
  } else if (mode == 2 && ls <= 2 && !far_rec &&
             (nrec == 0 || kmax - kmin + 1 == static_cast<std::uint32_t>(nrec)) &&
             nd - (has_empty ? 1 : 0) <= 2) {
    f = 1ull;  // small compact: one 16-byte unit
  } else if (mode == 2 && ls <= 2 && nd <= 3 && nrec <= 12 && !far_rec &&
             (nrec == 0 || kmax - kmin + 1 == static_cast<std::uint32_t>(nrec))) {
    f = 2ull;  // compact: two 16-byte units
  } else {
    f = 1ull << 32;
  }
  flag[b] = f;
}

// Palette sub-block (approx covers): u32 palette[3], then 2-bit codes per
// cell in row-major order -- 16 bytes for ls <= 2 (codes at +12), 32 bytes
// for ls = 3 (codes at +16).
__host__ __device__ constexpr int palette_words(int ls) { return ls <= 2 ? 4 : 8; }

__global__ void __launch_bounds__(256)
    block_write_kernel(const std::uint32_t* __restrict__ fine, int nx, int ny, int bnx, int bny,
                       int ls, int mode, const unsigned long long* __restrict__ flag,
                       const unsigned long long* __restrict__ idx, std::uint32_t* __restrict__ blocks,
                       std::uint32_t* __restrict__ sub, std::uint32_t* __restrict__ pal) {
  const std::uint64_t b = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= static_cast<std::uint64_t>(bnx) * bny) return;
  const int by = static_cast<int>(b / bnx), bx = static_cast<int>(b - static_cast<std::uint64_t>(by) * bnx);
  const int S = 1 << ls;
  const int x0 = bx << ls, y0 = by << ls;
  const unsigned long long f = flag[b];
  if (!f) {
    blocks[b] = fine[static_cast<std::size_t>(y0) * nx + x0];
    return;
  }
  if (f == 1ull && mode == 2) {  // exact small sub-block (16 bytes)
    const unsigned long long k = idx[b] & 0xFFFFFFFFull;
    blocks[b] = fm::kRecordBit | fm::kHalfBit | fm::kSmallBit | static_cast<std::uint32_t>(k);
    std::uint32_t* dst = pal + k * 4;
    std::uint32_t v[2] = {fm::kEmpty, fm::kEmpty};
    int nd = 0;
    std::uint32_t base = 0xFFFFFFFFu, codes = 0u;
    for (int j = 0; j < S; ++j) {
      for (int i = 0; i < S; ++i) {
        if (y0 + j >= ny || x0 + i >= nx) continue;
        const std::uint32_t x = fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i];
        if (x != fm::kEmpty && x >= fm::kRecordBit) base = min(base, x & fm::kSlotIndexMask);
      }
    }
    for (int j = 0; j < S; ++j) {
      for (int i = 0; i < S; ++i) {
        const bool in = y0 + j < ny && x0 + i < nx;
        const std::uint32_t x = in ? fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i] : fm::kEmpty;
        std::uint32_t code;
        if (x == fm::kEmpty) {
          code = 3u;
        } else if (x >= fm::kRecordBit) {
          code = 2u;  // slot base + rank among the block's slot cells
        } else {
          code = 0;
          while (static_cast<int>(code) < nd && v[code] != x) ++code;
          if (static_cast<int>(code) == nd) v[nd++] = x;
        }
        codes |= code << (2 * ((j << ls) + i));
      }
    }
    dst[0] = v[0];
    dst[1] = v[1];
    dst[2] = base;
    dst[3] = codes;
    return;
  }
  if (f == 2ull && mode == 2) {  // exact compact sub-block (32 bytes)
    const unsigned long long k = idx[b] & 0xFFFFFFFFull;
    blocks[b] = fm::kRecordBit | fm::kHalfBit | static_cast<std::uint32_t>(k);
    std::uint32_t* dst = pal + k * 4;
    std::uint32_t v[3] = {fm::kEmpty, fm::kEmpty, fm::kEmpty};
    int nd = 0;
    std::uint32_t base = 0xFFFFFFFFu;
    for (int j = 0; j < S; ++j) {
      for (int i = 0; i < S; ++i) {
        if (y0 + j >= ny || x0 + i >= nx) continue;
        const std::uint32_t x = fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i];
        if (x != fm::kEmpty && x >= fm::kRecordBit) base = min(base, x & fm::kSlotIndexMask);
      }
    }
    std::uint32_t codes[2] = {0u, 0u}, half = 0u;
    for (int j = 0; j < S; ++j) {
      for (int i = 0; i < S; ++i) {
        const bool in = y0 + j < ny && x0 + i < nx;
        const std::uint32_t x = in ? fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i] : fm::kEmpty;
        std::uint32_t code;
        if (in && x != fm::kEmpty && x >= fm::kRecordBit) {
          const std::uint32_t off = (x & fm::kSlotIndexMask) - base;
          code = 4u + off;
          if (x & fm::kHalfBit) half |= 1u << off;
        } else {
          code = 0;
          while (static_cast<int>(code) < nd && v[code] != x) ++code;
          if (static_cast<int>(code) == nd) v[nd++] = x;
        }
        const int c = (j << ls) + i;
        codes[c >> 3] |= code << (4 * (c & 7));
      }
    }
    dst[0] = v[0];
    dst[1] = v[1];
    dst[2] = v[2];
    dst[3] = base;
    dst[4] = codes[0];
    dst[5] = codes[1];
    dst[6] = half;
    dst[7] = 0;
    return;
  }
  if (f == 1ull) {  // palette
    const unsigned long long k = idx[b] & 0xFFFFFFFFull;
    blocks[b] = fm::kRecordBit | fm::kHalfBit | static_cast<std::uint32_t>(k);
    std::uint32_t* dst = pal + k * palette_words(ls);
    std::uint32_t v[3] = {fm::kEmpty, fm::kEmpty, fm::kEmpty};
    int nd = 0;
    const int cw = ls <= 2 ? 3 : 4;
    for (int w = 0; w < palette_words(ls); ++w) dst[w] = 0;
    for (int j = 0; j < S; ++j) {
      for (int i = 0; i < S; ++i) {
        const bool in = y0 + j < ny && x0 + i < nx;
        const std::uint32_t x = in ? fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i] : v[0];
        int code = 0;
        while (code < nd && v[code] != x) ++code;
        if (code == nd) v[nd++] = x;
        const int c = (j << ls) + i;
        dst[cw + (c >> 4)] |= static_cast<std::uint32_t>(code) << (2 * (c & 15));
      }
    }
    dst[0] = v[0];
    dst[1] = v[1];
    dst[2] = v[2];
    return;
  }
  const unsigned long long k = idx[b] >> 32;
  blocks[b] = fm::kRecordBit | static_cast<std::uint32_t>(k);
  std::uint32_t* dst = sub + (k << (2 * ls));
  for (int j = 0; j < S; ++j) {
    for (int i = 0; i < S; ++i) {
      const bool in = y0 + j < ny && x0 + i < nx;
      dst[(j << ls) + i] = in ? fine[static_cast<std::size_t>(y0 + j) * nx + x0 + i] : fm::kEmpty;
    }
  }
}

// Tile-major, then block-major renumbering of the phase-1 slots
// (renumber_slots): position p walks tiles of 2^ts x 2^ts cells (the binned
// path's index tiles) in row-major tile order, inside each tile blocks of
// 2^ls x 2^ls cells (the query-side fold) in row-major order, and cells
// row-major inside each block.  So every block's slots are consecutive (the
// fold's compact sub-blocks name them as base + offset) and every tile's
// slots are one contiguous range of the arena (the binned query walks one
// tile at a time).
struct RenumGeom {
  int ts, ls, tnx, nx, ny;
};

__device__ __forceinline__ bool block_major_cell(std::uint64_t p, const RenumGeom& R, std::uint64_t* cell) {
  const std::uint64_t t = p >> (2 * R.ts);
  const std::uint32_t o = static_cast<std::uint32_t>(p & ((1ull << (2 * R.ts)) - 1));
  const int ty = static_cast<int>(t / R.tnx), tx = static_cast<int>(t - static_cast<std::uint64_t>(ty) * R.tnx);
  const int bside = R.ts - R.ls;  // log2 blocks per tile side
  const std::uint32_t b = o >> (2 * R.ls), q = o & ((1u << (2 * R.ls)) - 1);
  const int bx = static_cast<int>(b & ((1u << bside) - 1)), by = static_cast<int>(b >> bside);
  const int x = (tx << R.ts) + (bx << R.ls) + static_cast<int>(q & ((1u << R.ls) - 1));
  const int y = (ty << R.ts) + (by << R.ls) + static_cast<int>(q >> R.ls);
  if (x >= R.nx || y >= R.ny) return false;
  *cell = static_cast<std::uint64_t>(y) * R.nx + x;
  return true;
}

__global__ void __launch_bounds__(256)
    renum_flag_kernel(const std::uint32_t* __restrict__ grid, RenumGeom R, std::uint64_t n_pos,
                      std::uint64_t n1, std::uint32_t* __restrict__ flag) {
  const std::uint64_t p = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n_pos) return;
  std::uint64_t c;
  std::uint32_t f = 0;
  if (block_major_cell(p, R, &c)) {  // slot indices the cell's phase-1 slot takes (double: 2)
    const std::uint32_t e = grid[c];
    f = (e != fm::kEmpty && e >= fm::kRecordBit && (e & fm::kSlotIndexMask) < n1)
            ? ((e & fm::kDoubleBit) && !(e & fm::kHalfBit) ? 2u : 1u)
            : 0u;
  }
  flag[p] = f;
}

__global__ void __launch_bounds__(256)
    renum_apply_kernel(std::uint32_t* __restrict__ grid, RenumGeom R, std::uint64_t n_pos,
                       const std::uint32_t* __restrict__ flag, const std::uint32_t* __restrict__ idx,
                       const uint4* __restrict__ old_slots, uint4* __restrict__ new_slots) {
  const std::uint64_t p = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n_pos || !flag[p]) return;
  std::uint64_t c;
  block_major_cell(p, R, &c);
  const std::uint32_t e = grid[c];
  const std::uint64_t ko = e & fm::kSlotIndexMask, kn = idx[p];
  const int nq = 8 * static_cast<int>(flag[p]);  // 16-byte chunks: 8 per slot index
  for (int q = 0; q < nq; ++q) new_slots[kn * 8 + q] = old_slots[ko * 8 + q];
  grid[c] = (e & ~fm::kSlotIndexMask) | static_cast<std::uint32_t>(kn);
}

// Boundary cells of the exact grid -> (centre point, cell) lists.
__global__ void __launch_bounds__(256)
    deem_collect_kernel(const std::uint32_t* __restrict__ grid, std::uint64_t ncell,
                        std::uint64_t nx, double gx0, double gy0, double w, double h,
                        double2* __restrict__ centres, std::uint64_t* __restrict__ cells,
                        unsigned long long* __restrict__ count) {
  const int lane = threadIdx.x & 31;
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t b0 = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
       b0 < ncell; b0 += stride) {
    const std::uint64_t c = b0 + lane;
    bool rec = false;
    if (c < ncell) {
      const std::uint32_t e = grid[c];
      rec = e != fm::kEmpty && (e & fm::kRecordBit);
    }
    const std::uint32_t m = __ballot_sync(0xFFFFFFFFu, rec);
    if (!m) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, static_cast<unsigned long long>(__popc(m)));
    base = __shfl_sync(0xFFFFFFFFu, base, 0);
    if (rec) {
      const std::uint64_t k = base + __popc(m & ((1u << lane) - 1u));
      const std::uint64_t iy = c / nx, ix = c - iy * nx;
      centres[k] = make_double2(gx0 + (static_cast<double>(ix) + 0.5) * w,
                                gy0 + (static_cast<double>(iy) + 0.5) * h);
      cells[k] = c;
    }
  }
}

// Deemed leaf: the exact answer at the cell centre when it has one (every
// point of the cell is then within half the diagonal of it), else the
// smallest candidate the cell's records list (min_leaf_of_entry).
__global__ void __launch_bounds__(256)
    deem_finish_kernel(fm::KParams P, const std::uint64_t* __restrict__ cells,
                       const int* __restrict__ centre_id, std::uint64_t nb,
                       std::uint32_t* __restrict__ agrid) {
  const std::uint64_t stride = static_cast<std::uint64_t>(gridDim.x) * blockDim.x;
  for (std::uint64_t k = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nb;
       k += stride) {
    const std::uint64_t c = cells[k];
    const int id = centre_id[k];
    agrid[c] = id >= 0 ? static_cast<std::uint32_t>(id) : fm::min_leaf_of_entry(P, P.grid[c]);
  }
}

int resident_blocks(int device, const void* kernel, int block, int smem) {
  // SM count x resident CTAs per SM, cached per (device, kernel, block,
  // smem).  Dynamic shared memory above 48 KB needs the kernel's opt-in
  // limit raised first -- per size, since the binned path's kernels size
  // theirs by the tile count (a launch above the limit would not run).
  struct Slot {
    int device;
    const void* kernel;
    int block, smem;
    int blocks;
  };
  struct Limit {
    int device;
    const void* kernel;
    int smem;
  };
  static std::mutex mu;
  static std::vector<Slot> cache;
  static std::vector<Limit> limits;
  std::lock_guard<std::mutex> lk(mu);
  if (smem > 48 * 1024) {
    bool raised = false;
    for (Limit& l : limits) {
      if (l.device == device && l.kernel == kernel) {
        if (l.smem < smem) {
          cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
          l.smem = smem;
        }
        raised = true;
      }
    }
    if (!raised) {
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      limits.push_back({device, kernel, smem});
    }
  }
  for (const Slot& s : cache) {
    if (s.device == device && s.kernel == kernel && s.block == block && s.smem == smem) return s.blocks;
  }
  int sms = 0, per_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
  const int blocks = std::max(1, sms) * std::max(1, per_sm);
  cache.push_back({device, kernel, block, smem, blocks});
  return blocks;
}

// A grid folded into blocks of 2^ls x 2^ls cells (see KParams).  `owned`
// is false when `blocks` aliases the flat grid (ls = 0).
struct Folded {
  std::uint32_t* blocks = nullptr;
  std::uint32_t* sub = nullptr;
  std::uint32_t* pal = nullptr;  // compact sub-blocks (approx palettes / exact compact)
  int ls = 0, bnx = 0, bny = 0;
  int compact = 0;               // 1: `pal` holds exact compact sub-blocks
  bool owned = false;
  std::uint64_t bytes = 0;
  void release() {
    if (owned && blocks) cudaFree(blocks);
    if (sub) cudaFree(sub);
    if (pal) cudaFree(pal);
    blocks = nullptr;
    sub = nullptr;
    pal = nullptr;
  }
};

}  // namespace

struct fm_index {
  int device = -1;
  fm::GridGeom g{};
  double ax0 = 0, ax1 = 0, ay0 = 0, ay1 = 0;
  std::uint32_t* d_grid = nullptr;
  Folded qgrid;                        // query-side folded copy of the exact grid
  Folded agrid;                        // fast-approx cover (folded), or empty
  TileGeom tiles;                      // binned query path: the index tiles
  int query_path = FM_PATH_AUTO;       // fm_query_path
  double tile_bytes = 0.0;             // index bytes per tile (0 = default)
  std::uint8_t* d_slots = nullptr;     // boundary slots (128 B each)
  std::uint8_t* d_overflow = nullptr;  // overflow records
  std::uint64_t grid_len = 0, slots_len = 0, overflow_len = 0;
  fm::HostIndex host;  // retained only for host-only (device < 0) indexes
  fm_index_stats stats{};
  // fm_query_host staging
  std::mutex mu;
  bool staged = false;
  cudaStream_t streams[kStreams] = {};
  double* d_in[kStreams] = {};
  int* d_out[kStreams] = {};
  unsigned long long* d_hist = nullptr;
  unsigned long long* d_counters = nullptr;  // fm_query_host_counted, per stream
};

namespace {

fm::KParams kparams(const fm_index* ix) {
  fm::KParams P;
  P.grid = ix->d_grid;
  P.slots = ix->d_slots;
  P.overflow = ix->d_overflow;
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
  P.blocks = ix->qgrid.blocks;
  P.sub = ix->qgrid.sub;
  P.pal = ix->qgrid.pal;
  P.compact = ix->qgrid.compact;
  P.bnx = ix->qgrid.bnx;
  P.ls = ix->qgrid.ls;
  return P;
}

template <bool kHist, bool kCount>
fm_status launch_t(const fm_index* ix, const double2* pts, std::uint64_t n, int* d_out,
                   HistT* d_hist, unsigned long long* d_counters, cudaStream_t stream) {
  const fm::KParams P = kparams(ix);
  // a flat query grid (no fold) gets its own instantiation without the
  // second-level code (all-hit stream: 0.50 -> 0.35 ms per 100M points);
  // folded grids read the block size at run time (measured faster on c2
  // than a constant-ls instantiation: 1.17 vs 1.21 ms)
  auto ka = ix->qgrid.ls == 0 ? stream_kernel<kHist, kCount, 0> : stream_kernel<kHist, kCount, -1>;
  auto kb = resolve_kernel<kHist, kCount>;
  const int blk_a = kAWarps * 32;
  const std::uint64_t tile = 32ull * kU;
  const std::uint64_t n_tiles = (n + tile - 1) / tile;
  const int grid_a = static_cast<int>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>((n_tiles + kAWarps - 1) / kAWarps,
                                 resident_blocks(ix->device, (const void*)ka, blk_a, 0))));
  const std::uint64_t n_regions = static_cast<std::uint64_t>(grid_a) * kAWarps;
  const std::uint64_t region_cap = (n_tiles + n_regions - 1) / n_regions * tile;
  // stream-ordered scratch: the boundary queue (24 B/item) and its counts
  void* scratch = nullptr;
  const std::uint64_t qbytes = n_regions * region_cap * sizeof(QItem);
  FM_CUDA(cudaMallocAsync(&scratch, qbytes + n_regions * 4 + 16, stream));
  QItem* q = static_cast<QItem*>(scratch);
  std::uint32_t* qcount = reinterpret_cast<std::uint32_t*>(static_cast<char*>(scratch) + qbytes);
  unsigned long long* next_region =
      reinterpret_cast<unsigned long long*>(static_cast<char*>(scratch) + qbytes + n_regions * 4);
  if ((reinterpret_cast<std::uintptr_t>(next_region) & 7u) != 0) {
    next_region = reinterpret_cast<unsigned long long*>((reinterpret_cast<std::uintptr_t>(next_region) + 7) & ~std::uintptr_t{7});
  }
  FM_CUDA(cudaMemsetAsync(next_region, 0, 8, stream));
  ka<<<grid_a, blk_a, 0, stream>>>(P, pts, n, d_out, d_hist, q, qcount, region_cap, d_counters);
  // persistent resolve grid: resident CTAs pull regions from a counter
  const int grid_b = static_cast<int>(std::min<std::uint64_t>(
      (n_regions + kBWarps - 1) / kBWarps,
      resident_blocks(ix->device, (const void*)kb, kBWarps * 32, kSmemB)));
  kb<<<grid_b, kBWarps * 32, kSmemB, stream>>>(P, q, qcount, n_regions, region_cap, next_region,
                                               d_out, d_hist, d_counters);
  const cudaError_t err = cudaGetLastError();
  FM_CUDA(cudaFreeAsync(scratch, stream));
  if (err != cudaSuccess) return set_err(FM_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(err));
  return FM_OK;
}

// The binned path (binned.cuh) over one batch of n <= kBinnedBatch points.
constexpr std::uint64_t kBinnedBatch = std::uint64_t{1} << 30;

std::uint64_t align256(std::uint64_t v) { return (v + 255) & ~std::uint64_t{255}; }

template <bool kHist, bool kCount>
fm_status launch_binned_t(const fm_index* ix, const double2* pts, std::uint64_t n, int* d_out,
                          HistT* d_hist, unsigned long long* d_counters, cudaStream_t stream) {
  const fm::KParams P = kparams(ix);
  const TileGeom& T = ix->tiles;
  const int nk = T.n_tiles + 1;
  const int nk4 = (nk + 3) & ~3;
  const int tile_smem = nk * 4;
  // sampled bin capacities, one scatter pass (binned.cuh)
  const std::uint64_t ovf_cap = bin_overflow_cap(n);
  const std::uint64_t nb = bin_capacity_bound(n, nk) + ovf_cap;  // binned length bound
  if (nb >= (std::uint64_t{1} << 31)) return set_err(FM_ERR_RUNTIME, "binned batch too large");  // the kernels index it in 32 bits
  // scratch: work counters + binned length, sample counts, the bin table,
  // binned points, binned positions, binned answers
  const std::uint64_t o_work = 0;
  const std::uint64_t o_cnt = 256;
  const std::uint64_t o_bin = o_cnt + align256(4 * static_cast<std::uint64_t>(nk));
  const std::uint64_t o_pts = o_bin + align256(4 * (3 * static_cast<std::uint64_t>(nk4) + 4));
  const std::uint64_t o_pos = o_pts + align256(16 * nb);
  // per point its sorted index inside its chunk (2 B), per chunk the run table
  const std::uint64_t n_chunks = (n + kChunk - 1) / kChunk;
  const std::uint64_t o_tab = o_pos + align256(2 * n);
  const std::uint64_t o_res = o_tab + align256(4 * tab_stride(nk4) * n_chunks);
  const std::uint64_t total = o_res + align256(4 * nb);
  char* scratch = nullptr;
  FM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), total, stream));
  unsigned long long* work = reinterpret_cast<unsigned long long*>(scratch + o_work);
  unsigned int* counts = reinterpret_cast<unsigned int*>(scratch + o_cnt);
  BinTable B;
  B.start = reinterpret_cast<unsigned int*>(scratch + o_bin);
  B.cap = B.start + nk4;
  B.cur = B.cap + nk4;
  B.hdr = B.cur + nk4;
  B.n_eff = work + kCtrCount;
  FM_CUDA(cudaMemsetAsync(scratch, 0, o_bin, stream));  // work counters, n_eff, sample counts
  double2* pts_b = reinterpret_cast<double2*>(scratch + o_pts);
  int* res = reinterpret_cast<int*>(scratch + o_res);
  {
    auto k0 = bin_sample_kernel;
    const std::uint64_t span = static_cast<std::uint64_t>(kSampleStride) * kSampleGroup;
    const std::uint64_t strata = (n + span - 1) / span;
    const int grid0 = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
        (strata + kSampleThreads - 1) / kSampleThreads,
        resident_blocks(ix->device, (const void*)k0, kSampleThreads, tile_smem))));
    k0<<<grid0, kSampleThreads, tile_smem, stream>>>(P, T, pts, n, counts);
  }
  bin_plan_kernel<<<1, kPlanThreads, 0, stream>>>(nk, ovf_cap, counts, B);
  std::uint16_t* pos16 = reinterpret_cast<std::uint16_t*>(scratch + o_pos);
  unsigned int* tab = reinterpret_cast<unsigned int*>(scratch + o_tab);
  auto ks = bin_scatter_kernel;
  const int sc_smem = sc2_smem(nk4);
  const int grid_s = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
      n_chunks, resident_blocks(ix->device, (const void*)ks, kSc2Threads, sc_smem))));
  ks<<<grid_s, kSc2Threads, sc_smem, stream>>>(P, T, pts, n, B, pts_b, pos16, tab);
  bin_seal_kernel<<<std::min(nk, 1184), 256, 0, stream>>>(nk, B, pts_b, kCount ? d_counters : nullptr);
  const unsigned long long* n_dev = B.n_eff;
  // the histogram is counted from res afterwards (binned_hist_kernel): in
  // binned order its leaves repeat within a chunk, and the query kernel
  // stays free of per-point counter atomics
  auto kq = ix->qgrid.ls == 0 ? binned_query_kernel<false, kCount, 0>
                              : binned_query_kernel<false, kCount, -1>;
  const std::uint64_t n_qt = (nb + 32ull * kU - 1) / (32ull * kU);
  const int grid_q = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
      (n_qt + kQWarps * kQGroup - 1) / (kQWarps * kQGroup),
      resident_blocks(ix->device, (const void*)kq, kQWarps * 32, kSmemQ))));
  kq<<<grid_q, kQWarps * 32, kSmemQ, stream>>>(P, pts_b, nb, n_dev, res, nullptr, d_counters, work);
  if (kHist) {
    auto kh = binned_hist_kernel;
    const int grid_h = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
        (nb + kHistStep - 1) / kHistStep, resident_blocks(ix->device, (const void*)kh, kHistThreads, kHistSmem))));
    kh<<<grid_h, kHistThreads, kHistSmem, stream>>>(res, nb, n_dev, d_hist);
  }
  auto ku = unbin_kernel;
  const int ub_smem = ub2_smem(nk4);
  const int grid_u = static_cast<int>(std::max<std::uint64_t>(1, std::min<std::uint64_t>(
      n_chunks, resident_blocks(ix->device, (const void*)ku, kUb2Threads, ub_smem))));
  ku<<<grid_u, kUb2Threads, ub_smem, stream>>>(pos16, tab, nk, B, res, n, d_out, work);
  unplaced_kernel<<<grid_u, 256, 0, stream>>>(B, n, P, pts, d_out, kHist ? d_hist : nullptr,
                                               kCount ? d_counters : nullptr);
  const cudaError_t err = cudaGetLastError();
  FM_CUDA(cudaFreeAsync(scratch, stream));
  if (err != cudaSuccess) return set_err(FM_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(err));
  return FM_OK;
}

// Query path for a batch of n points (fm_query_path): the binned path when
// the index is far larger than L2 and mostly boundary cells -- then the
// stream path's per-point gathers miss L2 (c3: 15 GB of slots, 60% boundary
// cells, binned 37.0 ms vs stream 46.8 ms per 1B points; c4: 6 GB, 50%,
// 8.2 vs 8.8 ms per 200M, profiles/r2u) -- and the batch is big enough to
// reuse tiles; the stream path otherwise (c1; c2: 9% boundary cells, 1.13
// vs 2.8 ms per 100M).
// The index side of the choice: far larger than L2 and mostly boundary cells.
bool binned_index(const fm_index* ix) {
  const double cells = static_cast<double>(ix->g.nx) * static_cast<double>(ix->g.ny);
  const double bfrac = cells > 0 ? static_cast<double>(ix->stats.cells_boundary) / cells : 0.0;
  const double bytes = static_cast<double>(ix->grid_len * 4 + ix->stats.arena_bytes);
  return bytes >= 1e9 && bfrac >= 0.25;
}
bool use_binned(const fm_index* ix, std::uint64_t n) {
  if (ix->query_path == FM_PATH_STREAM) return false;
  if (ix->query_path == FM_PATH_BINNED) return true;
  return n >= (std::uint64_t{1} << 24) && binned_index(ix);
}

// Tiles of 2^ts x 2^ts cells holding about `tile_bytes` of index (query
// grid + slot arena, averaged over the grid), at most kMaxTiles.
TileGeom plan_tiles(const fm::GridGeom& g, const fm_index_stats& st, double tile_bytes) {
  const double cells = std::max(1.0, static_cast<double>(g.nx) * static_cast<double>(g.ny));
  const double per_cell = static_cast<double>(st.query_grid_bytes + st.arena_bytes) / cells;
  const double side = std::sqrt(tile_bytes / std::max(per_cell, 1.0));
  int ts = std::max(2, static_cast<int>(std::lround(std::log2(std::max(side, 1.0)))));
  TileGeom T;
  for (;; ++ts) {
    T.ts = ts;
    T.tnx = static_cast<int>((g.nx + (1ll << ts) - 1) >> ts);
    T.tny = static_cast<int>((g.ny + (1ll << ts) - 1) >> ts);
    T.n_tiles = T.tnx * T.tny;
    if (T.n_tiles <= kMaxTiles) break;
  }
  return T;
}
constexpr double kTileBytes = 64e6;  // c3: 162 tiles (37.2 ms) vs 630 (40.3), profiles/r2u

template <bool kHist, bool kCount>
fm_status launch_approx_t(const fm_index* ix, const double2* pts, std::uint64_t n, int* d_out,
                          unsigned long long* d_hist, unsigned long long* d_counters,
                          cudaStream_t stream) {
  fm::KParams A = kparams(ix);
  A.blocks = ix->agrid.blocks;
  A.sub = ix->agrid.sub;
  A.pal = ix->agrid.pal;
  A.compact = ix->agrid.compact;
  A.bnx = ix->agrid.bnx;
  A.ls = ix->agrid.ls;
  auto k = approx_kernel<kHist, kCount>;
  const std::uint64_t chunk = static_cast<std::uint64_t>(kXThreads) * kXU;
  const int grid = static_cast<int>(std::max<std::uint64_t>(
      1, std::min<std::uint64_t>((n + chunk - 1) / chunk,
                                 resident_blocks(ix->device, (const void*)k, kXThreads, 0))));
  k<<<grid, kXThreads, 0, stream>>>(A, pts, n, d_out, d_hist, d_counters);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_err(FM_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(err));
  return FM_OK;
}

__global__ void __launch_bounds__(256)
    widen_hist_kernel(HistT* __restrict__ h32, unsigned long long* __restrict__ h64, std::uint64_t n) {
  const std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const HistT v = h32[i];
  if (v) {  // atomic: queries on other streams may add into the same histogram
    atomicAdd(h64 + i, static_cast<unsigned long long>(v));
    h32[i] = 0;
  }
}

fm_status launch(const fm_index* ix, const double* d_pts, std::uint64_t n, int* d_out,
                 unsigned long long* d_hist, unsigned long long* d_counters,
                 cudaStream_t stream, int mode = FM_MODE_EXACT) {
  const double2* pts = reinterpret_cast<const double2*>(d_pts);
  if (mode == FM_MODE_APPROX && ix->agrid.blocks) {
    if (d_hist && d_counters) return launch_approx_t<true, true>(ix, pts, n, d_out, d_hist, d_counters, stream);
    if (d_hist) return launch_approx_t<true, false>(ix, pts, n, d_out, d_hist, d_counters, stream);
    if (d_counters) return launch_approx_t<false, true>(ix, pts, n, d_out, d_hist, d_counters, stream);
    return launch_approx_t<false, false>(ix, pts, n, d_out, d_hist, d_counters, stream);
  }
  // slices of 2^28 points bound the stream path's queue scratch (24 B/point)
  // to 6.4 GB; binned batches of 2^30 points take 24 GB (binned.cuh).  Both
  // keep the u32 histogram counters from overflowing.
  const std::uint64_t slice = std::uint64_t{1} << 28;
  const std::uint64_t nh = ix->stats.n_polys;
  HistT* h32 = nullptr;
  if (d_hist && n > 0 && nh > 0) {
    FM_CUDA(cudaMallocAsync(&h32, nh * sizeof(HistT), stream));
    FM_CUDA(cudaMemsetAsync(h32, 0, nh * sizeof(HistT), stream));
  }
  fm_status st = FM_OK;
  const bool binned = use_binned(ix, n);
  const std::uint64_t step = binned ? kBinnedBatch : slice;
  for (std::uint64_t off = 0; off < n && st == FM_OK; off += step) {
    const std::uint64_t m = std::min(step, n - off);
    if (binned) {
      if (h32 && d_counters) {
        st = launch_binned_t<true, true>(ix, pts + off, m, d_out + off, h32, d_counters, stream);
      } else if (h32) {
        st = launch_binned_t<true, false>(ix, pts + off, m, d_out + off, h32, d_counters, stream);
      } else if (d_counters) {
        st = launch_binned_t<false, true>(ix, pts + off, m, d_out + off, nullptr, d_counters, stream);
      } else {
        st = launch_binned_t<false, false>(ix, pts + off, m, d_out + off, nullptr, d_counters, stream);
      }
    } else if (h32 && d_counters) {
      st = launch_t<true, true>(ix, pts + off, m, d_out + off, h32, d_counters, stream);
    } else if (h32) {
      st = launch_t<true, false>(ix, pts + off, m, d_out + off, h32, d_counters, stream);
    } else if (d_counters) {
      st = launch_t<false, true>(ix, pts + off, m, d_out + off, nullptr, d_counters, stream);
    } else {
      st = launch_t<false, false>(ix, pts + off, m, d_out + off, nullptr, d_counters, stream);
    }
    if (st == FM_OK && h32) {
      widen_hist_kernel<<<static_cast<unsigned>((nh + 255) / 256), 256, 0, stream>>>(h32, d_hist, nh);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) st = set_err(FM_ERR_CUDA, std::string("histogram: ") + cudaGetErrorString(e));
    }
  }
  if (h32) cudaFreeAsync(h32, stream);
  return st;
}

// Fold a flat nx x ny grid into blocks (KParams): the smallest ls <= max_ls
// whose block level fits `budget` bytes.  ls = 0 aliases the flat grid.
int fold_ls(int nx, int ny, std::uint64_t budget, int max_ls) {
  int ls = 0;
  while (ls < max_ls && static_cast<std::uint64_t>((nx + (1 << ls) - 1) >> ls) *
                                static_cast<std::uint64_t>((ny + (1 << ls) - 1) >> ls) * 4 > budget) {
    ++ls;
  }
  return ls;
}

// mode: 0 = full sub-blocks only, 1 = approx palettes, 2 = exact compact
// sub-blocks (slot references < n1 must be numbered block-major).
fm_status fold_grid(std::uint32_t* fine, int nx, int ny, std::uint64_t budget, int max_ls,
                    int mode, std::uint64_t n1, double max_ratio, Folded* out) {
  const int ls = fold_ls(nx, ny, budget, max_ls);
  const int bnx = (nx + (1 << ls) - 1) >> ls, bny = (ny + (1 << ls) - 1) >> ls;
  const std::uint64_t nblk = static_cast<std::uint64_t>(bnx) * bny;
  out->ls = ls;
  out->compact = mode == 2 ? 1 : 0;
  out->bnx = bnx;
  out->bny = bny;
  if (ls == 0) {
    out->blocks = fine;
    out->owned = false;
    FM_CUDA(cudaMalloc(&out->sub, 64));
    FM_CUDA(cudaMalloc(&out->pal, 64));
    out->bytes = nblk * 4;
    return FM_OK;
  }
  unsigned long long *flag = nullptr, *idx = nullptr;
  void* tmp = nullptr;
  std::size_t tmp_bytes = 0;
  unsigned long long tot = 0;
  cudaError_t e = cudaMalloc(&flag, (nblk + 1) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&idx, (nblk + 1) * 8);
  if (e == cudaSuccess) e = cudaMemset(flag + nblk, 0, 8);
  const unsigned g1 = static_cast<unsigned>((nblk + 255) / 256);
  if (e == cudaSuccess) {
    block_flag_kernel<<<g1, 256>>>(fine, nx, ny, bnx, bny, ls, mode, n1, flag);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, idx, static_cast<std::int64_t>(nblk + 1));
  }
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes + 16);
  if (e == cudaSuccess) {
    e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, idx, static_cast<std::int64_t>(nblk + 1));
  }
  if (e == cudaSuccess) e = cudaMemcpy(&tot, idx + nblk, 8, cudaMemcpyDeviceToHost);
  const std::uint64_t n_pal = tot & 0xFFFFFFFFull, n_sub = tot >> 32;
  const int pw0 = mode == 2 ? 4 : palette_words(ls);
  const double folded = static_cast<double>(nblk * 4 + (n_sub << (2 * ls + 2)) + n_pal * pw0 * 4);
  if (e == cudaSuccess && folded > max_ratio * 4.0 * nx * static_cast<double>(ny)) {
    // the fold would not shrink the grid enough to pay for its second
    // gather (c3: 67% boundary cells): query the flat grid directly
    cudaFree(tmp);
    cudaFree(flag);
    cudaFree(idx);
    out->ls = 0;
    out->bnx = nx;
    out->bny = ny;
    out->compact = 0;
    out->blocks = fine;
    out->owned = false;
    FM_CUDA(cudaMalloc(&out->sub, 64));
    FM_CUDA(cudaMalloc(&out->pal, 64));
    out->bytes = static_cast<std::uint64_t>(nx) * ny * 4;
    return FM_OK;
  }
  if (e == cudaSuccess) {
    out->owned = true;
    e = cudaMalloc(&out->blocks, nblk * 4);
  }
  if (e == cudaSuccess) e = cudaMalloc(&out->sub, std::max<std::uint64_t>(n_sub, 1) << (2 * ls + 2));
  const int pw = mode == 2 ? 4 : palette_words(ls);
  if (e == cudaSuccess) e = cudaMalloc(&out->pal, std::max<std::uint64_t>(n_pal, 1) * pw * 4);
  if (e == cudaSuccess) {
    block_write_kernel<<<g1, 256>>>(fine, nx, ny, bnx, bny, ls, mode, flag, idx, out->blocks,
                                    out->sub, out->pal);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  out->bytes = nblk * 4 + (n_sub << (2 * ls + 2)) + n_pal * pw * 4;
  cudaFree(tmp);
  cudaFree(flag);
  cudaFree(idx);
  if (e != cudaSuccess) return set_err(FM_ERR_CUDA, std::string("grid folding: ") + cudaGetErrorString(e));
  return FM_OK;
}

// Renumber the phase-1 slots tile-major (tiles of 2^ts cells), block-major
// inside tiles (blocks of 2^ls cells), so every block's phase-1 slots are
// consecutive and its sub-block can name them as base + offset (exact
// compact sub-blocks), and every tile's are contiguous.  Phase-2 slots
// (split / overflow subtrees and double slots) keep their numbers.
fm_status renumber_slots(fm_index* ix, int ts, int ls) {
  const std::uint64_t n1 = ix->host.n_phase1_slots;
  if (n1 == 0) return FM_OK;
  const int nx = static_cast<int>(ix->g.nx), ny = static_cast<int>(ix->g.ny);
  ts = std::max(ts, ls);
  RenumGeom R{ts, ls, (nx + (1 << ts) - 1) >> ts, nx, ny};
  const int tny = (ny + (1 << ts) - 1) >> ts;
  const std::uint64_t n_pos = (static_cast<std::uint64_t>(R.tnx) * tny) << (2 * ts);
  std::uint32_t *flag = nullptr, *idx = nullptr;
  std::uint8_t* fresh = nullptr;
  void* tmp = nullptr;
  std::size_t tmp_bytes = 0;
  cudaError_t e = cudaMalloc(&flag, n_pos * 4);
  if (e == cudaSuccess) e = cudaMalloc(&idx, n_pos * 4);
  if (e == cudaSuccess) e = cudaMalloc(&fresh, ix->slots_len);
  const unsigned g1 = static_cast<unsigned>((n_pos + 255) / 256);
  if (e == cudaSuccess) {
    renum_flag_kernel<<<g1, 256>>>(ix->d_grid, R, n_pos, n1, flag);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, idx, static_cast<std::int64_t>(n_pos));
  }
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes + 16);
  if (e == cudaSuccess) {
    e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, idx, static_cast<std::int64_t>(n_pos));
  }
  if (e == cudaSuccess) {
    renum_apply_kernel<<<g1, 256>>>(ix->d_grid, R, n_pos, flag, idx,
                                    reinterpret_cast<const uint4*>(ix->d_slots),
                                    reinterpret_cast<uint4*>(fresh));
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && ix->slots_len > n1 * fm::kSlotBytes) {  // phase-2 tail
    e = cudaMemcpy(fresh + n1 * fm::kSlotBytes, ix->d_slots + n1 * fm::kSlotBytes,
                   ix->slots_len - n1 * fm::kSlotBytes, cudaMemcpyDeviceToDevice);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(tmp);
  cudaFree(flag);
  cudaFree(idx);
  if (e != cudaSuccess) {
    cudaFree(fresh);
    return set_err(FM_ERR_CUDA, std::string("slot renumbering: ") + cudaGetErrorString(e));
  }
  cudaFree(ix->d_slots);
  ix->d_slots = fresh;
  return FM_OK;
}

// Query-side block level of the exact grid: a 2x2 fold when the flat grid
// exceeds kQueryBudget (c2: 105 MB flat -> 26 MB blocks + 16-byte sub-blocks).
constexpr std::uint64_t kQueryBudget = std::uint64_t{32} << 20;
#ifndef FM_QUERY_MAX_LS
#define FM_QUERY_MAX_LS 2
#endif
constexpr int kQueryMaxLs = FM_QUERY_MAX_LS;
// ...and only when the folded copy is at most this fraction of the flat grid
constexpr double kQueryMaxRatio = 0.75;

// The approx cover: copy the exact grid, query every boundary cell's centre
// through the exact path, write the deemed leaves, then fold the fine grid
// into S x S blocks (the smallest S whose block level fits kBlockBudget).
constexpr std::uint64_t kBlockBudget = std::uint64_t{48} << 20;

fm_status build_approx(fm_index* ix) {
  const std::uint64_t ncell = ix->grid_len;
  const std::uint64_t nb = ix->stats.cells_boundary;
  std::uint32_t* fine = nullptr;
  FM_CUDA(cudaMalloc(&fine, ncell * 4));
  FM_CUDA(cudaMemcpy(fine, ix->d_grid, ncell * 4, cudaMemcpyDeviceToDevice));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
  const int blocks = std::max(1, sms) * 8;
  fm_status st = FM_OK;
  cudaError_t e = cudaSuccess;
  if (nb > 0) {
    void* scratch = nullptr;
    const std::uint64_t bytes = nb * (16 + 8 + 4) + 64;
    e = cudaMalloc(&scratch, bytes);
    if (e == cudaSuccess) {
      double2* centres = static_cast<double2*>(scratch);
      std::uint64_t* cells = reinterpret_cast<std::uint64_t*>(centres + nb);
      int* ids = reinterpret_cast<int*>(cells + nb);
      unsigned long long* count = reinterpret_cast<unsigned long long*>(
          (reinterpret_cast<std::uintptr_t>(ids + nb) + 7) & ~std::uintptr_t{7});
      e = cudaMemset(count, 0, 8);
      if (e == cudaSuccess) {
        deem_collect_kernel<<<blocks, 256>>>(ix->d_grid, ncell, static_cast<std::uint64_t>(ix->g.nx),
                                             ix->g.gx0, ix->g.gy0, ix->g.w, ix->g.h, centres,
                                             cells, count);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) {
        st = launch(ix, reinterpret_cast<const double*>(centres), nb, ids, nullptr, nullptr, 0);
        if (st == FM_OK) {
          deem_finish_kernel<<<blocks, 256>>>(kparams(ix), cells, ids, nb, fine);
          e = cudaGetLastError();
          if (e == cudaSuccess) e = cudaDeviceSynchronize();
        }
      }
      cudaFree(scratch);
    }
  }
  if (st == FM_OK && e == cudaSuccess) {
    st = fold_grid(fine, static_cast<int>(ix->g.nx), static_cast<int>(ix->g.ny), kBlockBudget, 3,
                   1, 0, 1e30, &ix->agrid);
    if (st == FM_OK && ix->agrid.ls == 0) {
      ix->agrid.owned = true;  // the approx copy itself is the block level
      fine = nullptr;
    }
    ix->stats.approx_grid_bytes = ix->agrid.bytes;
    ix->stats.approx_block_log2 = ix->agrid.ls;
  }
  if (fine) cudaFree(fine);
  if (st != FM_OK) return st;
  if (e != cudaSuccess) return set_err(FM_ERR_CUDA, std::string("approx cover: ") + cudaGetErrorString(e));
  return FM_OK;
}

// Query-side layout of a device index (shared by fm_index_build and
// fm_index_load): mempool policy, block-major slot numbering + the folded
// grid, and the approx cover when epsilon > 0.
fm_status finish_device(fm_index* ix, double approx_epsilon) {
  DeviceGuard guard(ix->device);
  if (!guard.ok) return set_err(FM_ERR_CUDA, "cudaSetDevice failed");
  // keep stream-ordered scratch (the boundary queue) cached between calls
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, ix->device) == cudaSuccess) {
    std::uint64_t thr = ~std::uint64_t{0};
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  const int nx = static_cast<int>(ix->g.nx), ny = static_cast<int>(ix->g.ny);
  // An index the binned path will take (binned_index below) keeps its flat
  // grid: a tile's 4 MB of flat entries are L2-resident while the tile is
  // walked, so the fold only adds a dependent gather (c3 at 7 / 8 cells per
  // leaf side: 31.5 / 30.6 ms per 1B points folded, 23.2 / 22.3 flat; the
  // stream path 43.4 / 43.1 against 40.4 / 39.3 -- profiles/r2bz, r2ca).
  const int max_ls = binned_index(ix) ? 0 : kQueryMaxLs;
  const int qls = fold_ls(nx, ny, kQueryBudget, max_ls);
  // the binned path's default tiles (index bytes per cell before the fold:
  // the flat grid plus the slot arena)
  fm_index_stats pre = ix->stats;
  pre.query_grid_bytes = ix->grid_len * 4;
  const TileGeom T0 = plan_tiles(ix->g, pre, kTileBytes);
  fm_status st = renumber_slots(ix, T0.ts, qls);
  if (st == FM_OK) {
    st = fold_grid(ix->d_grid, nx, ny, kQueryBudget, max_ls, 2, ix->host.n_phase1_slots,
                   kQueryMaxRatio, &ix->qgrid);
  }
  if (st != FM_OK) return st;
  ix->stats.query_grid_bytes = ix->qgrid.bytes;
  ix->stats.query_block_log2 = ix->qgrid.ls;
  ix->tiles = ix->tile_bytes > 0 ? plan_tiles(ix->g, ix->stats, ix->tile_bytes) : T0;
  ix->stats.approx_epsilon = approx_epsilon;
  // an epsilon too fine for the uniform approx grid: approximate queries
  // take the exact path (fm_index_stats.approx_grid_bytes stays 0)
  if (approx_epsilon > 0.0 && !ix->host.stats.approx_served_exact) return build_approx(ix);
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
  if (ix->d_counters) cudaFree(ix->d_counters);
  if (ix->d_grid) cudaFree(ix->d_grid);
  ix->qgrid.release();
  ix->agrid.release();
  if (ix->d_slots) cudaFree(ix->d_slots);
  if (ix->d_overflow) cudaFree(ix->d_overflow);
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

// For simple.cu (not part of the C-ABI): the query-side kernel parameters
// of a device index, for device-side single-point lookups.
__attribute__((visibility("hidden"))) bool fm_index_kparams(const fm_index* ix, fm::KParams* out) {
  if (!ix || ix->device < 0) return false;
  *out = kparams(ix);
  return true;
}

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
  // validate_cover_params (cell_index.hpp:382-394): the level-30 diagonal floor
  const double eps_floor = std::hypot(360.0 / 1073741824.0, 180.0 / 1073741824.0);
  if (std::isnan(p.approx_epsilon) || p.approx_epsilon < 0.0 ||
      (p.approx_epsilon > 0.0 && p.approx_epsilon < eps_floor)) {
    return set_err(FM_ERR_INVALID_ARGUMENT,
                   "approx epsilon must be at least the level-30 cell diagonal (" +
                       std::to_string(eps_floor) + " degrees)");
  }
  opt.approx_epsilon = p.approx_epsilon;

  fm_index* ix = new (std::nothrow) fm_index();
  if (!ix) return set_err(FM_ERR_OOM, "host allocation failed");
  const auto t0 = std::chrono::steady_clock::now();
  const bool on_gpu = p.build_on_gpu && p.device >= 0;
  try {
    if (on_gpu) {
      fm::build_index_gpu(soup, opt, p.device, ix->host, &ix->d_grid, &ix->d_slots, &ix->slots_len,
                          &ix->d_overflow, &ix->overflow_len);
      ix->device = p.device;
    } else {
      ix->host = fm::build_index_host(soup, opt);
    }
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
  ix->grid_len = static_cast<std::uint64_t>(ix->g.nx * ix->g.ny);
  if (!on_gpu) {
    ix->slots_len = ix->host.slots.size();
    ix->overflow_len = ix->host.overflow.size();
  }

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
  s.arena_bytes = ix->host.n_slots * fm::kSlotBytes + (ix->overflow_len - 512);
  s.built_on_gpu = on_gpu ? 1 : 0;
  s.cells_split = ix->host.stats.cells_split;
  s.slots_double = ix->host.stats.slots_double;
  for (int k = 0; k < 6; ++k) s.build_phase_seconds[k] = ix->host.stats.phase_s[k];
  s.slots_phase1 = ix->host.n_phase1_slots;
  s.slots_total = ix->host.n_slots;
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

  if (ix->device >= 0 && !on_gpu) {
    DeviceGuard guard(ix->device);
    if (!guard.ok) {
      delete ix;
      return set_err(FM_ERR_CUDA, "cudaSetDevice failed");
    }
    cudaError_t e1 = cudaMalloc(&ix->d_grid, ix->grid_len * 4);
    cudaError_t e2 = cudaMalloc(&ix->d_slots, ix->slots_len);
    cudaError_t e3 = cudaMalloc(&ix->d_overflow, ix->overflow_len);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      free_device(ix);
      delete ix;
      return set_err(FM_ERR_OOM, "device allocation of the index failed");
    }
    e1 = cudaMemcpy(ix->d_grid, ix->host.grid.data(), ix->grid_len * 4, cudaMemcpyHostToDevice);
    e2 = cudaMemcpy(ix->d_slots, ix->host.slots.data(), ix->slots_len, cudaMemcpyHostToDevice);
    e3 = cudaMemcpy(ix->d_overflow, ix->host.overflow.data(), ix->overflow_len, cudaMemcpyHostToDevice);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      free_device(ix);
      delete ix;
      return set_err(FM_ERR_CUDA, "index upload failed");
    }
    // the device copy is authoritative; drop the host arrays
    std::vector<std::uint32_t>().swap(ix->host.grid);
    std::vector<std::uint8_t>().swap(ix->host.slots);
    std::vector<std::uint8_t>().swap(ix->host.overflow);
  }
  if (ix->device >= 0) {
    const fm_status st = finish_device(ix, p.approx_epsilon);
    if (st != FM_OK) {
      free_device(ix);
      delete ix;
      return st;
    }
  }
  s.approx_epsilon = p.approx_epsilon;
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

}  // extern "C"

namespace {
fm_status check_mode(const fm_index* index, int mode) {
  if (mode != FM_MODE_EXACT && mode != FM_MODE_APPROX) {
    return set_err(FM_ERR_INVALID_ARGUMENT, "unknown cover mode");
  }
  if (mode == FM_MODE_APPROX && index->stats.approx_epsilon <= 0.0) {  // cell_index.hpp:532-535
    return set_err(FM_ERR_INVALID_ARGUMENT, "approximate queries require an approximate-mode cover");
  }
  return FM_OK;
}
}  // namespace

__attribute__((visibility("hidden"))) fm_status query_host_impl(
    const fm_index* cindex, int mode, const double* h_lonlat, std::uint64_t n, std::int32_t* h_out,
    std::int64_t* h_hist, std::int64_t* d_hist_accum, fm_query_counters* h_counters);

extern "C" {

fm_status fm_query(const fm_index* index, const double* d_lonlat, std::uint64_t n,
                   std::int32_t* d_out, std::int64_t* d_hist, fm_query_counters* d_counters,
                   void* stream) {
  return fm_query_mode(index, FM_MODE_EXACT, d_lonlat, n, d_out, d_hist, d_counters, stream);
}

fm_status fm_query_host(const fm_index* index, const double* h_lonlat, std::uint64_t n,
                        std::int32_t* h_out, std::int64_t* h_hist) {
  return fm_query_host_mode(index, FM_MODE_EXACT, h_lonlat, n, h_out, h_hist);
}

fm_status fm_query_mode(const fm_index* index, int mode, const double* d_lonlat, std::uint64_t n,
                        std::int32_t* d_out, std::int64_t* d_hist, fm_query_counters* d_counters,
                        void* stream) {
  g_err.clear();
  if (!index) return set_err(FM_ERR_INVALID_ARGUMENT, "index is null");
  if (check_mode(index, mode) != FM_OK) return FM_ERR_INVALID_ARGUMENT;
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
                static_cast<cudaStream_t>(stream), mode);
}

fm_status fm_query_host_mode(const fm_index* cindex, int mode, const double* h_lonlat,
                             std::uint64_t n, std::int32_t* h_out, std::int64_t* h_hist) {
  return fm_query_host_counted(cindex, mode, h_lonlat, n, h_out, h_hist, nullptr);
}

fm_status fm_query_host_counted(const fm_index* cindex, int mode, const double* h_lonlat,
                                std::uint64_t n, std::int32_t* h_out, std::int64_t* h_hist,
                                fm_query_counters* h_counters) {
  return query_host_impl(cindex, mode, h_lonlat, n, h_out, h_hist, nullptr, h_counters);
}

}  // extern "C"

// The host-buffer pipeline behind fm_query_host*: 8M-point chunks over
// kStreams streams (H2D copy, fm_query, D2H copy).  The histogram goes to
// the HOST array h_hist (accumulated into), or -- for the multi-GPU entry
// (multi.cu) -- stays on the device in d_hist_accum (n_polys int64 on the
// index's device, accumulated into), so it can be reduced over NCCL there.
__attribute__((visibility("hidden"))) fm_status query_host_impl(
    const fm_index* cindex, int mode, const double* h_lonlat, std::uint64_t n, std::int32_t* h_out,
    std::int64_t* h_hist, std::int64_t* d_hist_accum, fm_query_counters* h_counters) {
  g_err.clear();
  if (!cindex) return set_err(FM_ERR_INVALID_ARGUMENT, "index is null");
  if (check_mode(cindex, mode) != FM_OK) return FM_ERR_INVALID_ARGUMENT;
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
  unsigned long long* dh = reinterpret_cast<unsigned long long*>(d_hist_accum);
  if (h_hist && !dh) {
    if (!index->d_hist) FM_CUDA(cudaMalloc(&index->d_hist, std::max<std::uint64_t>(1, index->stats.n_polys) * 8));
    dh = index->d_hist;
    FM_CUDA(cudaMemsetAsync(dh, 0, std::max<std::uint64_t>(1, index->stats.n_polys) * 8, index->streams[0]));
    FM_CUDA(cudaStreamSynchronize(index->streams[0]));
  }
  unsigned long long* dc = nullptr;  // work counters: one set per stream
  if (h_counters) {
    if (!index->d_counters) FM_CUDA(cudaMalloc(&index->d_counters, kStreams * 4 * 8));
    dc = index->d_counters;
    FM_CUDA(cudaMemsetAsync(dc, 0, kStreams * 4 * 8, index->streams[0]));
    FM_CUDA(cudaStreamSynchronize(index->streams[0]));
  }
  const std::uint64_t n_chunks = (n + kChunkPoints - 1) / kChunkPoints;
  for (std::uint64_t c = 0; c < n_chunks; ++c) {
    const int s = static_cast<int>(c % kStreams);
    const std::uint64_t off = c * kChunkPoints;
    const std::uint64_t m = std::min(kChunkPoints, n - off);
    FM_CUDA(cudaMemcpyAsync(index->d_in[s], h_lonlat + 2 * off, m * 16, cudaMemcpyHostToDevice,
                            index->streams[s]));
    const fm_status st = launch(index, index->d_in[s], m, index->d_out[s], dh,
                                dc ? dc + 4 * s : nullptr, index->streams[s], mode);
    if (st != FM_OK) return st;
    FM_CUDA(cudaMemcpyAsync(h_out + off, index->d_out[s], m * 4, cudaMemcpyDeviceToHost,
                            index->streams[s]));
  }
  for (int s = 0; s < kStreams; ++s) FM_CUDA(cudaStreamSynchronize(index->streams[s]));
  if (h_hist && !d_hist_accum) {
    std::vector<std::int64_t> tmp(index->stats.n_polys);
    FM_CUDA(cudaMemcpy(tmp.data(), dh, index->stats.n_polys * 8, cudaMemcpyDeviceToHost));
    for (std::uint64_t k = 0; k < index->stats.n_polys; ++k) h_hist[k] += tmp[k];
  }
  if (h_counters) {
    unsigned long long v[kStreams * 4];
    FM_CUDA(cudaMemcpy(v, dc, sizeof(v), cudaMemcpyDeviceToHost));
    for (int s = 0; s < kStreams; ++s) {
      h_counters->points += v[4 * s];
      h_counters->boundary_points += v[4 * s + 1];
      h_counters->candidate_tests += v[4 * s + 2];
      h_counters->edge_tests += v[4 * s + 3];
    }
  }
  return FM_OK;
}

extern "C" {

// ---------------------------------------------------------------------------
// Index persistence (the FMCI save/load analogue, cell_index.hpp:641-726):
// "FMGI", u32 version, u32 sizeof(fm_index_stats), the stats, the grid
// geometry, n_phase1_slots, then grid / slot arena / overflow arena, each
// u64 length-prefixed.  Little endian (the only target).  The query-side
// layout (fold, approx cover) is rebuilt on load.
namespace {
constexpr char kIndexMagic[4] = {'F', 'M', 'G', 'I'};
constexpr std::uint32_t kIndexVersion = 1;

bool write_all(std::FILE* f, const void* p, std::uint64_t n) {
  return n == 0 || std::fwrite(p, 1, n, f) == n;
}
bool read_all(std::FILE* f, void* p, std::uint64_t n) {
  return n == 0 || std::fread(p, 1, n, f) == n;
}
}  // namespace

fm_status fm_index_save(const fm_index* index, const char* path) {
  g_err.clear();
  if (!index || !path) return set_err(FM_ERR_INVALID_ARGUMENT, "null argument");
  std::vector<std::uint32_t> grid;
  std::vector<std::uint8_t> slots, ovf;
  const std::uint32_t* gp;
  const std::uint8_t *sp, *op;
  if (index->device < 0) {
    gp = index->host.grid.data();
    sp = index->host.slots.data();
    op = index->host.overflow.data();
  } else {
    DeviceGuard guard(index->device);
    grid.resize(index->grid_len);
    slots.resize(index->slots_len);
    ovf.resize(index->overflow_len);
    FM_CUDA(cudaMemcpy(grid.data(), index->d_grid, index->grid_len * 4, cudaMemcpyDeviceToHost));
    FM_CUDA(cudaMemcpy(slots.data(), index->d_slots, index->slots_len, cudaMemcpyDeviceToHost));
    FM_CUDA(cudaMemcpy(ovf.data(), index->d_overflow, index->overflow_len, cudaMemcpyDeviceToHost));
    gp = grid.data();
    sp = slots.data();
    op = ovf.data();
  }
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return set_err(FM_ERR_RUNTIME, std::string("cannot open for writing: ") + path);
  const std::uint32_t ver = kIndexVersion, ssz = sizeof(fm_index_stats);
  const fm::GridGeom& g = index->g;
  const double geo[9] = {g.gx0, g.gx1, g.gy0, g.gy1, g.w, g.h, g.inv_w, g.inv_h, g.margin};
  const std::int64_t dims[2] = {g.nx, g.ny};
  const std::uint64_t counts[5] = {index->host.n_slots, index->host.n_phase1_slots,
                                   index->grid_len, index->slots_len, index->overflow_len};
  bool ok = write_all(f, kIndexMagic, 4) && write_all(f, &ver, 4) && write_all(f, &ssz, 4) &&
            write_all(f, &index->stats, ssz) && write_all(f, geo, sizeof(geo)) &&
            write_all(f, dims, sizeof(dims)) && write_all(f, counts, sizeof(counts)) &&
            write_all(f, gp, index->grid_len * 4) && write_all(f, sp, index->slots_len) &&
            write_all(f, op, index->overflow_len);
  ok = (std::fclose(f) == 0) && ok;
  if (!ok) return set_err(FM_ERR_RUNTIME, std::string("write failed: ") + path);
  return FM_OK;
}

fm_status fm_index_load(const char* path, int device, fm_index** out_index) {
  g_err.clear();
  if (!path || !out_index) return set_err(FM_ERR_INVALID_ARGUMENT, "null argument");
  *out_index = nullptr;
  if (device >= 0) {
    const fm_status st = check_device(device);
    if (st != FM_OK) return st;
  }
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return set_err(FM_ERR_RUNTIME, std::string("cannot open for reading: ") + path);
  auto fail = [&](const std::string& msg) {
    std::fclose(f);
    return set_err(FM_ERR_RUNTIME, msg + ": " + path);
  };
  char magic[4];
  std::uint32_t ver = 0, ssz = 0;
  if (!read_all(f, magic, 4) || std::memcmp(magic, kIndexMagic, 4) != 0) {
    return fail("not an index file (bad magic)");
  }
  if (!read_all(f, &ver, 4) || ver != kIndexVersion) return fail("unsupported index file version");
  if (!read_all(f, &ssz, 4) || ssz != sizeof(fm_index_stats)) return fail("index file stats layout differs");
  fm_index* ix = new (std::nothrow) fm_index();
  if (!ix) {
    std::fclose(f);
    return set_err(FM_ERR_OOM, "host allocation failed");
  }
  double geo[9];
  std::int64_t dims[2];
  std::uint64_t counts[5];
  if (!read_all(f, &ix->stats, ssz) || !read_all(f, geo, sizeof(geo)) ||
      !read_all(f, dims, sizeof(dims)) || !read_all(f, counts, sizeof(counts))) {
    delete ix;
    return fail("truncated index file");
  }
  fm::GridGeom& g = ix->g;
  g.gx0 = geo[0];
  g.gx1 = geo[1];
  g.gy0 = geo[2];
  g.gy1 = geo[3];
  g.w = geo[4];
  g.h = geo[5];
  g.inv_w = geo[6];
  g.inv_h = geo[7];
  g.margin = geo[8];
  g.nx = dims[0];
  g.ny = dims[1];
  ix->host.g = g;
  ix->host.n_slots = counts[0];
  ix->host.n_phase1_slots = counts[1];
  ix->grid_len = counts[2];
  ix->slots_len = counts[3];
  ix->overflow_len = counts[4];
  if (g.nx <= 0 || g.ny <= 0 || ix->grid_len != static_cast<std::uint64_t>(g.nx * g.ny) ||
      ix->slots_len < ix->host.n_slots * fm::kSlotBytes || ix->overflow_len < 512) {
    delete ix;
    return fail("corrupt index file header");
  }
  try {
    ix->host.grid.resize(ix->grid_len);
    ix->host.slots.resize(ix->slots_len);
    ix->host.overflow.resize(ix->overflow_len);
  } catch (const std::bad_alloc&) {
    delete ix;
    std::fclose(f);
    return set_err(FM_ERR_OOM, "host allocation failed while loading the index");
  }
  if (!read_all(f, ix->host.grid.data(), ix->grid_len * 4) ||
      !read_all(f, ix->host.slots.data(), ix->slots_len) ||
      !read_all(f, ix->host.overflow.data(), ix->overflow_len)) {
    delete ix;
    return fail("truncated index file");
  }
  std::fclose(f);
  ix->device = device;
  ix->ax0 = std::max(g.gx0, -180.0);
  ix->ax1 = std::min(g.gx1, 180.0);
  ix->ay0 = std::max(g.gy0, -90.0);
  ix->ay1 = std::min(g.gy1, 90.0);
  const double eps = ix->stats.approx_epsilon;
  // the grid itself tells whether the approx cover fits (cells within epsilon)
  ix->host.stats.approx_served_exact =
      eps > 0.0 && !(std::hypot(ix->g.w + 2.0 * ix->g.margin, ix->g.h + 2.0 * ix->g.margin) <= eps);
  ix->stats.query_grid_bytes = 0;
  ix->stats.query_block_log2 = 0;
  ix->stats.approx_grid_bytes = 0;
  ix->stats.approx_block_log2 = 0;
  if (device >= 0) {
    DeviceGuard guard(device);
    cudaError_t e1 = cudaMalloc(&ix->d_grid, ix->grid_len * 4);
    cudaError_t e2 = cudaMalloc(&ix->d_slots, ix->slots_len);
    cudaError_t e3 = cudaMalloc(&ix->d_overflow, ix->overflow_len);
    if (e1 == cudaSuccess && e2 == cudaSuccess && e3 == cudaSuccess) {
      e1 = cudaMemcpy(ix->d_grid, ix->host.grid.data(), ix->grid_len * 4, cudaMemcpyHostToDevice);
      e2 = cudaMemcpy(ix->d_slots, ix->host.slots.data(), ix->slots_len, cudaMemcpyHostToDevice);
      e3 = cudaMemcpy(ix->d_overflow, ix->host.overflow.data(), ix->overflow_len, cudaMemcpyHostToDevice);
    }
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      free_device(ix);
      delete ix;
      return set_err(FM_ERR_CUDA, "index upload failed");
    }
    std::vector<std::uint32_t>().swap(ix->host.grid);
    std::vector<std::uint8_t>().swap(ix->host.slots);
    std::vector<std::uint8_t>().swap(ix->host.overflow);
    const fm_status st = finish_device(ix, eps);
    if (st != FM_OK) {
      free_device(ix);
      delete ix;
      return st;
    }
  }
  *out_index = ix;
  return FM_OK;
}

fm_status fm_index_set_query_path(fm_index* index, int path, double tile_bytes) {
  g_err.clear();
  if (!index) return set_err(FM_ERR_INVALID_ARGUMENT, "index is null");
  if (path != FM_PATH_AUTO && path != FM_PATH_STREAM && path != FM_PATH_BINNED) {
    return set_err(FM_ERR_INVALID_ARGUMENT, "unknown query path");
  }
  if (!(tile_bytes >= 0.0) || std::isinf(tile_bytes)) {
    return set_err(FM_ERR_INVALID_ARGUMENT, "tile_bytes must be finite and >= 0");
  }
  index->query_path = path;
  index->tile_bytes = tile_bytes;
  if (index->device >= 0) index->tiles = plan_tiles(index->g, index->stats, tile_bytes > 0 ? tile_bytes : kTileBytes);
  return FM_OK;
}

fm_status fm_index_query_plan(const fm_index* index, std::uint64_t n, int* path, std::int32_t* tile_log2,
                              std::int32_t* n_tiles) {
  g_err.clear();
  if (!index) return set_err(FM_ERR_INVALID_ARGUMENT, "index is null");
  if (path) *path = use_binned(index, n) ? FM_PATH_BINNED : FM_PATH_STREAM;
  if (tile_log2) *tile_log2 = index->tiles.ts;
  if (n_tiles) *n_tiles = index->tiles.n_tiles;
  return FM_OK;
}

fm_status fm_index_export(const fm_index* index, std::uint32_t* grid, std::uint64_t* grid_len,
                          std::uint8_t* arena, std::uint64_t* arena_len, double* geometry16) {
  if (!index || !grid_len || !arena_len) return set_err(FM_ERR_INVALID_ARGUMENT, "null argument");
  *grid_len = index->grid_len;
  *arena_len = index->slots_len + index->overflow_len;
  if (geometry16) {
    const fm::GridGeom& g = index->g;
    const double v[16] = {g.gx0, g.gx1, g.gy0, g.gy1, g.w, g.h, g.inv_w, g.inv_h,
                          static_cast<double>(g.nx), static_cast<double>(g.ny), g.margin,
                          static_cast<double>(index->stats.n_polys),
                          static_cast<double>(index->slots_len), 0.0, 0.0, 0.0};
    std::memcpy(geometry16, v, sizeof(v));
  }
  if (!grid && !arena) return FM_OK;
  if (index->device < 0) {
    if (grid) std::memcpy(grid, index->host.grid.data(), index->grid_len * 4);
    if (arena) {
      std::memcpy(arena, index->host.slots.data(), index->slots_len);
      std::memcpy(arena + index->slots_len, index->host.overflow.data(), index->overflow_len);
    }
    return FM_OK;
  }
  DeviceGuard guard(index->device);
  if (grid) FM_CUDA(cudaMemcpy(grid, index->d_grid, index->grid_len * 4, cudaMemcpyDeviceToHost));
  if (arena) {
    FM_CUDA(cudaMemcpy(arena, index->d_slots, index->slots_len, cudaMemcpyDeviceToHost));
    FM_CUDA(cudaMemcpy(arena + index->slots_len, index->d_overflow, index->overflow_len,
                       cudaMemcpyDeviceToHost));
  }
  return FM_OK;
}

}  // extern "C"
