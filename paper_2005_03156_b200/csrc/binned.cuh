// binned.cuh -- the tile-binned query path (north star item 2, "point
// binning"), included by fastmap_b200.cu inside its anonymous namespace
// (it reuses QItem, eval_staged and emit from there).
//
// The reference sorts its pending (leaf, point) pairs and walks them leaf
// by leaf (cell_index.hpp:546-588, std::sort at :567) so each polygon's
// edges are touched once per batch.  Here the analogue is a one-pass
// partition of the point stream by coarse *tile* of the cell grid (a
// 2^ts x 2^ts block of cells whose grid entries and slots total a few tens
// of MB), so that the query pass walks the index tile by tile and every
// grid sector and boundary slot is fetched from HBM about once per tile
// instead of once per point.  It pays off when the index is far larger
// than L2 and most points land in boundary cells (c3, c4); the stream path
// (stream_kernel + resolve_kernel) stays the choice for small or mostly
// true-hit indexes (c1, c2) -- see use_binned() in fastmap_b200.cu.  An
// index this path takes keeps a flat query grid (finish_device): a tile's
// entries are L2-resident while the tile is walked.
//
// Per batch of n <= 2^30 points:
//   bin_sample_kernel   one point in 64 (four consecutive ones per 256-point
//                       stratum): sampled bin counts
//   bin_plan_kernel     bin capacities (estimate + 3 sigma + pad), their
//                       scan as bin starts, the overflow bin after them
//   bin_scatter_kernel  a chunk of 4K points at a time, copied into shared
//                       memory by cp.async: a counting sort by tile, one
//                       global atomic per non-empty bin claims the run's
//                       space, runs written whole (pts_b); per point its
//                       sorted index inside the chunk (pos16, 2 bytes), per
//                       chunk the table of its runs
//   bin_seal_kernel     unused bin tails become NaN points; the binned length
//   binned_query_kernel the query over pts_b in order: locate, true hits
//                       answered at once, boundary points through
//                       warp-private shared-memory rings (full, half and
//                       double slots apart) whose batches of 32 slots are
//                       staged by cp.async one batch ahead of their
//                       evaluation; answers to res[k]
//   unbin_kernel        out[i] = res[binned position of i], read run by run
//                       (coalesced) through the chunk's run table
//   unplaced_kernel     points no bin could take (returns at once normally)
// Iterations are walked with a grid stride, so at any moment the grid reads
// one window of the stream and every tile's points stay in about input
// order: the scattered writes and the gather in unbin_kernel stay coherent
// in L2 and the TLB.
// Points outside the grid (and NaN) are clamped into the border tiles; the
// query pass answers them -1 by its own acceptance test, like every path.
//
// Only performance depends on the binning: every point is answered by the
// same locate_n and the same slot algebra (edge_bit, eval_leaf_slot,
// eval_double_slot; eval_half_leaf is eval_leaf_slot over a half slot's 64
// bytes) as the stream path, so the answers are identical whatever tile or
// order a point ends up in.

#ifndef FM_QMINB
#define FM_QMINB 2
#endif

constexpr int kMaxTiles = 2048;                         // keys < kMaxTiles + 1

// Work counters (zeroed per launch): the ordered passes hand out their
// units -- scatter chunks, query tile groups, gather blocks -- in increasing
// order from an atomic counter instead of a static grid stride, so the
// units in flight at any moment are a compact window of the stream.  (With a
// grid stride the persistent warps drift apart over thousands of
// iterations and the window, and with it the L2 working set, spreads over
// the whole array.)
enum { kCtrQuery = 1, kCtrUnbin = 2, kCtrCount = 4 };

__device__ __forceinline__ unsigned long long cta_grab(unsigned long long* ctr, unsigned long long* s_slot) {
  __syncthreads();
  if (threadIdx.x == 0) *s_slot = atomicAdd(ctr, 1ull);
  __syncthreads();
  return *s_slot;
}

struct TileGeom {
  int ts = 0;        // log2 tile side in cells
  int tnx = 1, tny = 1;
  int n_tiles = 1;   // tnx * tny (bin n_tiles stays empty: points outside the grid are clamped into border tiles)
};

// The tile of a point, straight from the tile's inverse width: only locality
// depends on the binning (the query locates every point exactly by itself),
// so a point within rounding of a tile border may land in the neighbouring
// tile, and points outside the grid (and NaN, which converts to 0) are
// clamped into the border tiles.
struct TileKey {
  double gx0, gy0, inv_tw, inv_th;
  int tnx, tny;
};
__device__ __forceinline__ TileKey tile_key_params(const fm::KParams& P, const TileGeom& T) {
  TileKey K;
  K.gx0 = P.gx0;
  K.gy0 = P.gy0;
  const double scale = __longlong_as_double(static_cast<long long>(1023 - T.ts) << 52);  // 2^-ts, exactly
  K.inv_tw = __dmul_rn(P.inv_w, scale);
  K.inv_th = __dmul_rn(P.inv_h, scale);
  K.tnx = T.tnx;
  K.tny = T.tny;
  return K;
}
__device__ __forceinline__ int tile_key(const TileKey& K, double px, double py) {
  int tx = static_cast<int>(__dmul_rn(__dsub_rn(px, K.gx0), K.inv_tw));
  int ty = static_cast<int>(__dmul_rn(__dsub_rn(py, K.gy0), K.inv_th));
  tx = min(max(tx, 0), K.tnx - 1);
  ty = min(max(ty, 0), K.tny - 1);
  return ty * K.tnx + tx;
}

constexpr int kSampleThreads = 256;

// ---- single-pass binning with sampled bin capacities ----------------------
// Sizing the bins exactly takes a counting pass over the whole stream (16
// B/point: 2.8 ms per 1B c3 points, round 2's first cut).  Instead, one point in
// kSampleStride (kSampleGroup consecutive points at a hashed place of every
// stratum of kSampleStride * kSampleGroup; a spatially correlated stream
// just sees a noisier estimate and uses more of the overflow bin) is counted,
// every bin gets the sampled estimate plus a kSigmas margin plus kBinPad,
// and the scatter claims bin space with one global atomic per (iteration,
// bin).  Points past their bin's capacity go to an overflow bin at the end
// of the binned array; points past *that* (an adversarial stream whose
// sample missed them) get pos = kUnplaced and unplaced_kernel answers them
// straight from the index.  Only performance depends on the estimate: every
// point is answered by the same code wherever it lands.
constexpr int kSampleStride = 64;
constexpr int kSampleGroup = 4;
constexpr unsigned int kBinPad = 256;
// bin margin in standard deviations of the sampled estimate: every unused
// slot is a NaN point the query still reads, every overflowing point loses
// its tile's locality
constexpr double kSigmas = 3.0;
constexpr unsigned int kUnplaced = 0xFFFFFFFFu;

// The bin table in the batch's scratch: per bin start, capacity, fill
// cursor; then the overflow bin and the binned length the query walks.
struct BinTable {
  unsigned int* start;
  unsigned int* cap;
  unsigned int* cur;
  unsigned int* hdr;  // [0] overflow start, [1] overflow capacity, [2] overflow fill
  unsigned long long* n_eff;  // points the query walks: overflow start + fill
};

__device__ __forceinline__ std::uint32_t stratum_hash(std::uint64_t j) {
  std::uint64_t z = j * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 31)) * 0xBF58476D1CE4E5B9ull;
  return static_cast<std::uint32_t>(z >> 40);
}

__global__ void __launch_bounds__(kSampleThreads)
    bin_sample_kernel(fm::KParams P, TileGeom T, const double2* __restrict__ pts, std::uint64_t n,
                      unsigned int* __restrict__ counts) {
  extern __shared__ unsigned int s_hist[];
  const TileKey K = tile_key_params(P, T);
  const int nk = T.n_tiles + 1;
  for (int k = threadIdx.x; k < nk; k += blockDim.x) s_hist[k] = 0u;
  __syncthreads();
  // kSampleGroup consecutive points (one 64-byte DRAM burst) at a hashed
  // place of every stratum of kSampleStride * kSampleGroup points: the same
  // sampling rate as one point per kSampleStride, a quarter of the bursts
  // (consecutive points of a stream are independent draws)
  constexpr std::uint64_t kSpan = static_cast<std::uint64_t>(kSampleStride) * kSampleGroup;
  const std::uint64_t strata = (n + kSpan - 1) / kSpan;
  for (std::uint64_t j = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < strata;
       j += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
    const std::uint64_t lo = j * kSpan;
    const std::uint64_t groups = (min(kSpan, n - lo) + kSampleGroup - 1) / kSampleGroup;
    const std::uint64_t g0 = lo + (stratum_hash(j) % groups) * kSampleGroup;
#pragma unroll
    for (int c = 0; c < kSampleGroup; ++c) {
      if (g0 + c < n) {
        const double2 p = __ldg(pts + g0 + c);
        atomicAdd(s_hist + tile_key(K, p.x, p.y), 1u);
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nk; k += blockDim.x) {
    if (s_hist[k]) atomicAdd(counts + k, s_hist[k]);
  }
}

// Upper bound of the planned bins' total capacity (host side, sizes the
// scratch): sum est <= n + S, and by Cauchy-Schwarz the margins sum to at
// most kSigmas sqrt(nk * sum(S est + S^2)).
std::uint64_t bin_capacity_bound(std::uint64_t n, int nk) {
  const double S = kSampleStride, K = nk, N = static_cast<double>(n) + S;
  const double margin = kSigmas * std::sqrt(K * (S * N + K * S * S));
  return static_cast<std::uint64_t>(N + margin) + static_cast<std::uint64_t>(nk) * (kBinPad + 8);  // + fp32 rounding of the margins
}
std::uint64_t bin_overflow_cap(std::uint64_t n) { return std::min<std::uint64_t>(n, n / 32 + 65536); }

// One CTA: capacities from the sampled counts, their exclusive scan as bin
// starts, cursors zeroed, the overflow bin after the last bin.
constexpr int kPlanThreads = 1024;
__global__ void __launch_bounds__(kPlanThreads)
    bin_plan_kernel(int nk, std::uint64_t ovf_cap, const unsigned int* __restrict__ counts, BinTable B) {
  constexpr int kPer = (kMaxTiles + 1 + kPlanThreads - 1) / kPlanThreads;
  __shared__ unsigned long long s_warp[kPlanThreads / 32];
  const int k0 = threadIdx.x * kPer;
  unsigned long long c[kPer], sum = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    c[q] = 0;
    if (k0 + q < nk) {
      // the margin in fp32 (a size, not a predicate: no fp64 FMA in the library
      // outside the builder's division, tests/test_sass.py)
      const unsigned long long est = static_cast<unsigned long long>(counts[k0 + q]) * kSampleStride;
      const float var = static_cast<float>(kSampleStride) * static_cast<float>(est + kSampleStride);
      c[q] = est + static_cast<unsigned long long>(static_cast<float>(kSigmas) * sqrtf(var)) + 1 + kBinPad;
    }
    sum += c[q];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += x;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long w = s_warp[lane];
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long x = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += x;
    }
    s_warp[lane] = wi - w;
  }
  __syncthreads();
  unsigned long long run = s_warp[warp] + incl - sum;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    if (k0 + q < nk) {
      B.start[k0 + q] = static_cast<unsigned int>(run);
      B.cap[k0 + q] = static_cast<unsigned int>(c[q]);
      B.cur[k0 + q] = 0u;
    }
    run += c[q];
  }
  if (k0 < nk && nk <= k0 + kPer) {  // the thread holding the last bin
    B.hdr[0] = static_cast<unsigned int>(run);
    B.hdr[1] = static_cast<unsigned int>(ovf_cap);
    B.hdr[2] = 0u;
  }
}

// ---- the scatter and its gather ---------------------------------------------
// Two CTAs of 512 threads per SM each stream chunks of kChunk points through
// a shared-memory window filled by cp.async (while one CTA waits for its
// window the other sorts or writes), so no point lives in a register:
//   raw[kChunk]     the chunk's points as loaded (16 B each)
//   perm[k]         source index of the point at sorted position k
//   sdst[k]         its binned position
// The chunk is counting-sorted by tile key; the runs are then written
// whole, pts_b[sdst[k]] = raw[perm[k]] for consecutive k.  Round 2's first
// scatter held the points in registers (127 registers, 16 warps per SM):
// 10.1 ms per 1B c3 points against 8.1 ms (profiles/r2al, r2am); a
// double-buffered window with one 1024-thread CTA per SM measured 9.4 ms.
// (A placement pass specialised for chunks without overflow cut the
// kernel's instructions by a quarter but measured 7.9 against 7.4 ms, with
// 76 GB instead of 55 GB of L2 traffic: profiles/r2bl, r2bm.)
// Instead of a 4-byte binned position per point, the scatter leaves
//   pos16[i]        the point's sorted index k inside its chunk (2 B), and
//   tab[c][key]     {binned position of the run's first point,
//                    first sorted index | points that fit the bin << 16}
//                   (+ the run's overflow-bin offset, read only for runs
//                   that did not fit),
// and unbin_kernel turns the per-point gather res[pos[i]] -- one L2 sector
// per point, bound by the L2 gather rate (4.3 ms per 1B points) -- into
// coalesced reads of res in sorted order (3.4 ms).  (Eight consecutive points
// per thread -- one 16-byte index load, two 16-byte id stores -- measured
// 3.9 ms: profiles/r2au.)
#ifndef FM_SC2_THREADS
#define FM_SC2_THREADS 512
#endif
#ifndef FM_SC2_PER
#define FM_SC2_PER 8
#endif
#ifndef FM_SC2_BUFS
#define FM_SC2_BUFS 1  // 2: a double-buffered window, one CTA per SM (r2am: 9.4 vs 8.1 ms); 1: 1: one window per CTA (two CTAs per SM overlap instead)
#endif
#ifndef FM_SC2_MINB
#define FM_SC2_MINB 2
#endif
constexpr int kSc2Threads = FM_SC2_THREADS;
constexpr int kSc2Per = FM_SC2_PER;
constexpr int kChunk = kSc2Threads * kSc2Per;  // points per chunk
static_assert(kChunk <= 32768, "sorted indices and counts are 16-bit fields");
constexpr int kUnplacedId = INT_MIN;  // out[i] of a point no bin could take, until unplaced_kernel

// Words per chunk of the run table: nk4 x {dst, off | av << 16}, nk4 x overflow offset.
__host__ __device__ inline std::uint64_t tab_stride(int nk4) { return 3ull * static_cast<std::uint64_t>(nk4); }
inline int sc2_smem(int nk4) { return kChunk * (16 + 4 + 2) + 5 * nk4 * 4; }

__global__ void __launch_bounds__(kSc2Threads, FM_SC2_MINB)
    bin_scatter_kernel(fm::KParams P, TileGeom T, const double2* __restrict__ pts, std::uint64_t n,
                        BinTable B, double2* __restrict__ pts_b, std::uint16_t* __restrict__ pos16,
                        unsigned int* __restrict__ tab) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nk = T.n_tiles + 1;
  const int nk4 = (nk + 3) & ~3;
  double2* raw = reinterpret_cast<double2*>(smem_raw);
  unsigned int* sdst = reinterpret_cast<unsigned int*>(smem_raw + kChunk * 16);
  unsigned int* s_cnt = sdst + kChunk;
  unsigned int* s_off = s_cnt + nk4;
  unsigned int* s_dst = s_off + nk4;  // destination of the run's first point
  unsigned int* s_av = s_dst + nk4;   // points of the run that fit the bin
  unsigned int* s_ob = s_av + nk4;    // overflow destination of the rest
  std::uint16_t* perm = reinterpret_cast<std::uint16_t*>(s_ob + nk4);
  __shared__ unsigned int s_part[64];
  const TileKey K = tile_key_params(P, T);
  constexpr int kScanPer = (kMaxTiles + 1 + kSc2Threads - 1) / kSc2Threads;
  const unsigned int ovf_base = B.hdr[0], ovf_cap = B.hdr[1];
  const std::uint64_t n_it = (n + kChunk - 1) / kChunk;
  const std::uint64_t stride = tab_stride(nk4);
  const int tid = threadIdx.x;
  auto prefetch = [&](std::uint64_t it) {
    if (it < n_it) {
      const std::uint64_t base = it * kChunk;
      const int left = static_cast<int>(min(static_cast<std::uint64_t>(kChunk), n - base));
      const double2* src = pts + base + tid;
      double2* dst = raw + tid;
#pragma unroll
      for (int j = 0; j < kSc2Per; ++j) {
        if (j * kSc2Threads + tid < left) cp_async16(dst + j * kSc2Threads, src + j * kSc2Threads);
      }
    }
    cp_async_commit();
  };
  for (int k = tid; k < nk; k += kSc2Threads) s_cnt[k] = 0u;
  prefetch(blockIdx.x);
  for (std::uint64_t it = blockIdx.x; it < n_it; it += gridDim.x) {
    const std::uint64_t base = it * kChunk;
    const std::uint64_t hi = min(n, base + kChunk);
    const int cnt = static_cast<int>(hi - base);
    cp_async_wait0();
    __syncthreads();  // the window landed, s_cnt zeroed
    const bool full = cnt == kChunk;  // every chunk but the stream's last: no per-point bounds tests
    unsigned int kr[kSc2Per];
    if (full) {
#pragma unroll
      for (int j = 0; j < kSc2Per; ++j) {
        const double2 p = raw[j * kSc2Threads + tid];
        const unsigned int key = static_cast<unsigned int>(tile_key(K, p.x, p.y));
        kr[j] = (key << 16) | atomicAdd(s_cnt + key, 1u);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kSc2Per; ++j) {
        const int q = j * kSc2Threads + tid;
        kr[j] = 0xFFFFFFFFu;
        if (q < cnt) {
          const double2 p = raw[q];
          const unsigned int key = static_cast<unsigned int>(tile_key(K, p.x, p.y));
          kr[j] = (key << 16) | atomicAdd(s_cnt + key, 1u);
        }
      }
    }
    __syncthreads();
    {  // exclusive scan of s_cnt -> s_off
      const int k0 = tid * kScanPer;
      unsigned int v[kScanPer], sum = 0;
#pragma unroll
      for (int q = 0; q < kScanPer; ++q) {
        v[q] = k0 + q < nk ? s_cnt[k0 + q] : 0u;
        sum += v[q];
      }
      const int lane = tid & 31, warp = tid >> 5;
      unsigned int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane == 31) s_part[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const unsigned int w = lane < kSc2Threads / 32 ? s_part[lane] : 0u;
        unsigned int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int x = __shfl_up_sync(0xFFFFFFFFu, wi, o);
          if (lane >= o) wi += x;
        }
        if (lane < kSc2Threads / 32) s_part[32 + lane] = wi - w;
      }
      __syncthreads();
      unsigned int run = s_part[32 + warp] + incl - sum;
#pragma unroll
      for (int q = 0; q < kScanPer; ++q) {
        if (k0 + q < nk) s_off[k0 + q] = run;
        run += v[q];
      }
    }
    __syncthreads();
    // the claims (one bin per thread, so the atomics' round trips overlap) and the chunk's run table
    unsigned int* tb = tab + it * stride;
    for (int k = tid; k < nk; k += kSc2Threads) {
      const unsigned int v = s_cnt[k];
      unsigned int dst = 0u, av = 0u;
      if (v) {
        const unsigned int got = atomicAdd(B.cur + k, v);
        const unsigned int cap = __ldg(B.cap + k);
        av = got < cap ? min(cap - got, v) : 0u;
        dst = __ldg(B.start + k) + got;
        s_dst[k] = dst;
        s_av[k] = av;
        if (av < v) {
          const unsigned int ob = atomicAdd(B.hdr + 2, v - av);
          s_ob[k] = ob;
          tb[2 * nk4 + k] = ob;
        }
      }
      reinterpret_cast<uint2*>(tb)[k] = make_uint2(dst, s_off[k] | (av << 16));
    }
    __syncthreads();
    {
#pragma unroll
      for (int j = 0; j < kSc2Per; ++j) {
        const int q = j * kSc2Threads + tid;
        if (q < cnt) {
          const unsigned int key = kr[j] >> 16, r = kr[j] & 0xFFFFu;
          const unsigned int k = s_off[key] + r, av = s_av[key];
          unsigned int dst;
          if (r < av) {
            dst = s_dst[key] + r;
          } else {
            const unsigned int o = s_ob[key] + (r - av);
            dst = o < ovf_cap ? ovf_base + o : kUnplaced;
          }
          perm[k] = static_cast<std::uint16_t>(q);
          sdst[k] = dst;
          __stcs(pos16 + base + q, static_cast<std::uint16_t>(k));
        }
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int k = tid; k < cnt; k += kSc2Threads) {
      const unsigned int d = sdst[k];
      if (d != kUnplaced) pts_b[d] = raw[perm[k]];  // run by run
    }
    for (int k = tid; k < nk; k += kSc2Threads) s_cnt[k] = 0u;
    __syncthreads();  // the window is free
    prefetch(it + gridDim.x);
  }
  cp_async_wait0();
}

// After the scatter: every bin's unfilled tail becomes NaN points (answered
// -1 and never read back), the query's length is the overflow bin's end,
// and the point counter forgets the padding.
__global__ void __launch_bounds__(256)
    bin_seal_kernel(int nk, BinTable B, double2* __restrict__ pts_b, unsigned long long* __restrict__ counters) {
  for (int k = blockIdx.x; k < nk; k += gridDim.x) {
    const unsigned int cap = B.cap[k], fill = min(B.cur[k], cap), s = B.start[k];
    for (unsigned int i = fill + threadIdx.x; i < cap; i += blockDim.x) pts_b[s + i] = make_double2(NAN, NAN);
    if (counters && threadIdx.x == 0 && cap > fill) atomicAdd(counters, 0ull - static_cast<unsigned long long>(cap - fill));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *B.n_eff = static_cast<unsigned long long>(B.hdr[0]) + min(B.hdr[2], B.hdr[1]);
  }
}

// The query over the binned stream.  Warps take consecutive 32*kU-point
// tiles with a grid stride, so at any moment the whole grid works on one
// window of the binned array -- one or two index tiles.  Boundary points
// wait in a warp-private ring (kQCap items).  Full batches of 32 are staged
// into one of two slot pools by cp.async and evaluated one round later, so
// the slot fetches of batch k+1 overlap the evaluation of batch k and the
// next point tile's loads and grid gathers; split cells put their child
// entry back into the ring.
// Points in half slots and in double slots (kDoubleBit; polygon corners)
// wait in rings of their own (below), so every batch is of one slot width
// and the leaf-slot batches never run the wider double-slot code.
#ifndef FM_QWARPS
#define FM_QWARPS 8
#endif
constexpr int kQWarps = FM_QWARPS;
constexpr int kQCap = 128;
constexpr int kDCap = 128;
#ifndef FM_QLD
#define FM_QLD __ldg  // the staged batch re-reads its points: ld.cs (evict-first) made those DRAM reads (r2ap: 49.9 vs 36.3 GB)
#endif
// Three rings of (binned index, entry) pairs: full leaf slots (and whatever
// a split cell descends to), half slots (kHalfBit: the content lies in the
// slot's first 64 bytes -- at most 2 candidates, 2 edges, 1 breakpoint; half
// of c3's boundary cells), double slots.  A batch is all of one kind, so a
// half batch runs half the copies, half the shared-memory reads and a
// 2-edge, 2-candidate evaluation.  The point itself is re-read from pts_b
// when its batch is staged (an L2 hit, one round before it is needed).
struct WarpSmemQ {
  alignas(16) std::uint8_t pool[2][32 * fm::kSlotBytes];
  std::uint32_t qk[kQCap], qe[kQCap];
  std::uint32_t hk[kQCap], he[kQCap];
  std::uint32_t dk[kDCap], de[kDCap];
};
constexpr int kSmemQ = static_cast<int>(sizeof(WarpSmemQ)) * kQWarps;

struct RingState {
  int head = 0, qn = 0;  // ring items not yet staged
  int pend = 0;          // items of the staged batch in pool[pb]
  int pb = 0;
  QItem pit;             // this lane's staged item
  int dhead = 0, dn = 0; // double-slot ring
  int hhead = 0, hn = 0; // half-slot ring
  int pkind = 0;         // kind of the staged batch: 0 full, 1 half, 2 double
};

// Slot staging of the binned query.  A batch's slots are copied by cp.async,
// 16 bytes per lane: 8 lanes per full slot (4 slots per instruction), 4 per
// half slot (8), 16 per double slot (2).  The copy's source is
// slots + 16 * (8 * index + chunk): the entry shifted left by 3 drops its
// flag bits, so one integer multiply-add and one wide multiply-add form the
// address; its destination is a per-lane constant plus 512 bytes per
// instruction.  (stage_slots, the stream path's copy, recomputed both per
// copy: about 14 instructions each, 17% of this kernel's instructions, most
// on the integer pipe that bounds it -- profiles/r2ax.)
__device__ __forceinline__ void cp_async16_s(unsigned saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem) : "memory");
}
__device__ __forceinline__ const std::uint8_t* chunk_ptr(const std::uint8_t* slots, std::uint32_t er, int c) {
  return slots + static_cast<std::size_t>(er * 8u + static_cast<std::uint32_t>(c)) * 16u;
}

// Full slots (128 bytes): chunk c of slot r at chunk c ^ (r & 7) of row r.
__device__ __forceinline__ void stage_full(const fm::KParams& P, std::uint8_t* buf, std::uint32_t e, int n,
                                           int lane) {
  const int c = lane & 7, j = lane >> 3;
  const std::uint8_t* slots = P.slots;
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(buf)) + j * 128;
  const unsigned d0 = b + 16 * (c ^ j), d1 = b + (16 * (c ^ j) ^ 64);  // r & 7 = 4 (q & 1) + j
  if (n == 32) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const std::uint32_t er = __shfl_sync(0xFFFFFFFFu, e, 4 * q + j);
      cp_async16_s(((q & 1) ? d1 : d0) + q * 512, chunk_ptr(slots, er, c));
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const std::uint32_t er = __shfl_sync(0xFFFFFFFFu, e, 4 * q + j);
      if (4 * q + j < n) cp_async16_s(((q & 1) ? d1 : d0) + q * 512, chunk_ptr(slots, er, c));
    }
  }
  cp_async_commit();
}

// Half slots (their first 64 bytes): chunk c of slot r at chunk
// c ^ ((r >> 1) & 3) of its 64-byte row, so the owner lanes' 16-byte reads
// are bank-conflict free.
__device__ __forceinline__ void stage_half(const fm::KParams& P, std::uint8_t* buf, std::uint32_t e, int n,
                                           int lane) {
  const int c = lane & 3, j = lane >> 2;
  const std::uint8_t* slots = P.slots;
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(buf)) + j * 64 + 16 * (c ^ ((j >> 1) & 3));
  if (n == 32) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const std::uint32_t er = __shfl_sync(0xFFFFFFFFu, e, 8 * q + j);
      cp_async16_s(d + q * 512, chunk_ptr(slots, er, c));
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const std::uint32_t er = __shfl_sync(0xFFFFFFFFu, e, 8 * q + j);
      if (8 * q + j < n) cp_async16_s(d + q * 512, chunk_ptr(slots, er, c));
    }
  }
  cp_async_commit();
}

// A half leaf slot (index_format.h: bytes 0..63 of kind 1 with <= 2
// candidates and <= 2 vertices + <= 1 breakpoint, or 3 vertices): one
// chain, at most two edges.
template <bool kCount>
__device__ __forceinline__ int eval_half_leaf(const uint4 (&c)[4], double px, double py, fm::WorkCount& wc) {
  const std::uint32_t h = c[0].x;
  const std::uint32_t nv = (h >> 8) & 0xFFu, nc = (h >> 16) & 0xFFu, nb = h >> 24;
  const double v0x = fm::as_f64(c[1].x, c[1].y), v0y = fm::as_f64(c[1].z, c[1].w);
  const double v1x = fm::as_f64(c[2].x, c[2].y), v1y = fm::as_f64(c[2].z, c[2].w);
  const double v2x = fm::as_f64(c[3].x, c[3].y), v2y = fm::as_f64(c[3].z, c[3].w);
  std::uint32_t m = 0;
  if (nv >= 2u) {
    if (kCount) wc.edges++;
    m |= fm::edge_bit(px, py, v0x, v0y, v1x, v1y);
  }
  if (nv >= 3u) {
    if (kCount) wc.edges++;
    m |= fm::edge_bit(px, py, v1x, v1y, v2x, v2y) << 1;
  }
  const std::uint32_t bm = (nv < 3u && nb > 0u && py > v2x) ? 1u : 0u;  // +48: break[0] when n_verts < 3
  const std::uint32_t w = c[0].y;  // edge_mask[0..1], info[0..1]
  int id = -1;
#pragma unroll
  for (int q = 1; q >= 0; --q) {  // descending, so the smallest odd candidate wins
    const std::uint32_t mk = (w >> (8 * q)) & 0xFFu, inf = (w >> (16 + 8 * q)) & 0xFFu;
    const std::uint32_t par = (inf >> 7) ^ __popc(m & mk) ^ __popc(bm & inf & 3u);
    if (static_cast<std::uint32_t>(q) < nc && (par & 1u)) id = static_cast<int>(q == 0 ? c[0].z : c[0].w);
  }
  if (kCount) wc.cands += nc;
  return id;
}

// Evaluate a staged half batch (leaf, split or overflow slots; all live in
// their first 64 bytes).  Returns like eval_staged.
template <bool kHist, bool kCount>
__device__ __forceinline__ std::uint32_t eval_staged_half(const fm::KParams& P, const std::uint8_t* buf,
                                                          const QItem& it, int n, int lane,
                                                          int* __restrict__ out, const HistSink& hist,
                                                          fm::WorkCount& wc) {
  std::uint32_t requeue = 0;
  if (lane < n) {
    const std::uint8_t* base = buf + lane * 64;
    const int s = (lane >> 1) & 3;
    uint4 c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = *reinterpret_cast<const uint4*>(base + 16 * (k ^ s));
    const std::uint32_t kind = c[0].x & 0xFFu;
    int id = -1;
    bool done = true;
    if (kind == fm::kSlotLeaf) {
      if (kCount) wc.boundary++;
      id = eval_half_leaf<kCount>(c, it.px, it.py, wc);
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
    } else {  // overflow record
      if (kCount) wc.boundary++;
      id = fm::resolve_overflow<kCount>(P, (static_cast<std::uint64_t>(c[0].w) << 32) | c[0].z, it.px,
                                        it.py, wc);
    }
    if (done) emit<kHist>(out, hist, it.i, id);
  }
  return requeue;
}

// Double slots (256 bytes) go through the same pools 16 at a time: 16 lanes
// per slot, 2 slots per instruction; chunk c of slot r is stored at chunk
// c ^ (r & 7) of its 256-byte row.  (Loading them straight from global
// memory, 16 uncoalesced 16-byte loads per lane, cost 16 L1 tag cycles per
// item against about 5 here; the kernel is bound by L1 throughput.)
constexpr int kDblBatch = 16;
__device__ __forceinline__ void stage_double(const fm::KParams& P, std::uint8_t* buf, std::uint32_t e, int n,
                                             int lane) {
  const int c = lane & 15, j = lane >> 4;
  const std::uint8_t* slots = P.slots;
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(buf)) + j * 256;
  const unsigned t = 16 * (c ^ j);  // r & 7 = (2 (q & 3)) ^ j
#pragma unroll
  for (int q = 0; q < kDblBatch / 2; ++q) {
    const std::uint32_t er = __shfl_sync(0xFFFFFFFFu, e, 2 * q + j);
    if (2 * q + j < n) cp_async16_s(b + (t ^ (32 * (q & 3))) + q * 512, chunk_ptr(slots, er, c));
  }
  cp_async_commit();
}

template <bool kHist, bool kCount>
__device__ __forceinline__ void eval_staged_double(const std::uint8_t* buf, const QItem& it, int n, int lane,
                                                   int* __restrict__ out, const HistSink& hist,
                                                   fm::WorkCount& wc) {
  if (lane < n) {
    const std::uint8_t* base = buf + lane * 256;
    const int s = lane & 7;
    uint4 a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = *reinterpret_cast<const uint4*>(base + 16 * (k ^ s));
#pragma unroll
    for (int k = 0; k < 8; ++k) b[k] = *reinterpret_cast<const uint4*>(base + 128 + 16 * (k ^ s));
    if (kCount) wc.boundary++;
    emit<kHist>(out, hist, it.i, fm::eval_double_slot<kCount>(a, b, it.px, it.py, wc));
  }
}

// Stage the next batch -- a full-slot batch when 32 such items wait, else a
// half-slot batch (any when draining) -- and evaluate the previously staged
// one; repeat while whole batches remain.  Split cells put their child
// entry into the full ring, whose evaluation takes every slot kind.
template <bool kHist, bool kCount>
__device__ __forceinline__ void pump(const fm::KParams& P, const double2* __restrict__ pts, WarpSmemQ& S,
                                     RingState& R, bool drain, int lane, int* __restrict__ res,
                                     const HistSink& hist, fm::WorkCount& wc) {
  for (;;) {
    const bool sf = R.qn >= 32 || (drain && R.qn > 0);
    const bool sh = !sf && (R.hn >= 32 || (drain && R.hn > 0));
    const bool sd = !sf && !sh && (R.dn >= kDblBatch || (drain && R.dn > 0));
    const bool stage = sf || sh || sd;
    if (!stage && !(drain && R.pend > 0)) break;
    int m = 0;
    QItem nit;
    nit.px = nit.py = 0.0;
    nit.i = 0;
    nit.e = fm::kEmpty;
    if (sf) {
      m = min(R.qn, 32);
      if (lane < m) {
        const int s = (R.head + lane) & (kQCap - 1);
        nit.i = S.qk[s];
        nit.e = S.qe[s];
      }
      R.head = (R.head + m) & (kQCap - 1);
      R.qn -= m;
    } else if (sh) {
      m = min(R.hn, 32);
      if (lane < m) {
        const int s = (R.hhead + lane) & (kQCap - 1);
        nit.i = S.hk[s];
        nit.e = S.he[s];
      }
      R.hhead = (R.hhead + m) & (kQCap - 1);
      R.hn -= m;
    } else if (sd) {
      m = min(R.dn, kDblBatch);
      if (lane < m) {
        const int s = (R.dhead + lane) & (kDCap - 1);
        nit.i = S.dk[s];
        nit.e = S.de[s];
      }
      R.dhead = (R.dhead + m) & (kDCap - 1);
      R.dn -= m;
    }
    if (stage) {
      __syncwarp();
      if (lane < m) {
        const double2 p = __ldg(pts + nit.i);
        nit.px = p.x;
        nit.py = p.y;
      }
      if (sf) {
        stage_full(P, S.pool[R.pb ^ 1], nit.e, m, lane);  // commits one group
      } else if (sh) {
        stage_half(P, S.pool[R.pb ^ 1], nit.e, m, lane);
      } else {
        stage_double(P, S.pool[R.pb ^ 1], nit.e, m, lane);
      }
    }
    if (R.pend > 0) {
      if (stage) {
        cp_async_wait1();
      } else {
        cp_async_wait0();
      }
      __syncwarp();
      std::uint32_t ce = 0u;
      if (R.pkind == 0) {
        ce = eval_staged<kHist, kCount>(P, S.pool[R.pb], R.pit, R.pend, lane, res, hist, wc);
      } else if (R.pkind == 1) {
        ce = eval_staged_half<kHist, kCount>(P, S.pool[R.pb], R.pit, R.pend, lane, res, hist, wc);
      } else {
        eval_staged_double<kHist, kCount>(S.pool[R.pb], R.pit, R.pend, lane, res, hist, wc);
      }
      const std::uint32_t rq = __ballot_sync(0xFFFFFFFFu, ce != 0u);
      if (ce != 0u) {  // split cell: the child entry goes into the full ring
        const int s = (R.head + R.qn + __popc(rq & ((1u << lane) - 1u))) & (kQCap - 1);
        S.qk[s] = R.pit.i;
        S.qe[s] = ce;
      }
      R.qn += __popc(rq);
      __syncwarp();
    }
    if (stage) R.pb ^= 1;
    R.pit = nit;
    R.pend = m;
    R.pkind = sf ? 0 : (sh ? 1 : 2);
    if (!drain && R.qn < 32 && R.hn < 32 && R.dn < kDblBatch) break;
  }
}

// Tile groups a warp takes per grab of the query pass's work counter.
constexpr int kQGroup = 8;

template <bool kHist, bool kCount, int kLs>
__global__ void __launch_bounds__(kQWarps * 32, FM_QMINB)
    binned_query_kernel(fm::KParams P, const double2* __restrict__ pts, std::uint64_t n,
                        const unsigned long long* __restrict__ n_dev, int* __restrict__ res,
                        HistT* __restrict__ hist, unsigned long long* __restrict__ counters,
                        unsigned long long* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  if (n_dev) n = min(n, static_cast<std::uint64_t>(*n_dev));  // the sealed binned length
  // a batch (<= 2^30 points) and its bin padding stay below 2^31 points: 32-bit indices throughout
  const std::uint32_t n32 = static_cast<std::uint32_t>(n);
  __shared__ HotSmem<kHist> hot;
  const HistSink hs = hist_open<kHist>(hist, hot);
  WarpSmemQ& S = reinterpret_cast<WarpSmemQ*>(dsmem)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  constexpr std::uint32_t tile = 32u * kU;
  const std::uint32_t n_tiles = (n32 + tile - 1) / tile;
  const std::uint32_t lt_mask = (1u << lane) - 1u;
  fm::WorkCount wc;
  RingState R;
  R.pit.px = R.pit.py = 0.0;
  R.pit.i = 0;
  R.pit.e = fm::kEmpty;
  // the warp's tiles: groups of kQGroup consecutive tiles from the counter
  auto grab = [&]() -> std::uint32_t {
    std::uint32_t g = 0;
    if (lane == 0) g = static_cast<std::uint32_t>(min(atomicAdd(work + kCtrQuery, 1ull), 0x3FFFFFFull));
    return __shfl_sync(0xFFFFFFFFu, g, 0) * kQGroup;
  };
  // software pipeline over the warp's tiles t < t1 < t2: the points of t2
  // are loading and the grid entries of t1 are in flight while tile t is
  // answered, so neither latency is exposed (16 warps per SM do not hide
  // the grid gather on their own)
  auto next_tile = [&](std::uint32_t x, std::uint32_t& g_end) -> std::uint32_t {
    std::uint32_t y = x + 1;
    if (y == g_end) {
      y = grab();
      g_end = y + kQGroup;
    }
    return y;
  };
  auto load_pts = [&](std::uint32_t x, double2 (&q)[kU]) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const std::uint32_t i = x * tile + u * 32 + lane;
      q[u] = (x < n_tiles && i < n32) ? FM_QLD(pts + i) : make_double2(NAN, NAN);
    }
  };
  std::uint32_t g_end = 0;
  std::uint32_t t = grab();
  g_end = t + kQGroup;
  std::uint32_t t1 = t < n_tiles ? next_tile(t, g_end) : n_tiles;
  double2 p[kU], p1[kU], p2[kU];
  std::uint32_t e[kU], e1[kU];
  load_pts(t, p);
  load_pts(t1, p1);
  fm::locate_n<kU, true, kLs>(P, p, e);
  unsigned long long done = 0;
  while (t < n_tiles) {
    const std::uint32_t base = t * tile;
    const std::uint32_t t2 = t1 < n_tiles ? next_tile(t1, g_end) : n_tiles;
    load_pts(t2, p2);
    fm::locate_n<kU, true, kLs>(P, p1, e1);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const std::uint32_t i = base + u * 32 + lane;
      const bool valid = i < n32;
      const bool is_rec = valid && e[u] >= fm::kRecordBit && e[u] != fm::kEmpty;
      const bool is_dbl = is_rec && (e[u] & fm::kDoubleBit) && !(e[u] & fm::kHalfBit);
      if (valid && !is_rec) emit<kHist>(res, hs, i, e[u] < fm::kRecordBit ? static_cast<int>(e[u]) : -1);
      const bool is_half = is_rec && (e[u] & fm::kHalfBit);
      const std::uint32_t b = __ballot_sync(0xFFFFFFFFu, is_rec && !is_dbl && !is_half);
      if (is_rec && !is_dbl && !is_half) {
        const int s = (R.head + R.qn + __popc(b & lt_mask)) & (kQCap - 1);
        S.qk[s] = i;
        S.qe[s] = e[u];
      }
      R.qn += __popc(b);
      const std::uint32_t bh = __ballot_sync(0xFFFFFFFFu, is_half);
      if (is_half) {
        const int s = (R.hhead + R.hn + __popc(bh & lt_mask)) & (kQCap - 1);
        S.hk[s] = i;
        S.he[s] = e[u];
      }
      R.hn += __popc(bh);
      const std::uint32_t bd = __ballot_sync(0xFFFFFFFFu, is_dbl);
      if (is_dbl) {
        const int s = (R.dhead + R.dn + __popc(bd & lt_mask)) & (kDCap - 1);
        S.dk[s] = i;
        S.de[s] = e[u];
      }
      R.dn += __popc(bd);
    }
    if (kCount) done += min(tile, n32 - base);
    __syncwarp();
    pump<kHist, kCount>(P, pts, S, R, false, lane, res, hs, wc);
    t = t1;
    t1 = t2;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      p[u] = p1[u];
      p1[u] = p2[u];
      e[u] = e1[u];
    }
  }
  pump<kHist, kCount>(P, pts, S, R, true, lane, res, hs, wc);
  hist_close<kHist>(hs);
  if (kCount) {
    unsigned long long v[4] = {lane == 0 ? done : 0ull, wc.boundary, wc.cands, wc.edges};
#pragma unroll
    for (int k = 1; k < 4; ++k) {
      for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xFFFFFFFFu, v[k], o);
    }
    if (lane == 0) {
      for (int k = 0; k < 4; ++k) atomicAdd(counters + k, v[k]);
    }
  }
}

// The per-block histogram of a binned batch, from res[] in binned order
// (after binned_query_kernel, which then runs without histogram code).
// One CTA per SM takes one contiguous range of the answers -- a few index
// tiles at most, so a bounded set of leaves and, in clustered streams, long
// repeats -- and aggregates them in a shared-memory hash table (open
// addressing, kHistSlots keys) that lives across the whole range: it is
// flushed to the global counters (one atomic per distinct leaf) only when
// half full and at the end.  Answers whose probe sequence finds no slot go
// straight to the global counters.  (Round 2's first version flushed a
// 4096-slot table after every 4096 answers: 12.7 ms per 1B c3 answers,
// close to one global atomic per answer; profiles/r2aa.)
constexpr int kHistThreads = 1024;
constexpr int kHistSlots = 16384;
constexpr int kHistProbes = 16;
constexpr int kHistSmem = kHistSlots * 8;
constexpr int kHistStep = kHistThreads * 4;  // answers per round: one 16-byte load per thread

__global__ void __launch_bounds__(kHistThreads, 1)
    binned_hist_kernel(const int* __restrict__ res, std::uint64_t n, const unsigned long long* __restrict__ n_dev,
                       HistT* __restrict__ hist) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned int* s_key = reinterpret_cast<unsigned int*>(smem_raw);
  unsigned int* s_cnt = s_key + kHistSlots;
  __shared__ unsigned int s_ins;
  if (n_dev) n = min(n, static_cast<std::uint64_t>(*n_dev));
  for (int k = threadIdx.x; k < kHistSlots; k += kHistThreads) {
    s_key[k] = fm::kEmpty;
    s_cnt[k] = 0u;
  }
  if (threadIdx.x == 0) s_ins = 0u;
  // the CTA's range: whole steps, so every 16-byte load is aligned
  const std::uint64_t steps = (n + kHistStep - 1) / kHistStep;
  const std::uint64_t per = (steps + gridDim.x - 1) / gridDim.x;
  const std::uint64_t s0 = min(steps, per * blockIdx.x), s1 = min(steps, s0 + per);
  auto flush = [&]() {
    __syncthreads();
    for (int k = threadIdx.x; k < kHistSlots; k += kHistThreads) {
      const unsigned int key = s_key[k];
      if (key != fm::kEmpty) {
        atomicAdd(hist + key, s_cnt[k]);
        s_key[k] = fm::kEmpty;
        s_cnt[k] = 0u;
      }
    }
    if (threadIdx.x == 0) s_ins = 0u;
    __syncthreads();
  };
  auto add = [&](int id) {
    if (id < 0) return;
    const unsigned int u = static_cast<unsigned int>(id);
    unsigned int h = (u * 2654435761u) >> 18;  // 14-bit multiplicative hash
    for (int q = 0; q < kHistProbes; ++q, h = (h + 1) & (kHistSlots - 1)) {
      unsigned int t = s_key[h];
      if (t == fm::kEmpty) {
        t = atomicCAS(s_key + h, fm::kEmpty, u);
        if (t == fm::kEmpty) {
          atomicAdd(&s_ins, 1u);
          t = u;
        }
      }
      if (t == u) {
        atomicAdd(s_cnt + h, 1u);
        return;
      }
    }
    atomicAdd(hist + u, 1u);
  };
  __syncthreads();
  for (std::uint64_t st = s0; st < s1; ++st) {
    const std::uint64_t i = st * kHistStep + 4ull * threadIdx.x;
    if (i + 4 <= n) {
      const int4 v = __ldcs(reinterpret_cast<const int4*>(res + i));
      add(v.x);
      add(v.y);
      add(v.z);
      add(v.w);
    } else {
      for (std::uint64_t k = i; k < n; ++k) add(__ldcs(res + k));
    }
    if (__syncthreads_or(s_ins > kHistSlots / 2)) flush();  // a uniform vote, whenever each thread read s_ins
  }
  flush();
}

// A point the binning could not place (out[i] == kUnplacedId; see the sampled
// capacities above): answered straight from the index, histogram and
// counters included.  Never taken when the sample represents the stream.
__device__ __noinline__ int answer_unplaced(const fm::KParams& P, double2 p, HistT* __restrict__ hist,
                                            unsigned long long* __restrict__ counters) {
  double2 q[1] = {p};
  std::uint32_t e[1];
  fm::locate_n<1, true, -1>(P, q, e);
  fm::WorkCount wc;
  int id;
  if (e[0] == fm::kEmpty) {
    id = -1;
  } else if (e[0] < fm::kRecordBit) {
    id = static_cast<int>(e[0]);
  } else {
    id = fm::resolve_slot_global<true>(P, e[0], p.x, p.y, wc);
  }
  if (hist && id >= 0) atomicAdd(hist + id, 1u);
  if (counters) {
    atomicAdd(counters, 1ull);
    atomicAdd(counters + 1, wc.boundary);
    atomicAdd(counters + 2, wc.cands);
    atomicAdd(counters + 3, wc.edges);
  }
  return id;
}

// out[i] = res[binned position of i], through the chunk's run table (see
// bin_scatter_kernel): coalesced reads of res in sorted order, then the
// chunk's answers through shared memory.
#ifndef FM_UB2_THREADS
#define FM_UB2_THREADS 512
#endif
constexpr int kUb2Threads = FM_UB2_THREADS;
constexpr int kUb2Per = kChunk / kUb2Threads;
static_assert(kChunk % kUb2Threads == 0, "whole rounds");
inline int ub2_smem(int nk4) { return kChunk * 6 + (kChunk / 32) * 2 + 2 * nk4 * 4; }

// Per chunk: the run table into shared memory; one flag per run head
// (s_flag[first sorted index] = key + 1) and, per 32 sorted indices, the key
// at the segment's start (binary search, one per segment); then sorted index
// k's key is the running maximum of the flags over its segment (a warp
// scan), its answer res[run's first position + (k - first index)] -- all of
// a thread's loads issued before the first is used.
#ifndef FM_UB_MINB
#define FM_UB_MINB 4  // 32 registers: 4 x 512 threads per SM (3: 3.14 ms, 4: 2.8 ms per 1B points)
#endif
__global__ void __launch_bounds__(kUb2Threads, FM_UB_MINB)
    unbin_kernel(const std::uint16_t* __restrict__ pos16, const unsigned int* __restrict__ tab, int nk,
                  BinTable B, const int* __restrict__ res, std::uint64_t n, int* __restrict__ out,
                  unsigned long long* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ unsigned long long s_grab;
  const int nk4 = (nk + 3) & ~3;
  int* s_res = reinterpret_cast<int*>(smem_raw);
  uint2* s_tab = reinterpret_cast<uint2*>(smem_raw + kChunk * 4);  // {first position, first sorted index | fitting points << 16}
  std::uint16_t* s_flag = reinterpret_cast<std::uint16_t*>(s_tab + nk4);
  std::uint16_t* s_seg = s_flag + kChunk;
  const unsigned int ovf_base = B.hdr[0], ovf_cap = B.hdr[1];
  const std::uint64_t n_it = (n + kChunk - 1) / kChunk;
  const std::uint64_t stride = tab_stride(nk4);
  const int tid = threadIdx.x, lane = tid & 31;
  const bool vec = (reinterpret_cast<std::uintptr_t>(out) & 15u) == 0;
  for (int k = tid; k < kChunk; k += kUb2Threads) s_flag[k] = 0;
  std::uint64_t it = cta_grab(work + kCtrUnbin, &s_grab);
  while (it < n_it) {
    unsigned long long nxt = 0;
    if (tid == 0) nxt = atomicAdd(work + kCtrUnbin, 1ull);  // in flight while this chunk is answered
    const std::uint64_t base = it * kChunk;
    const int cnt = static_cast<int>(min(n, base + kChunk) - base);
    const unsigned int* tb = tab + it * stride;
    // whole chunks (every one but the stream's last) with a 16-byte aligned
    // output: four consecutive points per thread, one 8-byte load of their
    // sorted indices and one 16-byte store of their ids
    const bool whole = vec && cnt == kChunk && kUb2Per % 4 == 0;
    unsigned int kk[kUb2Per];
    if (whole) {
#pragma unroll
      for (int j = 0; j < kUb2Per / 4; ++j) {
        const uint2 w = __ldcs(reinterpret_cast<const uint2*>(pos16 + base) + j * kUb2Threads + tid);
        kk[4 * j + 0] = w.x & 0xFFFFu;
        kk[4 * j + 1] = w.x >> 16;
        kk[(4 * j + 2) % kUb2Per] = w.y & 0xFFFFu;
        kk[(4 * j + 3) % kUb2Per] = w.y >> 16;
      }
    } else {
#pragma unroll
      for (int j = 0; j < kUb2Per; ++j) {
        const int q = j * kUb2Threads + tid;
        kk[j] = q < cnt ? __ldcs(pos16 + base + q) : 0u;
      }
    }
    for (int k = tid; k < nk; k += kUb2Threads) s_tab[k] = __ldcs(reinterpret_cast<const uint2*>(tb) + k);
    __syncthreads();  // the table is in shared memory, every flag is zero
    bool ovf = false;
    for (int k = tid; k < nk; k += kUb2Threads) {
      const unsigned int w = s_tab[k].y, off = w & 0xFFFFu;
      const unsigned int end = k + 1 < nk ? (s_tab[k + 1].y & 0xFFFFu) : static_cast<unsigned int>(cnt);
      if (end > off) s_flag[off] = static_cast<std::uint16_t>(k + 1);
      ovf |= end - off > (w >> 16);  // some of the run went to the overflow bin
    }
    for (int sg = tid; sg * 32 < cnt; sg += kUb2Threads) {
      int lo = 0, hi = nk;  // the last key whose first sorted index is <= 32 sg
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((s_tab[mid].y & 0xFFFFu) <= static_cast<unsigned int>(32 * sg)) {
          lo = mid + 1;
        } else {
          hi = mid;
        }
      }
      s_seg[sg] = static_cast<std::uint16_t>(lo);  // key + 1
    }
    const bool plain = !__syncthreads_or(ovf) && cnt == kChunk;  // whole chunk, every run in its bin
    unsigned int idx[kUb2Per];
#pragma unroll
    for (int j = 0; j < kUb2Per; ++j) {
      const int k = j * kUb2Threads + tid;
      unsigned int f = s_flag[k];
      s_flag[k] = 0;
      // the last run head at or before this lane (run heads are sparse: one
      // ballot and one shuffle instead of a five-step scan), else the
      // segment's carry-in
      const unsigned int heads = __ballot_sync(0xFFFFFFFFu, f != 0u) & (0xFFFFFFFFu >> (31 - lane));
      const unsigned int hf = __shfl_sync(0xFFFFFFFFu, f, heads ? 31 - __clz(heads) : 0);
      f = heads ? hf : static_cast<unsigned int>(s_seg[k >> 5]);
      if (plain) {
        const uint2 e = s_tab[f - 1u];
        idx[j] = e.x + (static_cast<unsigned int>(k) - (e.y & 0xFFFFu));
      } else {
        idx[j] = kUnplaced;
        if (k < cnt) {
          const int key = static_cast<int>(f) - 1;
          const uint2 e = s_tab[key];
          const unsigned int r = static_cast<unsigned int>(k) - (e.y & 0xFFFFu), av = e.y >> 16;
          if (r < av) {
            idx[j] = e.x + r;
          } else {  // the run's tail went to the overflow bin (or nowhere)
            const unsigned int o = __ldg(tb + 2 * nk4 + key) + (r - av);
            if (o < ovf_cap) idx[j] = ovf_base + o;
          }
        }
      }
    }
    int v[kUb2Per];
    if (plain) {
#pragma unroll
      for (int j = 0; j < kUb2Per; ++j) v[j] = __ldcs(res + idx[j]);
    } else {
#pragma unroll
      for (int j = 0; j < kUb2Per; ++j) v[j] = idx[j] != kUnplaced ? __ldcs(res + idx[j]) : kUnplacedId;
    }
#pragma unroll
    for (int j = 0; j < kUb2Per; ++j) s_res[j * kUb2Threads + tid] = v[j];
    __syncthreads();
    if (whole) {
      int4* o4 = reinterpret_cast<int4*>(out + base);
#pragma unroll
      for (int j = 0; j < kUb2Per / 4; ++j) {
        __stcs(o4 + j * kUb2Threads + tid, make_int4(s_res[kk[4 * j]], s_res[kk[4 * j + 1]],
                                                     s_res[kk[(4 * j + 2) % kUb2Per]], s_res[kk[(4 * j + 3) % kUb2Per]]));
      }
    } else {
#pragma unroll
      for (int j = 0; j < kUb2Per; ++j) {
        const int q = j * kUb2Threads + tid;
        if (q < cnt) __stcs(out + base + q, s_res[kk[j]]);
      }
    }
    if (tid == 0) s_grab = nxt;
    __syncthreads();
    it = s_grab;
  }
}

__global__ void __launch_bounds__(256)
    unplaced_kernel(BinTable B, std::uint64_t n, fm::KParams P, const double2* __restrict__ pts,
                     int* __restrict__ out, HistT* __restrict__ hist, unsigned long long* __restrict__ counters) {
  if (B.hdr[2] <= B.hdr[1]) return;
  for (std::uint64_t i = static_cast<std::uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<std::uint64_t>(gridDim.x) * blockDim.x) {
    if (out[i] == kUnplacedId) out[i] = answer_unplaced(P, __ldg(pts + i), hist, counters);
  }
}
