// binned.cuh -- the tile-binned query path (north star item 2, "point
// binning"), included by fastmap_b200.cu inside its anonymous namespace
// (it reuses QItem, stage_slots, eval_staged and emit from there).
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
// true-hit indexes (c1, c2) -- see choose_path() in fastmap_b200.cu.
//
// Four launches (and a library scan) per batch of n <= 2^30 points
// (DESIGN.md sec. 5.3); the stream is cut into chunks of >= 4096 points:
//   bin_count_kernel    per chunk, a shared-memory histogram of tile keys:
//                       column c of the tile-major (n_tiles + 1) x n_chunks
//                       table
//   (cub exclusive scan of the table: entry (t, c) becomes the first
//    binned position of chunk c's points in tile t)
//   bin_scatter_kernel  per chunk, 4K points at a time: a shared-memory
//                       counting sort by tile, then the points written out
//                       run by run at the chunk's cursors (pts_b), their
//                       binned positions to pos[i] (coalesced)
//   binned_query_kernel the query over pts_b in order: locate, true hits
//                       answered at once, boundary points through a
//                       warp-private shared-memory ring whose batches of 32
//                       slots are staged by cp.async one batch ahead of
//                       their evaluation (exactly resolve_kernel's code);
//                       answers to res[k]
//   unbin_kernel        out[i] = res[pos[i]]
// Chunks are walked with a grid stride, so within a tile the points stay
// in about input order and any window of consecutive input points maps to
// about one contiguous range per tile: the gather in unbin_kernel and the
// scattered writes of the scatter stay coherent in L2 and the TLB.
// Points outside the acceptance box (and NaN) go to one extra bin; the
// query pass answers them -1 like every other path.
//
// Only performance depends on the binning: every point is answered by the
// same locate_n / eval_leaf_slot code as the stream path, so the answers
// are identical whatever tile or order a point ends up in.

#ifndef FM_QMINB
#define FM_QMINB 2
#endif

constexpr int kMaxTiles = 4096;                         // keys < kMaxTiles + 1

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
  int n_tiles = 1;   // tnx * tny; key n_tiles = outside the acceptance box
};

__device__ __forceinline__ int tile_key(const fm::KParams& P, const TileGeom& T, double px,
                                        double py) {
  const bool in = px >= P.ax0 && px <= P.ax1 && py >= P.ay0 && py <= P.ay1;
  int ix = in ? static_cast<int>(__dmul_rn(__dsub_rn(px, P.gx0), P.inv_w)) : 0;
  int iy = in ? static_cast<int>(__dmul_rn(__dsub_rn(py, P.gy0), P.inv_h)) : 0;
  ix = min(max(ix, 0), P.nx - 1);
  iy = min(max(iy, 0), P.ny - 1);
  return in ? (iy >> T.ts) * T.tnx + (ix >> T.ts) : T.n_tiles;
}

// The point stream is cut into chunks of ch = kScatterIter * m points
// (m >= 1 keeps the (n_tiles + 1) x n_chunks table under kMaxTableEntries),
// and both passes walk the chunks with a grid stride: at any moment the
// whole grid reads one narrow window of the stream and, in every tile, writes
// one narrow window of its runs.  (Contiguous per-CTA blocks measured 3.35
// TB/s for the same copy against 5.7 TB/s for a grid stride: hundreds of
// streams far apart in memory thrash the TLB -- tools/exp_copy.cu,
// profiles/r2q.)
#ifndef FM_SC_PER
#define FM_SC_PER 16
#endif
constexpr int kScatterThreads = 256;
constexpr int kScPer = FM_SC_PER;
constexpr int kScatterIter = kScatterThreads * kScPer;  // 4096 points
constexpr std::uint64_t kMaxTableEntries = std::uint64_t{64} << 20;

// table[t * n_chunks + c] = points of chunk c in tile t (a shared-memory
// histogram per chunk)
__global__ void __launch_bounds__(kScatterThreads)
    bin_count_kernel(fm::KParams P, TileGeom T, const double2* __restrict__ pts, std::uint64_t n,
                     std::uint64_t ch, unsigned int* __restrict__ table) {
  extern __shared__ unsigned int s_hist[];
  const std::uint64_t n_chunks = (n + ch - 1) / ch;
  for (std::uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    for (int k = threadIdx.x; k <= T.n_tiles; k += blockDim.x) s_hist[k] = 0u;
    __syncthreads();
    const std::uint64_t hi = min(n, (c + 1) * ch);
    for (std::uint64_t i0 = c * ch + threadIdx.x; i0 < hi; i0 += kScatterIter) {
      double2 p[kScPer];
#pragma unroll
      for (int j = 0; j < kScPer; ++j) {
        const std::uint64_t i = i0 + static_cast<std::uint64_t>(j) * kScatterThreads;
        p[j] = i < hi ? __ldcs(pts + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int j = 0; j < kScPer; ++j) {
        const std::uint64_t i = i0 + static_cast<std::uint64_t>(j) * kScatterThreads;
        if (i < hi) atomicAdd(s_hist + tile_key(P, T, p[j].x, p[j].y), 1u);
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k <= T.n_tiles; k += blockDim.x) table[static_cast<std::uint64_t>(k) * n_chunks + c] = s_hist[k];
    __syncthreads();
  }
}

// The scatter.  Per chunk, the global cursors start at the scanned table
// entries of the chunk; each kScatterIter-point iteration is counting-sorted
// by tile in shared memory and then written out run by run, so consecutive
// lanes store consecutive points of one run (whole lines) instead of each
// lane storing 16 bytes into a different tile's run: scattering 16-byte
// points into >= 16 interleaved fronts runs at 0.8-2.6 TB/s against 5.6 for
// a copy (tools/exp_copy.cu, profiles/r2s).  Each point's binned position
// goes to pos[i] (coalesced).  Within a tile the points stay in chunk order,
// i.e. in about input order, so the gather in unbin_kernel is coherent.
__global__ void __launch_bounds__(kScatterThreads)
    bin_scatter_kernel(fm::KParams P, TileGeom T, const double2* __restrict__ pts, std::uint64_t n,
                       std::uint64_t ch, const unsigned int* __restrict__ starts,
                       double2* __restrict__ pts_b, unsigned int* __restrict__ pos) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nk = T.n_tiles + 1;
  const int nk4 = (nk + 3) & ~3;
  double2* stage = reinterpret_cast<double2*>(smem_raw);
  unsigned int* sdst = reinterpret_cast<unsigned int*>(smem_raw + kScatterIter * 16);
  unsigned int* s_cnt = reinterpret_cast<unsigned int*>(smem_raw + kScatterIter * 20);
  unsigned int* s_off = s_cnt + nk4;
  unsigned int* s_gst = s_off + nk4;
  __shared__ unsigned int s_part[64];
  constexpr int kScanPer = (kMaxTiles + 1 + kScatterThreads - 1) / kScatterThreads;
  const std::uint64_t n_chunks = (n + ch - 1) / ch;
  for (int k = threadIdx.x; k < nk; k += blockDim.x) s_cnt[k] = 0u;
  for (std::uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    for (int k = threadIdx.x; k < nk; k += blockDim.x) s_gst[k] = starts[static_cast<std::uint64_t>(k) * n_chunks + c];
    const std::uint64_t hi = min(n, (c + 1) * ch);
    for (std::uint64_t base = c * ch; base < hi; base += kScatterIter) {
      double2 p[kScPer];
      unsigned int kr[kScPer];
#pragma unroll
      for (int j = 0; j < kScPer; ++j) {
        const std::uint64_t i = base + static_cast<std::uint64_t>(j) * kScatterThreads + threadIdx.x;
        p[j] = i < hi ? __ldcs(pts + i) : make_double2(0.0, 0.0);
      }
      __syncthreads();  // s_cnt zeroed, s_gst loaded / advanced
#pragma unroll
      for (int j = 0; j < kScPer; ++j) {
        const std::uint64_t i = base + static_cast<std::uint64_t>(j) * kScatterThreads + threadIdx.x;
        kr[j] = 0xFFFFFFFFu;
        if (i < hi) {
          const unsigned int key = static_cast<unsigned int>(tile_key(P, T, p[j].x, p[j].y));
          kr[j] = (key << 16) | atomicAdd(s_cnt + key, 1u);
        }
      }
      __syncthreads();
      {  // exclusive scan of s_cnt over the tiles -> s_off
        const int k0 = threadIdx.x * kScanPer;
        unsigned int v[kScanPer], sum = 0;
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) {
          v[q] = k0 + q < nk ? s_cnt[k0 + q] : 0u;
          sum += v[q];
        }
        // block-wide exclusive scan of the per-thread sums: shuffles within
        // each warp, the eight warp totals through shared memory (2 barriers)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        unsigned int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned int x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= o) incl += x;
        }
        if (lane == 31) s_part[warp] = incl;
        __syncthreads();
        if (warp == 0) {
          const unsigned int w = lane < kScatterThreads / 32 ? s_part[lane] : 0u;
          unsigned int wi = w;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned int x = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= o) wi += x;
          }
          if (lane < kScatterThreads / 32) s_part[32 + lane] = wi - w;  // exclusive warp offsets
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
#pragma unroll
      for (int j = 0; j < kScPer; ++j) {
        const std::uint64_t i = base + static_cast<std::uint64_t>(j) * kScatterThreads + threadIdx.x;
        if (kr[j] != 0xFFFFFFFFu) {
          const unsigned int key = kr[j] >> 16, r = kr[j] & 0xFFFFu;
          const unsigned int k = s_off[key] + r, dst = s_gst[key] + r;
          stage[k] = p[j];
          sdst[k] = dst;
          __stcs(pos + i, dst);
        }
      }
      __syncthreads();
      const int cnt = static_cast<int>(min(static_cast<std::uint64_t>(kScatterIter), hi - base));
#pragma unroll 4
      for (int k = threadIdx.x; k < cnt; k += kScatterThreads) pts_b[sdst[k]] = stage[k];  // run by run
      __syncthreads();
      for (int k = threadIdx.x; k < nk; k += blockDim.x) {
        s_gst[k] += s_cnt[k];
        s_cnt[k] = 0u;
      }
    }
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
// Points in double slots (kDoubleBit; polygon corners) wait in a second
// ring of (binned index, entry) pairs and are evaluated in whole batches of
// 32 straight from global memory (both halves of the 256-byte slot loaded
// at once), so the leaf-slot batches never run the wider double-slot code.
constexpr int kQWarps = 8;
constexpr int kQCap = 128;
constexpr int kDCap = 128;
struct WarpSmemQ {
  alignas(16) std::uint8_t pool[2][32 * fm::kSlotBytes];
  double qx[kQCap], qy[kQCap];
  std::uint32_t qk[kQCap], qe[kQCap];
  std::uint32_t dk[kDCap], de[kDCap];
};
constexpr int kSmemQ = static_cast<int>(sizeof(WarpSmemQ)) * kQWarps;

struct RingState {
  int head = 0, qn = 0;  // ring items not yet staged
  int pend = 0;          // items of the staged batch in pool[pb]
  int pb = 0;
  QItem pit;             // this lane's staged item
  int dhead = 0, dn = 0; // double-slot ring
};

// Evaluate double-slot points in batches of 32 (any remainder when draining).
template <bool kHist, bool kCount>
__device__ __forceinline__ void dpump(const fm::KParams& P, const double2* __restrict__ pts, WarpSmemQ& S,
                                      RingState& R, bool drain, int lane, int* __restrict__ res,
                                      const HistSink& hist, fm::WorkCount& wc) {
  while (R.dn >= 32 || (drain && R.dn > 0)) {
    const int m = min(R.dn, 32);
    std::uint32_t k = 0, e = 0;
    if (lane < m) {
      const int s = (R.dhead + lane) & (kDCap - 1);
      k = S.dk[s];
      e = S.de[s];
    }
    R.dhead = (R.dhead + m) & (kDCap - 1);
    R.dn -= m;
    __syncwarp();
    if (lane < m) {
      const double2 p = __ldg(pts + k);
      const uint4* g = reinterpret_cast<const uint4*>(fm::slot_ptr(P, e));
      uint4 a[8], b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = __ldg(g + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = __ldg(g + 8 + j);
      if (kCount) wc.boundary++;
      emit<kHist>(res, hist, k, fm::eval_double_slot<kCount>(a, b, p.x, p.y, wc));
    }
  }
}

// Stage the next batch (when 32 items wait, or any when draining) and
// evaluate the previously staged one; repeat while full batches remain.
template <bool kHist, bool kCount>
__device__ __forceinline__ void pump(const fm::KParams& P, WarpSmemQ& S, RingState& R, bool drain,
                                     int lane, int* __restrict__ res, const HistSink& hist,
                                     fm::WorkCount& wc) {
  for (;;) {
    const bool stage = R.qn >= 32 || (drain && R.qn > 0);
    if (!stage && !(drain && R.pend > 0)) break;
    int m = 0;
    QItem nit;
    nit.px = nit.py = 0.0;
    nit.i = 0;
    nit.e = fm::kEmpty;
    if (stage) {
      m = min(R.qn, 32);
      if (lane < m) {
        const int s = (R.head + lane) & (kQCap - 1);
        nit.px = S.qx[s];
        nit.py = S.qy[s];
        nit.i = S.qk[s];
        nit.e = S.qe[s];
      }
      R.head = (R.head + m) & (kQCap - 1);
      R.qn -= m;
      __syncwarp();
      stage_slots(P, S.pool[R.pb ^ 1], nit.e, m, lane);  // commits one group
    }
    if (R.pend > 0) {
      if (stage) {
        cp_async_wait1();
      } else {
        cp_async_wait0();
      }
      __syncwarp();
      const std::uint32_t ce = eval_staged<kHist, kCount>(P, S.pool[R.pb], R.pit, R.pend, lane, res,
                                                          hist, wc);
      const std::uint32_t rq = __ballot_sync(0xFFFFFFFFu, ce != 0u);
      if (ce != 0u) {  // split cell: the child entry goes back into the ring
        const int s = (R.head + R.qn + __popc(rq & ((1u << lane) - 1u))) & (kQCap - 1);
        S.qx[s] = R.pit.px;
        S.qy[s] = R.pit.py;
        S.qk[s] = R.pit.i;
        S.qe[s] = ce;
      }
      R.qn += __popc(rq);
      __syncwarp();
    }
    if (stage) R.pb ^= 1;
    R.pit = nit;
    R.pend = m;
    if (!drain && R.qn < 32) break;
  }
}

// Tile groups a warp takes per grab of the query pass's work counter.
constexpr int kQGroup = 8;

template <bool kHist, bool kCount, int kLs>
__global__ void __launch_bounds__(kQWarps * 32, FM_QMINB)
    binned_query_kernel(fm::KParams P, const double2* __restrict__ pts, std::uint64_t n,
                        int* __restrict__ res, HistT* __restrict__ hist,
                        unsigned long long* __restrict__ counters,
                        unsigned long long* __restrict__ work) {
  extern __shared__ __align__(16) unsigned char dsmem[];
  __shared__ HotSmem<kHist> hot;
  const HistSink hs = hist_open<kHist>(hist, hot);
  WarpSmemQ& S = reinterpret_cast<WarpSmemQ*>(dsmem)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const std::uint64_t tile = 32ull * kU;
  const std::uint64_t n_tiles = (n + tile - 1) / tile;
  const std::uint32_t lt_mask = (1u << lane) - 1u;
  fm::WorkCount wc;
  RingState R;
  R.pit.px = R.pit.py = 0.0;
  R.pit.i = 0;
  R.pit.e = fm::kEmpty;
  // the warp's tiles: groups of kQGroup consecutive tiles from the counter
  auto grab = [&]() -> std::uint64_t {
    unsigned long long g = 0;
    if (lane == 0) g = atomicAdd(work + kCtrQuery, 1ull);
    return static_cast<std::uint64_t>(__shfl_sync(0xFFFFFFFFu, g, 0)) * kQGroup;
  };
  // software pipeline over the warp's tiles t < t1 < t2: the points of t2
  // are loading and the grid entries of t1 are in flight while tile t is
  // answered, so neither latency is exposed (16 warps per SM do not hide
  // the grid gather on their own)
  auto next_tile = [&](std::uint64_t x, std::uint64_t& g_end) -> std::uint64_t {
    std::uint64_t y = x + 1;
    if (y == g_end) {
      y = grab();
      g_end = y + kQGroup;
    }
    return y;
  };
  auto load_pts = [&](std::uint64_t x, double2 (&q)[kU]) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const std::uint64_t i = x * tile + u * 32 + lane;
      q[u] = (x < n_tiles && i < n) ? __ldcs(pts + i) : make_double2(NAN, NAN);
    }
  };
  std::uint64_t g_end = 0;
  std::uint64_t t = grab();
  g_end = t + kQGroup;
  std::uint64_t t1 = t < n_tiles ? next_tile(t, g_end) : n_tiles;
  double2 p[kU], p1[kU], p2[kU];
  std::uint32_t e[kU], e1[kU];
  load_pts(t, p);
  load_pts(t1, p1);
  fm::locate_n<kU, true, kLs>(P, p, e);
  unsigned long long done = 0;
  while (t < n_tiles) {
    const std::uint64_t base = t * tile;
    const std::uint64_t t2 = t1 < n_tiles ? next_tile(t1, g_end) : n_tiles;
    load_pts(t2, p2);
    fm::locate_n<kU, true, kLs>(P, p1, e1);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const std::uint64_t i = base + u * 32 + lane;
      const bool valid = i < n;
      const bool is_rec = valid && e[u] >= fm::kRecordBit && e[u] != fm::kEmpty;
      const bool is_dbl = is_rec && (e[u] & fm::kDoubleBit) && !(e[u] & fm::kHalfBit);
      if (valid && !is_rec) emit<kHist>(res, hs, i, e[u] < fm::kRecordBit ? static_cast<int>(e[u]) : -1);
      const std::uint32_t b = __ballot_sync(0xFFFFFFFFu, is_rec && !is_dbl);
      if (is_rec && !is_dbl) {
        const int s = (R.head + R.qn + __popc(b & lt_mask)) & (kQCap - 1);
        S.qx[s] = p[u].x;
        S.qy[s] = p[u].y;
        S.qk[s] = static_cast<std::uint32_t>(i);
        S.qe[s] = e[u];
      }
      R.qn += __popc(b);
      const std::uint32_t bd = __ballot_sync(0xFFFFFFFFu, is_dbl);
      if (is_dbl) {
        const int s = (R.dhead + R.dn + __popc(bd & lt_mask)) & (kDCap - 1);
        S.dk[s] = static_cast<std::uint32_t>(i);
        S.de[s] = e[u];
      }
      R.dn += __popc(bd);
    }
    if (kCount) done += min(tile, n - base);
    __syncwarp();
    dpump<kHist, kCount>(P, pts, S, R, false, lane, res, hs, wc);
    pump<kHist, kCount>(P, S, R, false, lane, res, hs, wc);
    t = t1;
    t1 = t2;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      p[u] = p1[u];
      p1[u] = p2[u];
      e[u] = e1[u];
    }
  }
  dpump<kHist, kCount>(P, pts, S, R, true, lane, res, hs, wc);
  pump<kHist, kCount>(P, S, R, true, lane, res, hs, wc);
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
// (after binned_query_kernel, which then runs without histogram code).  A
// CTA takes chunks of kHistChunk consecutive answers -- one tile's points,
// so a few thousand distinct leaves at most and, in clustered streams, many
// repeats -- and aggregates them in a shared-memory hash table (open
// addressing, kHistSlots keys) before one global atomic per distinct leaf.
// Answers whose probe sequence finds no free slot go straight to the global
// counters.
constexpr int kHistThreads = 512;
#ifndef FM_HIST_CHUNK
#define FM_HIST_CHUNK 4096  // r2aa: 12.7 ms per 1B c3 answers (16384: 14.2, 65536: 15.4)
#endif
#ifndef FM_HIST_AGG
#define FM_HIST_AGG 0  // experiments: 1 = __match_any_sync aggregation before the table
#endif
constexpr int kHistChunk = FM_HIST_CHUNK;
constexpr int kHistSlots = 4096;
constexpr int kHistProbes = 8;

__global__ void __launch_bounds__(kHistThreads)
    binned_hist_kernel(const int* __restrict__ res, std::uint64_t n, HistT* __restrict__ hist) {
  __shared__ unsigned int s_key[kHistSlots];
  __shared__ unsigned int s_cnt[kHistSlots];
  for (int k = threadIdx.x; k < kHistSlots; k += blockDim.x) {
    s_key[k] = fm::kEmpty;
    s_cnt[k] = 0u;
  }
  const std::uint64_t n_chunks = (n + kHistChunk - 1) / kHistChunk;
  for (std::uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    __syncthreads();
    const std::uint64_t lo = c * kHistChunk, hi = min(n, lo + kHistChunk);
    for (std::uint64_t i = lo + threadIdx.x; i < hi; i += kHistThreads) {
      const int id = __ldcs(res + i);
#if FM_HIST_AGG
      const unsigned int peers = __match_any_sync(__activemask(), static_cast<unsigned int>(id));
      if (id < 0 || (threadIdx.x & 31) != static_cast<unsigned int>(__ffs(peers) - 1)) continue;
      const unsigned int inc = static_cast<unsigned int>(__popc(peers));
#else
      if (id < 0) continue;
      const unsigned int inc = 1u;
#endif
      const unsigned int u = static_cast<unsigned int>(id);
      unsigned int h = (u * 2654435761u) >> 20;  // 12-bit multiplicative hash
      bool done = false;
      for (int q = 0; q < kHistProbes && !done; ++q, h = (h + 1) & (kHistSlots - 1)) {
        unsigned int t = s_key[h];
        if (t == fm::kEmpty) {
          t = atomicCAS(s_key + h, fm::kEmpty, u);
          if (t == fm::kEmpty) t = u;
        }
        if (t == u) {
          atomicAdd(s_cnt + h, inc);
          done = true;
        }
      }
      if (!done) atomicAdd(hist + u, inc);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kHistSlots; k += blockDim.x) {
      const unsigned int key = s_key[k];
      if (key != fm::kEmpty) {
        atomicAdd(hist + key, s_cnt[k]);
        s_key[k] = fm::kEmpty;
        s_cnt[k] = 0u;
      }
    }
  }
}

// out[i] = res[pos[i]].  CTAs take blocks of kUnbinBlock points in
// increasing order from the work counter, four points per thread per round
// (16-byte pos loads and id stores when `out` is 16-byte aligned).
constexpr int kUnbinThreads = 256;
#ifndef FM_UNBIN_ROUNDS
#define FM_UNBIN_ROUNDS 8
#endif
constexpr int kUnbinRounds = FM_UNBIN_ROUNDS;
#ifndef FM_UNBIN_LD
#define FM_UNBIN_LD __ldg
#endif
constexpr std::uint64_t kUnbinBlock = 4ull * kUnbinThreads * kUnbinRounds;  // 8192 points

__global__ void __launch_bounds__(kUnbinThreads)
    unbin_kernel(const unsigned int* __restrict__ pos, const int* __restrict__ res, std::uint64_t n,
                 int* __restrict__ out, unsigned long long* __restrict__ work) {
  __shared__ unsigned long long s_grab;
  const bool vec = (reinterpret_cast<std::uintptr_t>(out) & 15u) == 0;
  const std::uint64_t n_blocks = (n + kUnbinBlock - 1) / kUnbinBlock;
  const uint4* p4 = reinterpret_cast<const uint4*>(pos);
  int4* o4 = reinterpret_cast<int4*>(out);
  for (std::uint64_t b = cta_grab(work + kCtrUnbin, &s_grab); b < n_blocks;
       b = cta_grab(work + kCtrUnbin, &s_grab)) {
    const std::uint64_t base = b * kUnbinBlock;
    if (vec && base + kUnbinBlock <= n) {
      // every pos load of the block, then every gather: 4 * kUnbinRounds
      // independent loads in flight per thread
      uint4 k[kUnbinRounds];
#pragma unroll
      for (int r = 0; r < kUnbinRounds; ++r) {
        k[r] = __ldcs(p4 + base / 4 + static_cast<std::uint64_t>(r) * kUnbinThreads + threadIdx.x);
      }
      int4 v[kUnbinRounds];
#pragma unroll
      for (int r = 0; r < kUnbinRounds; ++r) {
        v[r].x = FM_UNBIN_LD(res + k[r].x);
        v[r].y = FM_UNBIN_LD(res + k[r].y);
        v[r].z = FM_UNBIN_LD(res + k[r].z);
        v[r].w = FM_UNBIN_LD(res + k[r].w);
      }
#pragma unroll
      for (int r = 0; r < kUnbinRounds; ++r) {
        __stcs(o4 + base / 4 + static_cast<std::uint64_t>(r) * kUnbinThreads + threadIdx.x, v[r]);
      }
    } else {
      const std::uint64_t end = min(n, base + kUnbinBlock);
      for (std::uint64_t i = base + threadIdx.x; i < end; i += kUnbinThreads) {
        __stcs(out + i, __ldg(res + __ldcs(pos + i)));
      }
    }
  }
}
