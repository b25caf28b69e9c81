/*
 * oracle.c -- CPU restatement of the reference's point-to-block semantics.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only to check (never to produce) the
 * product's answers.  The product library (paper_2005_03156_b200/csrc)
 * never links or calls it.
 *
 * What it restates (citations are into /root/reference/proj):
 *   - the parity predicate detail::ray_crosses      include/fastmap/geometry.hpp:170-174
 *   - scalar even-odd point_in_polygon              include/fastmap/geometry.hpp:214-225
 *     over rings closed as PolygonGeometry::add_ring does  geometry.hpp:74-86
 *   - exhaustive_assign: first leaf (ascending) whose
 *     point_in_polygon is true, else -1             include/fastmap/synthetic.hpp:193-205
 *   - the lon/lat domain filter of query_leaves     include/fastmap/cell_index.hpp:549-552
 *
 * Build with -ffp-contract=off and WITHOUT -march=native: the predicate
 * must be evaluated as 2 products and 3 differences, each rounded, exactly
 * like the reference's default (x86-64 baseline, no FMA) build.
 *
 * Parity is pinned against the reference itself: tests compare this file's
 * answers with oracle/_ref/libfastmap_ref.so (the unmodified reference
 * headers compiled by oracle/Makefile) and with the golden vectors under
 * tests/golden/ that were produced from it by tools/make_golden.py.
 *
 * Polygon soup layout (shared with the product C-ABI):
 *   vxy[2*v+0], vxy[2*v+1]   lon, lat of vertex v (all rings concatenated)
 *   ring_off[r] .. ring_off[r+1]     vertices of ring r  (open ring, >= 3)
 *   poly_ring[p] .. poly_ring[p+1]   rings of polygon p (leaf p)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* geometry.hpp:170-174 */
static inline int ray_crosses(double px, double py, double lx, double ly,
                              double hx, double hy) {
  return (hx - lx) * (py - ly) - (hy - ly) * (px - lx) > 0.0;
}

/* geometry.hpp:214-225, one ring at a time (edges i -> i+1 and n-1 -> 0,
 * geometry.hpp:82-85).  Returns the parity contributed by the ring. */
static int ring_parity(double px, double py, const double* vxy, uint64_t b,
                       uint64_t e) {
  int in = 0;
  const uint64_t n = e - b;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t a = b + i;
    const uint64_t c = (i + 1 < n) ? a + 1 : b;
    double lx = vxy[2 * a], ly = vxy[2 * a + 1];
    double hx = vxy[2 * c], hy = vxy[2 * c + 1];
    if (ly > hy) {
      double t = lx; lx = hx; hx = t;
      t = ly; ly = hy; hy = t;
    }
    if (ly < py && py <= hy && ray_crosses(px, py, lx, ly, hx, hy)) in ^= 1;
  }
  return in;
}

int orc_point_in_polygon(double px, double py, const double* vxy,
                         const uint64_t* ring_off, const uint64_t* poly_ring,
                         uint64_t poly) {
  int in = 0;
  for (uint64_t r = poly_ring[poly]; r < poly_ring[poly + 1]; ++r) {
    in ^= ring_parity(px, py, vxy, ring_off[r], ring_off[r + 1]);
  }
  return in;
}

static inline int in_world(double px, double py) {
  /* cell_index.hpp:549-552 (kWorldBounds, cell_index.hpp:27); NaN fails */
  return px >= -180.0 && px <= 180.0 && py >= -90.0 && py <= 90.0;
}

/* synthetic.hpp:193-205, plus the world filter when world_check != 0. */
void orc_exhaustive_assign(const double* vxy, const uint64_t* ring_off,
                           const uint64_t* poly_ring, uint64_t n_polys,
                           const double* pts, uint64_t n_pts, int world_check,
                           int32_t* out) {
  for (uint64_t i = 0; i < n_pts; ++i) {
    const double px = pts[2 * i], py = pts[2 * i + 1];
    int32_t id = -1;
    if (!world_check || in_world(px, py)) {
      for (uint64_t l = 0; l < n_polys; ++l) {
        if (orc_point_in_polygon(px, py, vxy, ring_off, poly_ring, l)) {
          id = (int32_t)l;
          break;
        }
      }
    }
    out[i] = id;
  }
}

/* ------------------------------------------------------------------------
 * Bucketed exhaustive assignment.  Same answer as orc_exhaustive_assign:
 * a polygon can only test true for a point inside its closed bounding box
 * (an in-range edge needs lo.lat < y <= hi.lat; a crossing needs the point
 * left of the edge), so polygons are pre-bucketed by bbox on a uniform grid,
 * each bucket keeps ascending ids, and the bbox filter uses a pad of
 * 2^-30 * max(1, |coord|) so rounding in the predicate can never matter.
 * ---------------------------------------------------------------------- */

typedef struct {
  const double* vxy;
  const uint64_t* ring_off;
  const uint64_t* poly_ring;
  uint64_t n_polys;
  double* bbox; /* 4 per polygon, padded */
  double gx0, gy0, inv_w, inv_h;
  int64_t nx, ny;
  uint64_t* bucket_off; /* nx*ny + 1 */
  uint32_t* bucket_ids;
} orc_grid;

static void grid_cell_range(const orc_grid* g, double lo, double hi, double g0,
                            double inv, int64_t n, int64_t* a, int64_t* b) {
  double fa = floor((lo - g0) * inv) - 1.0, fb = floor((hi - g0) * inv) + 1.0;
  if (fa < 0) fa = 0;
  if (fb > (double)(n - 1)) fb = (double)(n - 1);
  *a = (int64_t)fa;
  *b = (int64_t)fb;
  (void)g;
}

static orc_grid* grid_build(const double* vxy, const uint64_t* ring_off,
                            const uint64_t* poly_ring, uint64_t n_polys) {
  orc_grid* g = (orc_grid*)calloc(1, sizeof(orc_grid));
  g->vxy = vxy;
  g->ring_off = ring_off;
  g->poly_ring = poly_ring;
  g->n_polys = n_polys;
  g->bbox = (double*)malloc(sizeof(double) * 4 * (n_polys ? n_polys : 1));
  double ux0 = INFINITY, ux1 = -INFINITY, uy0 = INFINITY, uy1 = -INFINITY;
  for (uint64_t p = 0; p < n_polys; ++p) {
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    const uint64_t vb = ring_off[poly_ring[p]], ve = ring_off[poly_ring[p + 1]];
    for (uint64_t v = vb; v < ve; ++v) {
      const double x = vxy[2 * v], y = vxy[2 * v + 1];
      if (x < x0) x0 = x;
      if (x > x1) x1 = x;
      if (y < y0) y0 = y;
      if (y > y1) y1 = y;
    }
    double m = fmax(fmax(fabs(x0), fabs(x1)), fmax(fabs(y0), fabs(y1)));
    if (!(m >= 1.0)) m = 1.0;
    const double pad = ldexp(m, -30);
    g->bbox[4 * p + 0] = x0 - pad;
    g->bbox[4 * p + 1] = x1 + pad;
    g->bbox[4 * p + 2] = y0 - pad;
    g->bbox[4 * p + 3] = y1 + pad;
    if (x0 - pad < ux0) ux0 = x0 - pad;
    if (x1 + pad > ux1) ux1 = x1 + pad;
    if (y0 - pad < uy0) uy0 = y0 - pad;
    if (y1 + pad > uy1) uy1 = y1 + pad;
  }
  if (n_polys == 0) { ux0 = uy0 = 0; ux1 = uy1 = 1; }
  int64_t side = (int64_t)ceil(sqrt((double)(n_polys ? n_polys : 1)));
  if (side < 1) side = 1;
  if (side > 8192) side = 8192;
  g->nx = side;
  g->ny = side;
  g->gx0 = ux0;
  g->gy0 = uy0;
  double w = (ux1 - ux0) / (double)side, h = (uy1 - uy0) / (double)side;
  if (!(w > 0)) w = 1;
  if (!(h > 0)) h = 1;
  g->inv_w = 1.0 / w;
  g->inv_h = 1.0 / h;
  const int64_t nc = g->nx * g->ny;
  g->bucket_off = (uint64_t*)calloc((size_t)nc + 1, sizeof(uint64_t));
  for (uint64_t p = 0; p < n_polys; ++p) {
    int64_t a, b, c, d;
    grid_cell_range(g, g->bbox[4 * p], g->bbox[4 * p + 1], g->gx0, g->inv_w, g->nx, &a, &b);
    grid_cell_range(g, g->bbox[4 * p + 2], g->bbox[4 * p + 3], g->gy0, g->inv_h, g->ny, &c, &d);
    for (int64_t iy = c; iy <= d; ++iy)
      for (int64_t ix = a; ix <= b; ++ix) g->bucket_off[iy * g->nx + ix + 1]++;
  }
  for (int64_t k = 0; k < nc; ++k) g->bucket_off[k + 1] += g->bucket_off[k];
  g->bucket_ids = (uint32_t*)malloc(sizeof(uint32_t) * (g->bucket_off[nc] + 1));
  uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)nc);
  memcpy(fill, g->bucket_off, sizeof(uint64_t) * (size_t)nc);
  for (uint64_t p = 0; p < n_polys; ++p) { /* ascending ids per bucket */
    int64_t a, b, c, d;
    grid_cell_range(g, g->bbox[4 * p], g->bbox[4 * p + 1], g->gx0, g->inv_w, g->nx, &a, &b);
    grid_cell_range(g, g->bbox[4 * p + 2], g->bbox[4 * p + 3], g->gy0, g->inv_h, g->ny, &c, &d);
    for (int64_t iy = c; iy <= d; ++iy)
      for (int64_t ix = a; ix <= b; ++ix)
        g->bucket_ids[fill[iy * g->nx + ix]++] = (uint32_t)p;
  }
  free(fill);
  return g;
}

static void grid_free(orc_grid* g) {
  free(g->bbox);
  free(g->bucket_off);
  free(g->bucket_ids);
  free(g);
}

static int32_t grid_assign_one(const orc_grid* g, double px, double py,
                               int world_check) {
  if (world_check && !in_world(px, py)) return -1;
  if (!(px == px) || !(py == py)) return -1; /* NaN: every PIP is false */
  if (g->n_polys == 0) return -1;
  const double tx = (px - g->gx0) * g->inv_w, ty = (py - g->gy0) * g->inv_h;
  if (!(tx >= 0.0 && ty >= 0.0 && tx < (double)g->nx && ty < (double)g->ny))
    return -1; /* outside every padded bbox */
  const int64_t k = (int64_t)ty * g->nx + (int64_t)tx;
  for (uint64_t q = g->bucket_off[k]; q < g->bucket_off[k + 1]; ++q) {
    const uint32_t p = g->bucket_ids[q];
    const double* bb = g->bbox + 4 * (uint64_t)p;
    if (px < bb[0] || px > bb[1] || py < bb[2] || py > bb[3]) continue;
    if (orc_point_in_polygon(px, py, g->vxy, g->ring_off, g->poly_ring, p))
      return (int32_t)p;
  }
  return -1;
}

typedef struct {
  const orc_grid* g;
  const double* pts;
  int32_t* out;
  uint64_t begin, end;
  int world_check;
  const uint64_t* order; /* NULL: points begin..end in input order */
} orc_job;

static void* orc_worker(void* arg) {
  orc_job* j = (orc_job*)arg;
  for (uint64_t k = j->begin; k < j->end; ++k) {
    const uint64_t i = j->order ? j->order[k] : k;
    j->out[i] = grid_assign_one(j->g, j->pts[2 * i], j->pts[2 * i + 1], j->world_check);
  }
  return NULL;
}

/* Large batches are visited bucket by bucket (a counting sort of the point
 * indices by bucket): consecutive points then test the same polygons, which
 * stay in cache.  Only the visiting order changes, not any answer. */
static uint64_t* bucket_order(const orc_grid* g, const double* pts, uint64_t n) {
  const int64_t nc = g->nx * g->ny;
  uint64_t* cnt = (uint64_t*)calloc((size_t)nc + 2, sizeof(uint64_t));
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n ? n : 1));
  int64_t* key = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  if (!cnt || !order || !key) {
    free(cnt);
    free(order);
    free(key);
    return NULL;
  }
  for (uint64_t i = 0; i < n; ++i) {
    const double tx = (pts[2 * i] - g->gx0) * g->inv_w, ty = (pts[2 * i + 1] - g->gy0) * g->inv_h;
    int64_t k = nc; /* outside (or NaN): one extra bucket */
    if (tx >= 0.0 && ty >= 0.0 && tx < (double)g->nx && ty < (double)g->ny)
      k = (int64_t)ty * g->nx + (int64_t)tx;
    key[i] = k;
    cnt[k + 1]++;
  }
  for (int64_t k = 0; k <= nc; ++k) cnt[k + 1] += cnt[k];
  for (uint64_t i = 0; i < n; ++i) order[cnt[key[i]]++] = i;
  free(cnt);
  free(key);
  return order;
}

/* Same semantics as orc_exhaustive_assign, bucketed and threaded. */
void orc_assign(const double* vxy, const uint64_t* ring_off,
                const uint64_t* poly_ring, uint64_t n_polys, const double* pts,
                uint64_t n_pts, int world_check, int threads, int32_t* out) {
  orc_grid* g = grid_build(vxy, ring_off, poly_ring, n_polys);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  uint64_t* order = n_pts >= (1u << 20) ? bucket_order(g, pts, n_pts) : NULL;
  pthread_t tid[256];
  orc_job jobs[256];
  const uint64_t per = (n_pts + (uint64_t)threads - 1) / (uint64_t)threads;
  int launched = 0;
  for (int t = 0; t < threads; ++t) {
    jobs[t].g = g;
    jobs[t].pts = pts;
    jobs[t].out = out;
    jobs[t].begin = per * (uint64_t)t;
    jobs[t].end = per * (uint64_t)(t + 1);
    if (jobs[t].begin > n_pts) jobs[t].begin = n_pts;
    if (jobs[t].end > n_pts) jobs[t].end = n_pts;
    jobs[t].world_check = world_check;
    jobs[t].order = order;
    if (t == threads - 1 || pthread_create(&tid[t], NULL, orc_worker, &jobs[t]) != 0) {
      orc_worker(&jobs[t]);
    } else {
      launched = t + 1;
    }
  }
  for (int t = 0; t < launched; ++t) pthread_join(tid[t], NULL);
  free(order);
  grid_free(g);
}

/* Per-point count of polygons whose PIP is true (diagnostic: >1 means the
 * input overlaps or self-intersects, where query_leaves and exhaustive
 * semantics can differ -- SURVEY.md sec. 0, finding 2). */
void orc_count_containing(const double* vxy, const uint64_t* ring_off,
                          const uint64_t* poly_ring, uint64_t n_polys,
                          const double* pts, uint64_t n_pts, int32_t* out) {
  orc_grid* g = grid_build(vxy, ring_off, poly_ring, n_polys);
  for (uint64_t i = 0; i < n_pts; ++i) {
    const double px = pts[2 * i], py = pts[2 * i + 1];
    int32_t cnt = 0;
    const double tx = (px - g->gx0) * g->inv_w, ty = (py - g->gy0) * g->inv_h;
    if (n_polys && tx >= 0.0 && ty >= 0.0 && tx < (double)g->nx && ty < (double)g->ny) {
      const int64_t k = (int64_t)ty * g->nx + (int64_t)tx;
      for (uint64_t q = g->bucket_off[k]; q < g->bucket_off[k + 1]; ++q) {
        const uint32_t p = g->bucket_ids[q];
        if (orc_point_in_polygon(px, py, vxy, ring_off, poly_ring, p)) ++cnt;
      }
    }
    out[i] = cnt;
  }
  grid_free(g);
}

/* tests/oracles.hpp:68-80: distance from p to segment ab (clamped projection). */
static double seg_distance(double px, double py, double ax, double ay, double bx, double by) {
  const double dx = bx - ax, dy = by - ay;
  const double len2 = dx * dx + dy * dy;
  double t = 0.0;
  if (len2 > 0.0) {
    t = ((px - ax) * dx + (py - ay) * dy) / len2;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  }
  const double ex = px - (ax + t * dx), ey = py - (ay + t * dy);
  return sqrt(ex * ex + ey * ey);
}

/* tests/oracles.hpp:92-95: distance to the polygon as a region -- zero
 * inside (parity rule), else the smallest edge distance over all rings. */
double orc_point_polygon_distance(double px, double py, const double* vxy,
                                  const uint64_t* ring_off, const uint64_t* poly_ring,
                                  uint64_t poly) {
  if (orc_point_in_polygon(px, py, vxy, ring_off, poly_ring, poly)) return 0.0;
  double best = INFINITY;
  for (uint64_t r = poly_ring[poly]; r < poly_ring[poly + 1]; ++r) {
    const uint64_t b = ring_off[r], n = ring_off[r + 1] - b;
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t a = b + i, c = (i + 1 < n) ? a + 1 : b;
      const double d = seg_distance(px, py, vxy[2 * a], vxy[2 * a + 1], vxy[2 * c], vxy[2 * c + 1]);
      if (d < best) best = d;
    }
  }
  return best;
}
