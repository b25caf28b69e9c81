"""Margin-scale exactness cases.

The index classifies every polygon edge against each cell's latitude slab
widened by the margin d = 2^-40 * max(1, |coords|) and evaluates only the
"near" edges exactly; the point's cell comes from the kernel's
(p - g0) * inv truncation while the builder forms cell rectangles as
g0 + i * w.  This module builds soups whose vertices and edges sit at
{0, +-0.5, +-1, +-2, +-4} * d from cell borders of a known grid, and points
at +-k ulps of those borders, exactly on vertices, on edges and at 1e-9 ..
1e-13 cell widths from edges -- the scale at which the margin argument is
tight.  The grid is pinned by a frame polygon spanning the domain (the last
leaf id, so every interior polygon takes precedence), so the cell borders
the cases are built against are the ones the builder uses
(index_host.cpp plan_grid: g0 = min - 4d, w = (max - min + 8d) / n).
Expected answers come from the CPU oracle's exhaustive_assign
(synthetic.hpp:193-205)."""
import math

import numpy as np

from paper_2005_03156_b200 import fastmap

X0, X1, Y0, Y1 = -125.0, -66.0, 24.0, 50.0
KS = (0.0, 0.5, -0.5, 1.0, -1.0, 2.0, -2.0, 4.0, -4.0)


def grid_geom(nx: int, ny: int) -> dict:
    """The builder's grid for a union bbox [X0, X1] x [Y0, Y1] (plan_grid)."""
    m = max(abs(X0), abs(X1), abs(Y0), abs(Y1), 1.0)
    d = math.ldexp(m, -40)
    gx0, gx1, gy0, gy1 = X0 - 4 * d, X1 + 4 * d, Y0 - 4 * d, Y1 + 4 * d
    return {"d": d, "gx0": gx0, "gy0": gy0, "w": (gx1 - gx0) / nx, "h": (gy1 - gy0) / ny,
            "nx": nx, "ny": ny}


def _ulps(v: float, k: int) -> float:
    for _ in range(abs(k)):
        v = float(np.nextafter(v, math.inf if k > 0 else -math.inf))
    return v


def build(nx: int, ny: int, n_polys: int = 160, seed: int = 0):
    """(soup, points, geometry) for a grid of nx x ny cells."""
    g = grid_geom(nx, ny)
    d, w, h = g["d"], g["w"], g["h"]
    rng = np.random.default_rng(seed + 1000 * nx + ny)

    def xb(i):  # cell border exactly as the builder forms it (cell_x0)
        return g["gx0"] + float(i) * w

    def yb(j):
        return g["gy0"] + float(j) * h

    def k():
        return float(KS[rng.integers(len(KS))])

    rings = []
    for p in range(n_polys):
        ix = int(rng.integers(2, nx - 3))
        iy = int(rng.integers(2, ny - 3))
        kind = p % 5
        if kind == 0:  # axis-aligned rectangle, every side at border + k d
            x0, x1 = xb(ix) + k() * d, xb(ix + 1 + int(rng.integers(0, 2))) + k() * d
            y0, y1 = yb(iy) + k() * d, yb(iy + 1 + int(rng.integers(0, 2))) + k() * d
            ring = [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]
        elif kind == 1:  # slanted quad, vertices on borders + k d
            ring = [(xb(ix) + k() * d, yb(iy) + rng.uniform(0.1, 0.9) * h),
                    (xb(ix) + rng.uniform(0.1, 0.9) * w, yb(iy) + k() * d),
                    (xb(ix + 1) + k() * d, yb(iy) + rng.uniform(0.1, 0.9) * h),
                    (xb(ix) + rng.uniform(0.1, 0.9) * w, yb(iy + 1) + k() * d)]
        elif kind == 2:  # triangle with a vertex at a cell corner + (k d, k d)
            cx, cy = xb(ix + 1) + k() * d, yb(iy + 1) + k() * d
            ring = [(cx, cy), (cx - rng.uniform(0.3, 1.7) * w, cy - rng.uniform(0.1, 0.5) * h),
                    (cx - rng.uniform(0.1, 0.5) * w, cy - rng.uniform(0.3, 1.7) * h)]
        elif kind == 3:  # sliver of width a few d along a vertical border
            xa = xb(ix + 1) + k() * d
            wd = float(rng.choice([0.5, 1.0, 2.0, 4.0])) * d
            ya, yz = yb(iy) + rng.uniform(-0.5, 0.5) * h, yb(iy + 2) + rng.uniform(-0.5, 0.5) * h
            ring = [(xa, ya), (xa + wd, ya), (xa + wd, yz), (xa, yz)]
        else:  # sliver along a horizontal border, plus a nearly flat edge
            ya = yb(iy + 1) + k() * d
            hd = float(rng.choice([0.5, 1.0, 2.0, 4.0])) * d
            xa, xz = xb(ix) + rng.uniform(-0.5, 0.5) * w, xb(ix + 2) + rng.uniform(-0.5, 0.5) * w
            ring = [(xa, ya), (xz, ya + k() * d), (xz, ya + hd), (xa, ya + hd)]
        rings.append(np.array(ring, dtype=np.float64))
    frame = np.array([(X0, Y0), (X1, Y0), (X1, Y1), (X0, Y1)], dtype=np.float64)
    soup = fastmap.Soup.from_rings([[r] for r in rings] + [[frame]])

    pts = []
    for r in rings:
        nv = len(r)
        for a in range(nv):
            vx, vy = float(r[a, 0]), float(r[a, 1])
            bx, by = float(r[(a + 1) % nv, 0]), float(r[(a + 1) % nv, 1])
            for dx in (-2, -1, 0, 1, 2):  # on and ulps around every vertex
                for dy in (-1, 0, 1):
                    pts.append((_ulps(vx, dx), _ulps(vy, dy)))
            for t in (0.5, 0.25, 1.0 / 3.0):  # on the edge (up to rounding)
                pts.append((vx + t * (bx - vx), vy + t * (by - vy)))
            ex, ey = bx - vx, by - vy
            ln = math.hypot(ex, ey)
            if ln > 0:
                for off in (1e-9, 1e-10, 1e-11, 1e-12, 1e-13):
                    for sgn in (1.0, -1.0):
                        s = sgn * off * w / ln
                        mx, my = vx + 0.5 * ex, vy + 0.5 * ey
                        pts.append((mx - s * ey, my + s * ex))
        # cell borders +- k ulps next to the polygon
        cx0 = int((float(r[:, 0].min()) - g["gx0"]) / w)
        cy0 = int((float(r[:, 1].min()) - g["gy0"]) / h)
        for i in range(cx0, cx0 + 3):
            for j in range(cy0, cy0 + 3):
                for du in (-2, -1, 0, 1, 2):
                    pts.append((_ulps(xb(i), du), yb(j) + rng.uniform(0, 1) * h))
                    pts.append((xb(i) + rng.uniform(0, 1) * w, _ulps(yb(j), du)))
                    pts.append((_ulps(xb(i), du), _ulps(yb(j), -du)))
                for _ in range(4):
                    pts.append((xb(i) + rng.uniform(0, 1) * w, yb(j) + rng.uniform(0, 1) * h))
    return soup, np.array(pts, dtype=np.float64), g


def near_edge_points(soup, n: int, cell_w: float, seed: int = 0) -> np.ndarray:
    """Points at 1e-9 .. 1e-13 cell widths from random edges of a soup
    (both sides), and exactly on random vertices."""
    rng = np.random.default_rng(seed)
    v = soup.vxy.reshape(-1, 2)
    ro = soup.ring_off.astype(np.int64)
    ring = rng.integers(0, len(ro) - 1, n)
    a = ro[ring] + (rng.random(n) * (ro[ring + 1] - ro[ring])).astype(np.int64)
    b = np.where(a + 1 < ro[ring + 1], a + 1, ro[ring])
    pa, pb = v[a], v[b]
    e = pb - pa
    ln = np.hypot(e[:, 0], e[:, 1])
    ln[ln == 0] = 1.0
    off = 10.0 ** -rng.integers(9, 14, n) * cell_w * rng.choice([-1.0, 1.0], n)
    t = rng.random(n)
    q = pa + t[:, None] * e + (off / ln)[:, None] * np.stack([-e[:, 1], e[:, 0]], 1)
    on_vertex = rng.random(n) < 0.1
    q[on_vertex] = pa[on_vertex]
    return np.ascontiguousarray(q)
