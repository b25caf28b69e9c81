"""Adversarial polygon soup + points for bit-exactness (shared by CPU and GPU
tests).  The reference tests keep query points >= 1e-9 from every edge
(test_geometry.cpp:113-129, acceptance.cpp:75-107), so nothing there pins
the on-edge tie rule; these cases do: points exactly on vertices, on
horizontal and sloped edges, on shared borders, a hair (1e-12..1e-15) off
edges, NaN/Inf/out-of-world, plus overlapping, self-intersecting, holed,
duplicated-edge and degenerate polygons."""
from __future__ import annotations

import numpy as np

from paper_2005_03156_b200.fastmap import Soup


def polygons():
    P = []
    # 0: unit square at (10, 10) (test_geometry.cpp:12-17 shape, translated)
    P.append([[(10, 10), (11, 10), (11, 11), (10, 11)]])
    # 1: square with a hole (test_geometry.cpp:19-26 shape)
    P.append([[(20, 10), (23, 10), (23, 13), (20, 13)], [(21, 11), (22, 11), (22, 12), (21, 12)]])
    # 2: bow-tie (self-intersecting)
    P.append([[(30, 10), (32, 12), (32, 10), (30, 12)]])
    # 3,4: two overlapping squares (min id wins where both contain)
    P.append([[(40, 10), (42, 10), (42, 12), (40, 12)]])
    P.append([[(41, 11), (43, 11), (43, 13), (41, 13)]])
    # 5,6: two squares sharing an edge (a watertight pair)
    P.append([[(50, 10), (51, 10), (51, 11), (50, 11)]])
    P.append([[(51, 10), (52, 10), (52, 11), (51, 11)]])
    # 7: polygon with a repeated vertex and a zero-length edge
    P.append([[(60, 10), (61, 10), (61, 10), (61, 11), (60, 11)]])
    # 8: polygon that traverses an edge twice (a slit)
    P.append([[(70, 10), (72, 10), (72, 12), (71, 12), (71, 11), (71, 12), (70, 12)]])
    # 9: thin sliver triangle
    P.append([[(80, 10), (81, 10.000000001), (80, 10.000000002)]])
    # 10: star-ish concave polygon with many horizontal edges
    P.append([[(90, 10), (91, 10), (91, 10.5), (92, 10.5), (92, 10), (93, 10), (93, 12),
               (92, 12), (92, 11.5), (91, 11.5), (91, 12), (90, 12)]])
    # 11: nested rings (three concentric squares: even-odd bands)
    P.append([[(100, 0), (106, 0), (106, 6), (100, 6)], [(101, 1), (105, 1), (105, 5), (101, 5)],
              [(102, 2), (104, 2), (104, 4), (102, 4)]])
    # 12: polygon on dyadic coordinates near the world corner
    P.append([[(179.5, 89.5), (180.0, 89.5), (180.0, 90.0), (179.5, 90.0)]])
    # 13: a large polygon containing several others (order matters: id 13 > inner ids)
    P.append([[(5, 5), (125, 5), (125, 20), (5, 20)]])
    # 14: tiny polygon far away (negative coords)
    P.append([[(-120.25, -45.5), (-120.0, -45.5), (-120.125, -45.25)]])
    return P


def build(seed: int = 7):
    P = polygons()
    soup = Soup.from_rings(P)
    rng = np.random.default_rng(seed)
    pts = []
    # every vertex, every edge midpoint, and points nudged around them
    for rings in P:
        for ring in rings:
            r = np.asarray(ring, dtype=np.float64)
            n = len(r)
            for i in range(n):
                a, b = r[i], r[(i + 1) % n]
                pts.append(a)
                pts.append(0.5 * (a + b))
                pts.append(a + 0.25 * (b - a))
                for eps in (1e-15, 1e-12, 1e-9):
                    for dx, dy in ((eps, 0), (-eps, 0), (0, eps), (0, -eps)):
                        pts.append(0.5 * (a + b) + (dx, dy))
                        pts.append(a + (dx, dy))
    # bbox corners and random points over each polygon's bbox
    for rings in P:
        r = np.concatenate([np.asarray(x, dtype=np.float64) for x in rings])
        x0, y0 = r.min(0)
        x1, y1 = r.max(0)
        pts.extend([(x0, y0), (x1, y1), (x0, y1), (x1, y0)])
        u = rng.random((200, 2))
        pts.extend(np.c_[x0 + (x1 - x0) * u[:, 0], y0 + (y1 - y0) * u[:, 1]])
        # points on horizontal lines through vertices (half-open rule)
        for y in np.unique(r[:, 1]):
            for x in np.linspace(x0 - 0.5, x1 + 0.5, 9):
                pts.append((x, y))
    # specials
    pts.extend([(np.nan, 10.5), (10.5, np.nan), (np.inf, 10.5), (10.5, -np.inf),
                (200.0, 10.5), (10.5, 95.0), (-180.0, -90.0), (180.0, 90.0),
                (179.75, 89.75), (180.0, 89.75), (0.0, 0.0)])
    return soup, np.ascontiguousarray(np.asarray(pts, dtype=np.float64))
