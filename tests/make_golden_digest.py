"""sha256 of a polygon soup (guards the golden fixtures against generator drift)."""
import hashlib

import numpy as np


def digest(soup) -> str:
    h = hashlib.sha256()
    for a in (soup.vxy, soup.ring_off, soup.poly_ring):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
