"""CPU restatement of the reference's transverse-minima scan and guide
partition -- TEST INFRASTRUCTURE ONLY (the checker for the GPU path; never
imported by the product package).

Algorithm of /root/reference/pkg/src/ctapsim:
  magfield.py:180-186   parabolic refinement of a minimum along one axis
  magfield.py:188-208   per-slice minima: interior points strictly below the
                        -x and -y neighbours and not above the +x and +y ones;
                        more than three -> the three lowest (numpy argsort);
                        the kept ones ordered by x, refined, NaN padded to 3;
                        n_guides = number kept (<= 3)
  magfield.py:239-240   one record per z slice (assemble_potential)
  observables.py:35-60  guide boundaries at the floor-profile ridge between
                        adjacent minima; midpoints of the wires if merged
  observables.py:63-69  ridge = argmax of min_y V between the two minima
Pinned against tests/golden/minima.npz, produced by the reference itself
(tests/golden/make_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SliceMinima:
    x: np.ndarray
    y: np.ndarray
    value: np.ndarray
    n_guides: int


def refine(v_lo, v_mid, v_hi):
    """(offset in cells, value change) of the vertex of the parabola through
    three equally spaced samples; zero unless the samples are convex."""
    curv = v_lo - 2.0 * v_mid + v_hi
    if curv <= 0:
        return 0.0, 0.0
    diff = v_lo - v_hi
    return 0.5 * diff / curv, -0.125 * diff ** 2 / curv


def minima_indices(v):
    """Row-major (i, j) of the interior local minima of one (nx, ny) slice."""
    c = v[1:-1, 1:-1]
    mask = (c < v[:-2, 1:-1]) & (c <= v[2:, 1:-1]) & (c < v[1:-1, :-2]) & (c <= v[1:-1, 2:])
    i, j = np.nonzero(mask)
    return i + 1, j + 1


def slice_minima(v, xs, ys, keep=3) -> SliceMinima:
    i, j = minima_indices(v)
    if i.size > keep:
        lowest = np.argsort(v[i, j])[:keep]
        i, j = i[lowest], j[lowest]
    count = int(i.size)  # the reference's n_guides counts the kept minima
    out = np.full((3, 3), np.nan)  # rows: x, y, value
    if count:
        hx, hy = xs[1] - xs[0], ys[1] - ys[0]
        for slot, m in enumerate(np.argsort(xs[i])):
            a, b = i[m], j[m]
            ox, dvx = refine(v[a - 1, b], v[a, b], v[a + 1, b])
            oy, dvy = refine(v[a, b - 1], v[a, b], v[a, b + 1])
            out[0, slot] = xs[a] + ox * hx
            out[1, slot] = ys[b] + oy * hy
            out[2, slot] = v[a, b] + dvx + dvy
    return SliceMinima(out[0].copy(), out[1].copy(), out[2].copy(), count)


def all_slice_minima(values, xs, ys):
    return tuple(slice_minima(values[:, :, k], xs, ys) for k in range(values.shape[2]))


def ridge(profile, xs, x_a, x_b):
    lo = int(np.searchsorted(xs, x_a))
    hi = int(np.searchsorted(xs, x_b))
    if hi <= lo + 1:
        return 0.5 * (x_a + x_b)
    return float(xs[lo + int(np.argmax(profile[lo:hi + 1]))])


def build_partition(values, minima, xs, wire_positions):
    """wire_positions[k] = the three wire x positions at slice k
    (layout.wire_positions_at), used where fewer than three minima exist."""
    nz = values.shape[2]
    floor = values.min(axis=1)
    xb = np.empty((2, nz))
    merged = np.zeros(nz, dtype=bool)
    for k in range(nz):
        m = minima[k]
        if m.n_guides >= 3:
            xb[0, k] = ridge(floor[:, k], xs, m.x[0], m.x[1])
            xb[1, k] = ridge(floor[:, k], xs, m.x[1], m.x[2])
        else:
            merged[k] = True
            w = sorted(wire_positions[k])
            xb[0, k] = 0.5 * (w[0] + w[1])
            xb[1, k] = 0.5 * (w[1] + w[2])
    return xb[0].copy(), xb[1].copy(), merged
