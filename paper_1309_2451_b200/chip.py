"""The three-wire chip as the potential kernel's input: segment arrays of the
reference's two shipped chips, generated on the product side.

The reference builds them in host code that is out of this build's scope
(`chipgeom`, reused unchanged): the raised-cosine centerlines and
`discretize_merged` (/root/reference/pkg/src/ctapsim/chipgeom.py:41-141,
174-222), the config files' `value unit` products (config.py:263-298) and the
segment concatenation of `assemble_potential` (magfield.py:229-235).  This
module restates exactly that arithmetic (same numpy calls, same operation
order), so a GPU run needs neither the reference package nor any test
fixture for its geometry; tests/test_chip.py checks the arrays bit for bit
against the ones the reference itself produced (tests/golden/segments_*.npz).

Where ctapsim is importable, `magfield.ChipSegments.from_layout` takes any
reference `ChipLayout` instead.
"""

from __future__ import annotations

import numpy as np

from .constants import muB, species_mass
from .magfield import ChipSegments

# cfg/paper.cfg and cfg/scaled.cfg: (magnitude, unit scale) as the config
# parser multiplies them (config.py:24-32, :298); keys absent from the files
# take the ChipConfig defaults (segment_length 0.125 um, g_f_m_f from file).
_UM, _A, _T, _HZ = 1e-6, 1.0, 1.0, 1.0
CHIPS = {
    "paper": dict(d0=(7, _UM), d_min=(4.3, _UM), bump_half_width=(300, _UM), xi=(50, _UM), z_pad=(500, _UM),
                  x_span=(20, _UM), z_max=(1000, _UM), i_left=(0.1, _A), i_middle=(0.07, _A), i_right=(0.1, _A),
                  b_bias=(0.014, _T), b_ioffe=(0.03, _T), f_z=(5, _HZ), g_f_m_f=0.5),
    "scaled": dict(d0=(7, _UM), d_min=(4.3, _UM), bump_half_width=(75, _UM), xi=(12.5, _UM), z_pad=(125, _UM),
                   x_span=(20, _UM), z_max=(250, _UM), i_left=(0.02, _A), i_middle=(0.014, _A),
                   i_right=(0.02, _A), b_bias=(1.964e-3, _T), b_ioffe=(0.03, _T), f_z=(20, _HZ), g_f_m_f=0.5),
}
SEGMENT_LENGTH = 0.125e-6


def _raised_cosine(base, depth, center, half_width, z):
    """chipgeom.py:49-53"""
    z = np.asarray(z, float)
    u = (z - center) / half_width
    bump = np.where(np.abs(u) < 1.0, 0.5 * (1.0 + np.cos(np.pi * u)), 0.0)
    return base - np.sign(base) * depth * bump


def _sample(z_lo, z_hi, seg_len):
    """chipgeom.py:99-101"""
    n = max(1, int(round((z_hi - z_lo) / seg_len)))
    return np.linspace(z_lo, z_hi, n + 1)


def _discretize_merged(x_of_z, curved, z_lo, z_hi, seg_len):
    """chipgeom.py:119-141: straight spans collapse to single segments."""
    spans = [s for s in curved if s[1] > z_lo and s[0] < z_hi]
    zs = [np.array([z_lo])]
    cursor = z_lo
    for lo, hi in sorted(spans):
        lo, hi = max(lo, z_lo), min(hi, z_hi)
        if lo > cursor:
            zs.append(np.array([lo]))
        zs.append(_sample(lo, hi, seg_len)[1:])
        cursor = hi
    if cursor < z_hi:
        zs.append(np.array([z_hi]))
    z = np.concatenate(zs)
    x = np.asarray(x_of_z(z), float)
    pts = np.column_stack([x, np.zeros_like(z), z])
    return pts[:-1], pts[1:]


def chip_segments(name: str = "paper", ordering: str = "counter_intuitive",
                  i_middle: float | None = None) -> ChipSegments:
    """ChipSegments of the reference chip `name` ("paper" or "scaled")."""
    if name not in CHIPS:
        raise ValueError(f"unknown chip {name!r} (known: {sorted(CHIPS)})")
    if ordering not in ("counter_intuitive", "intuitive"):
        raise ValueError(f"unknown ordering {ordering!r}")
    c = {k: (v[0] * v[1] if isinstance(v, tuple) else v) for k, v in CHIPS[name].items()}
    if i_middle is not None:
        c["i_middle"] = float(i_middle)
    d0, z_max, xi, hw = c["d0"], c["z_max"], c["xi"], c["bump_half_width"]
    depth = d0 - c["d_min"]                      # chipgeom.py:176-188
    zc_first = z_max / 2 - xi / 2
    zc_second = z_max / 2 + xi / 2
    if ordering == "counter_intuitive":
        zc_right, zc_left = zc_first, zc_second
    else:
        zc_right, zc_left = zc_second, zc_first
    z_lo, z_hi = -c["z_pad"], z_max + c["z_pad"]
    wires = [  # LEFT, MIDDLE, RIGHT: the dict order assemble_potential concatenates
        (lambda z: _raised_cosine(-d0, depth, zc_left, hw, z), ((zc_left - hw, zc_left + hw),), c["i_left"]),
        (lambda z: np.full_like(np.asarray(z, float), 0.0), (), c["i_middle"]),
        (lambda z: _raised_cosine(+d0, depth, zc_right, hw, z), ((zc_right - hw, zc_right + hw),), c["i_right"]),
    ]
    segs = [(*_discretize_merged(f, spans, z_lo, z_hi, SEGMENT_LENGTH), cur) for f, spans, cur in wires]
    seg_a = np.concatenate([a for a, _, _ in segs])
    seg_b = np.concatenate([b for _, b, _ in segs])
    seg_cur = np.concatenate([np.full(len(a), cur) for a, _, cur in segs])
    e = np.asarray((1.0, 0.0, 0.0), float)       # bias_direction (magfield.py:233-235)
    e = e / np.linalg.norm(e)
    b0 = c["b_bias"] * e + np.array([0.0, 0.0, c["b_ioffe"]])
    return ChipSegments(seg_a, seg_b, seg_cur, b0, c["g_f_m_f"] * muB, species_mass("li6"),
                        2 * np.pi * c["f_z"], z_max, c["x_span"])
