"""Chip-wire trapping potential on the B200 (drop-in for the kernel part of
ctapsim.magfield: magfield.py:107-144 and the validation/assembly of
assemble_potential, magfield.py:218-241).

V is evaluated once per (layout, grid) by ctap_potential, which is
bit-identical to the reference's numba kernel, and stays resident in HBM for
the propagator (north_star item 1).  The wire geometry itself (chipgeom) is
host-side bookkeeping: a ChipSegments carries the concatenated segment arrays
in the reference's order (LEFT, MIDDLE, RIGHT; discretize_merged order), built
either from a reference ChipLayout or from stored arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .constants import mu0

MU0_4PI = mu0 / (4.0 * np.pi)  # magfield.py:31


@dataclass(frozen=True, eq=False)
class ChipSegments:
    """Concatenated straight segments and trap constants of one chip layout."""

    seg_a: np.ndarray      # (n, 3) m
    seg_b: np.ndarray      # (n, 3) m
    seg_cur: np.ndarray    # (n,) A
    b0: np.ndarray         # bias + Ioffe field (3,) T  (magfield.py:233-235)
    mu_eff: float          # J/T
    mass: float            # kg
    omega_z: float         # rad/s
    z_max: float           # m
    x_span: float          # m

    @property
    def z_center(self) -> float:
        return self.z_max / 2.0

    @classmethod
    def from_arrays(cls, d) -> "ChipSegments":
        return cls(seg_a=np.asarray(d["seg_a"], float), seg_b=np.asarray(d["seg_b"], float),
                   seg_cur=np.asarray(d["seg_cur"], float), b0=np.asarray(d["b0"], float),
                   mu_eff=float(d["mu_eff"]), mass=float(d["mass"]), omega_z=float(d["omega_z"]),
                   z_max=float(d["z_max"]), x_span=float(d["x_span"]))

    @classmethod
    def from_layout(cls, layout, segments=None) -> "ChipSegments":
        """From a reference ChipLayout.  `segments` is the list of per-wire
        Segments (a, b, current); by default the reference's own
        discretize_merged is used (importable wherever ctapsim is)."""
        if segments is None:
            from ctapsim.chipgeom import discretize_merged  # reference host geometry

            segments = [discretize_merged(w) for w in layout.wires.values()]
        seg_a = np.concatenate([s.a for s in segments])
        seg_b = np.concatenate([s.b for s in segments])
        seg_cur = np.concatenate([np.full(len(s), s.current) for s in segments])
        e = np.asarray(layout.bias_direction, float)
        e = e / np.linalg.norm(e)
        b0 = layout.b_bias * e + np.array([0.0, 0.0, layout.b_ioffe])
        return cls(seg_a, seg_b, seg_cur, b0, float(layout.mu_eff), float(layout.mass),
                   float(layout.omega_z), float(layout.z_max), float(layout.x_span))


def validate_grid(chip: ChipSegments, grid):
    """The checks of assemble_potential (magfield.py:221-228)."""
    ys = grid.axis(1) if hasattr(grid, "axis") else grid.y
    if np.any(np.abs(ys) < 1e-9):
        raise ValueError("grid intersects the wire plane y = 0; offset the y origin")
    if (grid.origin[0] < -chip.x_span / 2 - 1e-12
            or grid.origin[0] + grid.extents[0] > chip.x_span / 2 + 1e-12
            or grid.origin[2] < -1e-12
            or grid.origin[2] + grid.extents[2] > chip.z_max + 1e-12):
        raise ValueError("grid extends beyond the layout extents")


def potential_on_axes(chip: ChipSegments, xs, ys, zs) -> torch.Tensor:
    """V(x, y, z) on the product of three axis arrays, as a CUDA float64 tensor
    of shape (len(xs), len(ys), len(zs)).  Bit-identical to _potential_kernel."""
    dev = _device.require_cuda()
    lib = _lib.load()
    xs_d, ys_d, zs_d = (_device.to_device_f64(np.asarray(a, float)) for a in (xs, ys, zs))
    a_d = _device.to_device_f64(chip.seg_a.reshape(-1, 3))
    b_d = _device.to_device_f64(chip.seg_b.reshape(-1, 3))
    c_d = _device.to_device_f64(chip.seg_cur.reshape(-1))
    out = torch.empty((xs_d.numel(), ys_d.numel(), zs_d.numel()), dtype=torch.float64, device=dev)
    _lib.check(lib.ctap_potential(
        xs_d.data_ptr(), xs_d.numel(), ys_d.data_ptr(), ys_d.numel(), zs_d.data_ptr(), zs_d.numel(),
        a_d.data_ptr(), b_d.data_ptr(), c_d.data_ptr(), c_d.numel(),
        float(chip.b0[0]), float(chip.b0[1]), float(chip.b0[2]), chip.mu_eff, chip.mass,
        chip.omega_z, chip.z_center, MU0_4PI, out.data_ptr(), _device.stream_handle()))
    return out


def potential_values(chip: ChipSegments, grid, x_slice=None) -> torch.Tensor:
    """V on `grid` (or on the x-planes `x_slice` of it, for a slab rank)."""
    validate_grid(chip, grid)
    xs = grid.axis(0) if hasattr(grid, "axis") else grid.x
    if x_slice is not None:
        xs = xs[x_slice]
    ys = grid.axis(1) if hasattr(grid, "axis") else grid.y
    zs = grid.axis(2) if hasattr(grid, "axis") else grid.z
    return potential_on_axes(chip, xs, ys, zs)


class MinimumAbsentError(LookupError):
    """The requested guide has no distinct transverse minimum (merged guides)."""


@dataclass(frozen=True)
class SliceMinima:
    """Transverse minima of one z slice sorted by x, NaN padded to 3
    (magfield.py:145-152)."""

    x: np.ndarray       # (3,)
    y: np.ndarray       # (3,)
    value: np.ndarray   # (3,) J
    n_guides: int


def _refine(v_lo, v_mid, v_hi):
    # parabolic vertex through three samples (magfield.py:180-186)
    curv = v_lo - 2.0 * v_mid + v_hi
    if curv <= 0:
        return 0.0, 0.0
    diff = v_lo - v_hi
    return 0.5 * diff / curv, -0.125 * diff ** 2 / curv


def slice_minima(values: torch.Tensor, grid) -> tuple:
    """Per-z-slice transverse minima of V, as assemble_potential's
    _find_slice_minima loop (magfield.py:188-208, :239-240).

    The scan over every interior point of every slice (and the selection of
    the three lowest minima) runs on the device (ctap_slice_minima); only
    the <= 3 winners per slice and their 4-neighbours come back to the host
    for the parabolic refinement, in the reference's float64 expressions.
    Ties in V between a 3rd and 4th minimum are broken by row-major index
    (numpy's argsort agrees for up to 16 minima per slice)."""
    v = _device.to_device_f64(values)
    nx, ny, nz = v.shape
    count = torch.empty(nz, dtype=torch.int64, device=v.device)
    best = torch.empty(3 * nz, dtype=torch.int64, device=v.device)
    _lib.call("ctap_slice_minima", v.data_ptr(), nx, ny, nz, count.data_ptr(), best.data_ptr(),
              _device.stream_handle())
    best = best.view(nz, 3)
    sel = best.clamp(min=0)
    i, j = sel // ny, sel % ny
    zz = torch.arange(nz, device=v.device)[:, None].expand(nz, 3)
    # the 5-point stencil around each selected point (clamped for padding)
    st = torch.stack([v[i, j, zz], v[(i - 1).clamp(min=0), j, zz], v[(i + 1).clamp(max=nx - 1), j, zz],
                      v[i, (j - 1).clamp(min=0), zz], v[i, (j + 1).clamp(max=ny - 1), zz]])
    st, count, best = (_device.to_host(t) for t in (st, count, best))
    xs = np.asarray(grid.axis(0) if hasattr(grid, "axis") else grid.x)
    ys = np.asarray(grid.axis(1) if hasattr(grid, "axis") else grid.y)
    hx, hy = xs[1] - xs[0], ys[1] - ys[0]
    out = []
    for k in range(nz):
        kept = [m for m in range(3) if best[k, m] >= 0]
        if count[k] <= 3:  # all minima kept, in the reference's row-major order
            kept.sort(key=lambda m: best[k, m])
        res = np.full((3, 3), np.nan)
        # x order; Python's sort is stable like numpy's argsort on <= 3 items
        for slot, m in enumerate(sorted(kept, key=lambda m: xs[best[k, m] // ny])):
            a, b = divmod(int(best[k, m]), ny)
            vc, vxm, vxp, vym, vyp = (st[q, k, m] for q in range(5))
            ox, dvx = _refine(vxm, vc, vxp)
            oy, dvy = _refine(vym, vc, vyp)
            res[0, slot] = xs[a] + ox * hx
            res[1, slot] = ys[b] + oy * hy
            res[2, slot] = vc + dvx + dvy
        out.append(SliceMinima(res[0].copy(), res[1].copy(), res[2].copy(), len(kept)))
    return tuple(out)


@dataclass(frozen=True, eq=False)
class PotentialGrid:
    """Mirror of magfield.PotentialGrid (magfield.py:155-176): `values` is the
    device tensor; `minima` holds one SliceMinima per z slice (device scan,
    slice_minima)."""

    values: torch.Tensor
    grid: object
    layout: object
    minima: tuple = None

    def host_values(self) -> np.ndarray:
        return _device.to_host(self.values)

    def slice_minima(self, iz: int) -> SliceMinima:
        return self.minima[iz]

    def guide_minimum(self, iz: int, guide_index: int):
        """(x, y, V) of guide 0/1/2 in slice iz (magfield.py:164-176)."""
        m = self.minima[iz]
        if guide_index >= max(m.n_guides, 0):
            raise MinimumAbsentError(
                f"slice {iz} has {m.n_guides} transverse minima (guides merged); "
                f"guide {guide_index} absent")
        return float(m.x[guide_index]), float(m.y[guide_index]), float(m.value[guide_index])


def assemble_potential(layout, grid, segments=None, with_minima: bool = True) -> PotentialGrid:
    """assemble_potential (magfield.py:218-241) with V and the per-slice
    minima scan computed on the device.

    `layout` is a reference ChipLayout or a ChipSegments."""
    chip = layout if isinstance(layout, ChipSegments) else ChipSegments.from_layout(layout, segments)
    values = potential_values(chip, grid)
    minima = slice_minima(values, grid) if with_minima else None
    return PotentialGrid(values=values, grid=grid, layout=layout, minima=minima)
