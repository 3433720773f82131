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


@dataclass(frozen=True, eq=False)
class PotentialGrid:
    """Mirror of magfield.PotentialGrid (magfield.py:157-176): `values` is the
    device tensor; `minima` is filled only when the reference's host minima
    search is importable (out of the GPU scope)."""

    values: torch.Tensor
    grid: object
    layout: object
    minima: tuple = None

    def host_values(self) -> np.ndarray:
        return _device.to_host(self.values)


def assemble_potential(layout, grid, segments=None, with_minima: bool = False) -> PotentialGrid:
    """assemble_potential (magfield.py:218-241) with V computed on the device.

    `layout` is a reference ChipLayout or a ChipSegments."""
    chip = layout if isinstance(layout, ChipSegments) else ChipSegments.from_layout(layout, segments)
    values = potential_values(chip, grid)
    minima = None
    if with_minima:
        from ctapsim.magfield import _find_slice_minima  # reference host bookkeeping

        v = _device.to_host(values)
        minima = tuple(_find_slice_minima(v[:, :, iz], grid.x, grid.y) for iz in range(grid.n[2]))
    return PotentialGrid(values=values, grid=grid, layout=layout, minima=minima)
