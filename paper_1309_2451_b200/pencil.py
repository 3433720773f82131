"""Pencil decomposition of the split-step propagator over a Pr x Pc grid of
GPUs (one process per GPU, torch.distributed over NCCL / NVLink) -- the
layout SURVEY §8(e) names for config 5 (1024 x 1024 x 512).

Rank r = a Pc + b owns, in position space, the (nx/Pr, ny/Pc, nz) block of
x block a and y block b; z is local.  A step needs whole z, y and x lines in
turn, so each 3D FFT transposes twice, inside a row (the Pc ranks of one a)
and inside a column (the Pr ranks of one b):

    [z^-1 V z]  on Zc = [b'][x][y][z']            (z chunk b' of nz/Pc)
    row all-to-all     Zc -> Yb = [b'][x][y'][z']  (y block b' of ny/Pc)
    y           Yb -> Xp = [a'][x][y'][z']         (y block a' of ny/Pr)
    column all-to-all  Xp -> Xr = natural (nx, ny/Pr, nz/Pc)
    [x K x^-1]  on Xr, in place
    column all-to-all  Xr -> Xp ;  y^-1  Xp -> Yb ;  row all-to-all  Yb -> Zc

Every pass reads and writes the exchange buffers in the order the
all-to-all wants (csrc/ctap_passes.cu, PASS_P*), so there is no pack or
unpack sweep; the z pass itself converts natural <-> z-chunked at segment
ends.  Four all-to-alls per step against the slab's two: per GPU
4 (Pc-1)/Pc-ish x 16 N/P bytes, i.e. ~43 % more NVLink traffic than a slab at
2 x 4; the slab stays the default on one node, the pencil is
for P > nx / 8 (a slab's minimum x thickness) or when ny, nz favour it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _lib
from .propagator import REAL_TIME, NativePlan
from .qgrid import as_simgrid


@dataclass(frozen=True)
class PencilLayout:
    """Block sizes of a Pr x Pc pencil decomposition of an (nx, ny, nz) grid."""

    n: tuple
    Pr: int
    Pc: int
    rank: int

    def __post_init__(self):
        nx, ny, nz = self.n
        if self.Pr < 1 or self.Pc < 2:
            raise ValueError(f"a pencil grid needs Pr >= 1 and Pc >= 2, got {self.Pr} x {self.Pc}")
        if nx % self.Pr or ny % self.Pr or ny % self.Pc or nz % (8 * self.Pc):
            raise ValueError(f"grid {self.n} does not split over a {self.Pr} x {self.Pc} pencil grid")
        if not 0 <= self.rank < self.Pr * self.Pc:
            raise ValueError(f"rank {self.rank} out of range for {self.Pr} x {self.Pc} ranks")

    @property
    def a(self) -> int:
        return self.rank // self.Pc

    @property
    def b(self) -> int:
        return self.rank % self.Pc

    @property
    def xa(self) -> int:
        return self.n[0] // self.Pr

    @property
    def yb(self) -> int:
        return self.n[1] // self.Pc

    @property
    def yd(self) -> int:
        return self.n[1] // self.Pr

    @property
    def zc(self) -> int:
        return self.n[2] // self.Pc

    @property
    def x_slice(self) -> slice:
        return slice(self.a * self.xa, (self.a + 1) * self.xa)

    @property
    def y_slice(self) -> slice:
        return slice(self.b * self.yb, (self.b + 1) * self.yb)

    @property
    def block_shape(self) -> tuple:     # position space
        return (self.xa, self.yb, self.n[2])

    @property
    def points(self) -> int:
        return self.xa * self.yb * self.n[2]

    def row_ranks(self) -> list:        # same a: the row all-to-all
        return [self.a * self.Pc + b for b in range(self.Pc)]

    def col_ranks(self) -> list:        # same b: the column all-to-all
        return [a * self.Pc + self.b for a in range(self.Pr)]

    def a2a_bytes_per_step(self, itemsize: int = 16) -> int:
        """Bytes this rank sends per split step (2 row + 2 column transposes)."""
        row = (self.Pc - 1) * self.points // self.Pc
        col = (self.Pr - 1) * self.points // self.Pr
        return 2 * (row + col) * itemsize


def pencil_schedule(n_steps: int):
    """Operations of n merged steps on one rank: ('pass', kind, src, dst) with
    buffers 'psi' (natural block), 'zc', 'yb', 'xp', 'xr', and
    ('a2a', 'row' | 'col', src, dst)."""
    if n_steps <= 0:
        return
    yield ("pass", _lib.PASS_PZ_FIRST, "psi", "zc")
    for j in range(n_steps):
        yield ("a2a", "row", "zc", "yb")
        yield ("pass", _lib.PASS_PY_FWD, "yb", "xp")
        yield ("a2a", "col", "xp", "xr")
        yield ("pass", _lib.PASS_PX_KIN, "xr", "xr")
        yield ("a2a", "col", "xr", "xp")
        yield ("pass", _lib.PASS_PY_INV, "xp", "yb")
        yield ("a2a", "row", "yb", "zc")
        if j < n_steps - 1:
            yield ("pass", _lib.PASS_PZ_MID, "zc", "zc")
        else:
            yield ("pass", _lib.PASS_PZ_LAST, "zc", "psi")


class PencilPropagator:
    """Real- or imaginary-time propagation of one rank's pencil block on its GPU.

    `row_group` / `col_group` are the torch.distributed groups of this rank's
    row and column (every rank must create all groups in the same order;
    `make_groups` does that)."""

    def __init__(self, grid, v_block, mass: float, dt: float, Pr: int, Pc: int, row_group=None,
                 col_group=None, mode: str = REAL_TIME, v_shift: float = 0.0, precision: str = "complex128",
                 rank: int | None = None):
        self.grid = as_simgrid(grid)
        if rank is None:
            rank = dist.get_rank() if dist.is_initialized() else 0
        self.layout = PencilLayout(tuple(self.grid.n), Pr, Pc, rank)
        if tuple(v_block.shape) != self.layout.block_shape:
            raise ValueError(f"local potential shape {tuple(v_block.shape)} != block {self.layout.block_shape}")
        self.row_group, self.col_group = row_group, col_group
        self.v_block = _device.to_device_f64(v_block)
        self.native = NativePlan(self.grid, self.v_block, mass, dt, mode, v_shift=v_shift, slab_p=Pr * Pc,
                                 slab_r=rank, precision=precision, pencil_c=Pc)
        dev, dt_ = self.v_block.device, self.native.torch_dtype
        self.bufs = {k: torch.empty(self.layout.points, dtype=dt_, device=dev) for k in ("zc", "yb", "xp", "xr")}

    def _a2a(self, which: str, src: torch.Tensor, dst: torch.Tensor):
        from .slab import all_to_all_c

        all_to_all_c(dst, src, self.row_group if which == "row" else self.col_group)

    def advance(self, psi_block: torch.Tensor, n_steps: int):
        """n telescoped steps on this rank's block (collective: all ranks call)."""
        if n_steps < 0:
            raise ValueError("n_steps must be >= 0")
        bufs = dict(self.bufs, psi=psi_block.reshape(-1))
        for op in pencil_schedule(n_steps):
            if op[0] == "pass":
                self.native.run_pass(op[1], bufs[op[2]], bufs[op[3]])
            else:
                self._a2a(op[1], bufs[op[2]], bufs[op[3]])

    def observe(self, psi_block: torch.Tensor, xb1=None, xb2=None, margin: int = 2) -> list:
        """Global [sum rho, left, middle, right, edge] (raw sums, rank-ordered)."""
        from .slab import combine_in_rank_order

        xs = _device.to_device_f64(self.grid.x[self.layout.x_slice])
        b1 = None if xb1 is None else _device.to_device_f64(np.asarray(xb1))
        b2 = None if xb2 is None else _device.to_device_f64(np.asarray(xb2))
        local = self.native.observe(psi_block, xs, b1, b2, margin)
        return combine_in_rank_order(local, None).tolist()


def make_groups(Pr: int, Pc: int):
    """(row_group, col_group) of this rank; creates every row and column group
    on every rank in the same order, as torch.distributed requires."""
    rank = dist.get_rank()
    mine = [None, None]
    for a in range(Pr):
        g = dist.new_group([a * Pc + b for b in range(Pc)])
        if rank // Pc == a:
            mine[0] = g
    for b in range(Pc):
        g = dist.new_group([a * Pc + b for a in range(Pr)])
        if rank % Pc == b:
            mine[1] = g
    return mine[0], mine[1]
