"""Pencil decomposition kernels on one GPU: Pr x Pc virtual ranks in one process.

Each virtual rank owns a pencil plan (its (nx/Pr, ny/Pc, nz) block of V and
psi and its four exchange buffers); the row and column all-to-alls are
emulated by device copies with torch.distributed.all_to_all_single's chunk
convention, and the ranks run one after another (no kernel waits on another).
This runs the z-chunked z passes, the blocked y passes and the pencil x pass
(warp-per-line ring for nx = 256/512) exactly as the NCCL path does; the
result must be bitwise equal to the single-GPU propagation.
"""

import numpy as np
import pytest
import torch

from paper_1309_2451_b200 import observables, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass
from paper_1309_2451_b200.pencil import PencilLayout, pencil_schedule
from paper_1309_2451_b200.propagator import NativePlan

pytestmark = pytest.mark.gpu
M = species_mass("li6")


def _case(n):
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(13)
    a0 = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    return grid, v, a0


def run_virtual_pencil(grid, v, a0, Pr, Pc, steps, mode=propagator.REAL_TIME):
    P = Pr * Pc
    lays = [PencilLayout(grid.n, Pr, Pc, r) for r in range(P)]
    plans, bufs = [], []
    for lay in lays:
        vb = torch.from_numpy(np.ascontiguousarray(v[lay.x_slice, lay.y_slice])).cuda()
        plans.append(NativePlan(grid, vb, M, 1e-6, mode, slab_p=P, slab_r=lay.rank, pencil_c=Pc))
        b = {k: torch.empty(lay.points, dtype=torch.complex128, device="cuda") for k in ("zc", "yb", "xp", "xr")}
        b["psi"] = torch.from_numpy(np.ascontiguousarray(a0[lay.x_slice, lay.y_slice])).cuda().reshape(-1)
        bufs.append(b)
    for op in pencil_schedule(steps):
        if op[0] == "pass":
            for r in range(P):
                plans[r].run_pass(op[1], bufs[r][op[2]], bufs[r][op[3]])
            continue
        _, which, src, dst = op
        groups = ([lays[0].__class__(grid.n, Pr, Pc, a * Pc).row_ranks() for a in range(Pr)] if which == "row"
                  else [lays[0].__class__(grid.n, Pr, Pc, b).col_ranks() for b in range(Pc)])
        for members in groups:
            G = len(members)
            chunk = lays[0].points // G
            for qi, q in enumerate(members):      # receiver q gets chunk qi of every sender
                for pi, p in enumerate(members):
                    bufs[q][dst][pi * chunk:(pi + 1) * chunk].copy_(bufs[p][src][qi * chunk:(qi + 1) * chunk])
    out = np.empty(grid.n, dtype=np.complex128)
    for lay, b in zip(lays, bufs):
        out[lay.x_slice, lay.y_slice] = b["psi"].reshape(lay.block_shape).cpu().numpy()
    return out, plans, bufs, lays


@pytest.mark.parametrize("Pr,Pc,n", [(2, 2, (32, 16, 32)), (1, 2, (16, 16, 32)), (2, 4, (32, 16, 64)),
                                     (4, 2, (256, 16, 32)), (2, 2, (512, 8, 16))])
def test_virtual_pencils_bitwise_equal_single_gpu(Pr, Pc, n):
    grid, v, a0 = _case(n)
    got, *_ = run_virtual_pencil(grid, v, a0, Pr, Pc, 5)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    plan = propagator.make_plan(grid, v, M, 1e-6, phase_tables=0)
    psi, _ = propagator.evolve_real(psi, plan, 5)
    assert np.array_equal(got, psi.amplitudes)


def test_virtual_pencil_observer_sums():
    """Per-rank observer partials of the pencil blocks (global x and y faces
    for the edge set) sum to the reference observables."""
    n = (32, 16, 32)
    grid, v, a0 = _case(n)
    got, plans, bufs, lays = run_virtual_pencil(grid, v, a0, 2, 2, 3)
    xb = np.full(grid.n[2], 3.5e-6)
    tot = None
    for pl, b, lay in zip(plans, bufs, lays):
        xs = torch.from_numpy(grid.x[lay.x_slice].copy()).cuda()
        s = pl.observe(b["psi"], xs, torch.from_numpy(-xb).cuda(), torch.from_numpy(xb.copy()).cuda(), 2)
        tot = s.clone() if tot is None else tot + s
    w = qgrid.Wavefunction(got, grid)
    part = observables.GuidePartition(xb1=-xb, xb2=xb, grid_ref=grid)
    pops = observables.populations(w, part)
    t = tot.tolist()
    assert np.allclose([t[1] * grid.dvol, t[2] * grid.dvol, t[3] * grid.dvol], pops, rtol=1e-13, atol=1e-300)
    assert t[4] * grid.dvol == pytest.approx(observables.edge_density(w, 2), rel=1e-13)
    assert t[0] * grid.dvol == pytest.approx(w.norm(), rel=1e-13)


def test_pencil_plan_validation():
    grid, v, a0 = _case((32, 16, 32))
    vb = torch.zeros((16, 8, 32), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="pencil grid"):
        NativePlan(grid, torch.zeros((16, 4, 32), dtype=torch.float64, device="cuda"), M, 1e-6, slab_p=8,
                   slab_r=0, pencil_c=8)  # nz = 32 < 8 Pc
    pl = NativePlan(grid, vb, M, 1e-6, slab_p=4, slab_r=1, pencil_c=2)
    x = torch.zeros(16 * 8 * 32, dtype=torch.complex128, device="cuda")
    from paper_1309_2451_b200 import _lib
    with pytest.raises(ValueError, match="pencil"):
        pl.run_pass(_lib.PASS_Z_MID, x, x)
    with pytest.raises(ValueError, match="out of place"):
        pl.run_pass(_lib.PASS_PY_FWD, x, x)
