"""Slab decomposition kernels on one GPU: P virtual ranks in one process.

Each virtual rank owns a ctap plan with slab_p = P, slab_r = r (its own x-slab
of V and psi, its own send/receive buffers); the all-to-all is emulated by
device copies between the ranks' buffers, and the ranks run one after
another (no kernel waits on another, so this is safe on one GPU).  This
exercises the peer-major layouts of the y passes and the y-slab x pass in
csrc/ exactly as the NCCL path uses them; the result must be bitwise equal
to the single-GPU propagation (identical per-line arithmetic).
"""

import numpy as np
import pytest
import torch

from paper_1309_2451_b200 import observables, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass
from paper_1309_2451_b200.propagator import NativePlan
from paper_1309_2451_b200.slab import SlabLayout, segment_schedule

pytestmark = pytest.mark.gpu
M = species_mass("li6")


def _case(n=(32, 16, 32)):
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(11)
    a0 = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    return grid, v, a0


def run_virtual(grid, v, a0, P, steps, tables=0):
    lays = [SlabLayout(grid.n, P, r) for r in range(P)]
    vs = [torch.from_numpy(np.ascontiguousarray(v[l.x_slice])).cuda() for l in lays]
    plans = [NativePlan(grid, vs[r], M, 1e-6, slab_p=P, slab_r=r, phase_tables=tables) for r in range(P)]
    bufs = [{"psi": torch.from_numpy(np.ascontiguousarray(a0[l.x_slice])).cuda().reshape(-1),
             "send": torch.empty(l.points, dtype=torch.complex128, device="cuda"),
             "recv": torch.empty(l.points, dtype=torch.complex128, device="cuda")} for l in lays]
    chunk = lays[0].points // P
    for op in segment_schedule(steps):
        if op[0] == "pass":
            for r in range(P):
                plans[r].run_pass(op[1], bufs[r][op[2]], bufs[r][op[3]])
        else:
            src, dst = op[1], op[2]
            for q in range(P):          # receiver q gets chunk q of every sender p
                for p in range(P):
                    bufs[q][dst][p * chunk:(p + 1) * chunk].copy_(bufs[p][src][q * chunk:(q + 1) * chunk])
    out = torch.cat([b["psi"] for b in bufs]).reshape(grid.n)
    return out.cpu().numpy(), plans, bufs, lays


@pytest.mark.parametrize("P,tables,n", [(2, 0, (32, 16, 32)), (4, 0, (32, 16, 32)), (8, 0, (32, 16, 32)),
                                         (2, 1, (32, 16, 32)), (4, 3, (32, 16, 32)), (4, 0, (256, 16, 16))])
def test_virtual_slabs_bitwise_equal_single_gpu(P, tables, n):
    grid, v, a0 = _case(n)
    got, *_ = run_virtual(grid, v, a0, P, 6, tables)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    plan = propagator.make_plan(grid, v, M, 1e-6, phase_tables=tables)
    psi, _ = propagator.evolve_real(psi, plan, 6)
    assert np.array_equal(got, psi.amplitudes)


def test_virtual_slab_observer_sums():
    grid, v, a0 = _case()
    P = 4
    got, plans, bufs, lays = run_virtual(grid, v, a0, P, 3)
    xb = np.full(grid.n[2], 3.5e-6)
    parts = []
    for r in range(P):
        xs = torch.from_numpy(grid.x[lays[r].x_slice].copy()).cuda()
        b1 = torch.from_numpy(-xb).cuda()
        b2 = torch.from_numpy(xb.copy()).cuda()
        parts.append(plans[r].observe(bufs[r]["psi"], xs, b1, b2, 2))
    tot = parts[0].clone()
    for p in parts[1:]:
        tot += p
    w = qgrid.Wavefunction(got, grid)
    part = observables.GuidePartition(xb1=-xb, xb2=xb, grid_ref=grid)
    dx, dy, dz = grid.spacing
    pops = observables.populations(w, part)
    t = tot.tolist()
    assert np.allclose([t[1] * dy * dx * dz, t[2] * dy * dx * dz, t[3] * dy * dx * dz], pops,
                       rtol=1e-13, atol=1e-300)
    assert t[4] * grid.dvol == pytest.approx(observables.edge_density(w, 2), rel=1e-13)


def test_yslab_kinetic_sums_compose():
    """k^2 sums of the y-slab layout summed over ranks equal the 1-GPU sums."""
    grid, v, a0 = _case()
    P = 2
    single = propagator._aux_plan(grid)
    phi = torch.from_numpy(a0.copy()).cuda()
    ref = single.k2_sums(phi).tolist()
    tot = [0.0, 0.0]
    for r in range(P):
        lay = SlabLayout(grid.n, P, r)
        pl = NativePlan(grid, None, M, 1e-6, slab_p=P, slab_r=r)
        ys = torch.from_numpy(np.ascontiguousarray(a0[:, lay.y_slice, :])).cuda()
        s = pl.k2_sums(ys).tolist()
        tot = [tot[0] + s[0], tot[1] + s[1]]
    assert tot[0] == pytest.approx(ref[0], rel=1e-13)
    assert tot[1] == pytest.approx(ref[1], rel=1e-13)


def run_virtual_fused(grid, v, a0, P, steps, tables=0):
    """The fused transport on one GPU: each virtual rank's y and x passes
    store directly into the other ranks' buffers through the peer tables
    (device addresses on the same GPU instead of NVLink peer mappings)."""
    from paper_1309_2451_b200.slab import segment_schedule_fused

    lays = [SlabLayout(grid.n, P, r) for r in range(P)]
    vs = [torch.from_numpy(np.ascontiguousarray(v[l.x_slice])).cuda() for l in lays]
    plans = [NativePlan(grid, vs[r], M, 1e-6, slab_p=P, slab_r=r, phase_tables=tables) for r in range(P)]
    psi = [torch.from_numpy(np.ascontiguousarray(a0[l.x_slice])).cuda().reshape(-1) for l in lays]
    yslab = [torch.empty(l.points, dtype=torch.complex128, device="cuda") for l in lays]
    peer = [torch.empty(l.points, dtype=torch.complex128, device="cuda") for l in lays]
    for pl in plans:
        pl.set_peer_buffers(0, [b.data_ptr() for b in yslab])
        pl.set_peer_buffers(1, [b.data_ptr() for b in peer])
    for op in segment_schedule_fused(steps):
        if op[0] == "barrier":
            continue  # ranks run one after another: every store has landed
        for r in range(P):
            bufs = {"psi": psi[r], "yslab": yslab[r], "peer": peer[r]}
            plans[r].run_pass(op[1], bufs[op[2]], bufs[op[3]])
    return torch.cat(psi).reshape(grid.n).cpu().numpy()


@pytest.mark.parametrize("P,n", [(2, (32, 16, 32)), (4, (32, 16, 32)), (8, (32, 16, 32)),
                                 (2, (256, 16, 16)), (8, (256, 16, 16)), (4, (512, 8, 16))])
def test_fused_transport_bitwise_equal_single_gpu(P, n):
    """nx = 512 runs the x pass through the warp-per-line ring with TMA stores
    into the peers' buffers; other nx through tile_kernel's peer stores."""
    grid, v, a0 = _case(n)
    got = run_virtual_fused(grid, v, a0, P, 6)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    plan = propagator.make_plan(grid, v, M, 1e-6, phase_tables=0)
    psi, _ = propagator.evolve_real(psi, plan, 6)
    assert np.array_equal(got, psi.amplitudes)


def test_fused_pass_requires_registered_peers():
    grid, v, a0 = _case()
    pl = NativePlan(grid, torch.from_numpy(np.ascontiguousarray(v[:16])).cuda(), M, 1e-6, slab_p=2, slab_r=0)
    x = torch.zeros(16 * 16 * 32, dtype=torch.complex128, device="cuda")
    with pytest.raises(ValueError, match="peer buffers not registered"):
        pl.run_pass(_lib_pass("PASS_Y_FWD_TO_PEERS"), x, x)


def _lib_pass(name):
    from paper_1309_2451_b200 import _lib

    return getattr(_lib, name)


def run_virtual_chunked(grid, v, a0, P, steps, K):
    """The NCCL transport by z chunks (segment_schedule_chunked, chunk-major
    buffers, ctap_pass_zchunk) with the all-to-alls emulated chunk by chunk."""
    from paper_1309_2451_b200.slab import segment_schedule_chunked

    lays = [SlabLayout(grid.n, P, r) for r in range(P)]
    vs = [torch.from_numpy(np.ascontiguousarray(v[l.x_slice])).cuda() for l in lays]
    plans = [NativePlan(grid, vs[r], M, 1e-6, slab_p=P, slab_r=r) for r in range(P)]
    bufs = [{"psi": torch.from_numpy(np.ascontiguousarray(a0[l.x_slice])).cuda().reshape(-1),
             "send": torch.empty(l.points, dtype=torch.complex128, device="cuda"),
             "recv": torch.empty(l.points, dtype=torch.complex128, device="cuda")} for l in lays]
    W = grid.n[2] // K
    csz = lays[0].points // K        # one chunk of a rank's buffer
    blk = csz // P                   # one peer's block inside a chunk
    for op in segment_schedule_chunked(steps, K):
        if op[0] == "pass":
            for r in range(P):
                plans[r].run_pass(op[1], bufs[r][op[2]], bufs[r][op[3]])
        elif op[0] == "cpass":
            _, kind, src, dst, c = op
            for r in range(P):
                s_ = bufs[r]["psi"] if src == "psi" else bufs[r][src][c * csz:(c + 1) * csz]
                d_ = bufs[r]["psi"] if dst == "psi" else bufs[r][dst][c * csz:(c + 1) * csz]
                plans[r].run_pass_zchunk(kind, s_, d_, c * W, W)
        else:
            _, src, dst, c = op
            for q in range(P):
                for p in range(P):
                    bufs[q][dst][c * csz + p * blk:c * csz + (p + 1) * blk].copy_(
                        bufs[p][src][c * csz + q * blk:c * csz + (q + 1) * blk])
    return torch.cat([b["psi"] for b in bufs]).reshape(grid.n).cpu().numpy()


@pytest.mark.parametrize("P,K,n", [(2, 2, (32, 16, 32)), (4, 4, (32, 16, 64)), (2, 4, (512, 8, 64)),
                                   (8, 2, (64, 16, 32))])
def test_virtual_slabs_zchunked_bitwise_equal_single_gpu(P, K, n):
    """The overlapped NCCL transport's chunked passes and per-chunk exchanges
    give bitwise the single-GPU propagation (and the unchunked slab's)."""
    grid, v, a0 = _case(n)
    got = run_virtual_chunked(grid, v, a0, P, 5, K)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    psi, _ = propagator.evolve_real(psi, propagator.make_plan(grid, v, M, 1e-6), 5)
    assert np.array_equal(got, psi.amplitudes)
