"""The fused slab transport end to end across processes: two ranks (processes)
share one GPU, map each other's exchange buffers through CUDA IPC
(ctap_ipc_handle / ctap_ipc_open) exactly as on an NVLink box, and run the
fused schedule.  The cross-rank barrier here is a device synchronize plus a
gloo barrier (no kernel ever waits on another process's kernel, so this is
safe on one GPU); on a multi-GPU box it is a stream-ordered NCCL all-reduce.
The result must be bitwise equal to the single-GPU propagation."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(n=(32, 16, 32)):
    from paper_1309_2451_b200 import qgrid
    from paper_1309_2451_b200.constants import muB, species_mass

    m = species_mass("li6")
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(21)
    a0 = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    return grid, v, a0, m


def _worker(rank, world, port, steps, out, n, barrier_mode="host"):
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_2451_b200 import slab

        grid, v, a0, m = _case(n)
        lay = slab.SlabLayout(grid.n, world, rank)

        def barrier():
            torch.cuda.synchronize()
            dist.barrier()

        graphs = barrier_mode == "flags_graph"
        prop = slab.SlabPropagator(grid, torch.from_numpy(np.ascontiguousarray(v[lay.x_slice])).cuda(), m, 1e-6,
                                   phase_tables=0, transport="fused", graphs=graphs,
                                   barrier=barrier if barrier_mode == "host" else "flags")
        assert prop.transport == "fused", prop.transport_fallback
        psi = torch.from_numpy(np.ascontiguousarray(a0[lay.x_slice])).cuda()
        prop.advance(psi, steps)
        if graphs:  # a second segment replays the captured graph
            prop.advance(psi, steps)
        torch.cuda.synchronize()
        np.save(f"{out}.{rank}.npy", psi.cpu().numpy())
        sums = prop.observe(psi, np.full(grid.n[2], -3.5e-6), np.full(grid.n[2], 3.5e-6), 2)
        np.save(f"{out}.{rank}.sums.npy", np.array(sums))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,barrier_mode", [(2, (32, 16, 32), "host"), (2, (512, 8, 16), "host"),
                                                  (2, (32, 16, 32), "flags"), (2, (512, 8, 16), "flags"),
                                                  (2, (32, 16, 32), "flags_graph"), (2, (512, 8, 16), "flags_graph")])
def test_fused_ipc_two_processes_bitwise(tmp_path, world, n, barrier_mode):
    """n = (512, ...) runs the x pass through the warp-per-line ring, whose TMA
    stores then target the other process's IPC-mapped buffer.  barrier_mode
    "flags": the transport's own stream-ordered barrier (ctap_flag_barrier:
    peer-mapped epoch flags written and awaited by stream memory operations,
    no kernel spins), the default on a multi-GPU box."""
    from paper_1309_2451_b200 import propagator, qgrid

    out = str(tmp_path / "psi")
    mp.spawn(_worker, args=(world, _port(), 5, out, n, barrier_mode), nprocs=world, join=True)
    got = np.concatenate([np.load(f"{out}.{r}.npy") for r in range(world)])
    grid, v, a0, m = _case(n)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    plan = propagator.make_plan(grid, v, m, 1e-6, phase_tables=0)
    psi, _ = propagator.evolve_real(psi, plan, 5)
    if barrier_mode == "flags_graph":  # two segments of 5 (the second a graph replay)
        psi, _ = propagator.evolve_real(psi, plan, 5)
    assert np.array_equal(got, psi.amplitudes)
    s0, s1 = (np.load(f"{out}.{r}.sums.npy") for r in range(world))
    assert np.array_equal(s0, s1)  # rank-ordered combination: identical on every rank
    assert s0[0] * grid.dvol == pytest.approx(psi.norm(), rel=1e-13)


def _fallback_worker(rank, world, port, out, fail_rank):
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_2451_b200 import slab

        if rank == fail_rank:
            def refuse(handle):
                raise RuntimeError("peer mapping refused (test)")
            slab.open_ipc = refuse
        grid, v, a0, m = _case()
        lay = slab.SlabLayout(grid.n, world, rank)
        prop = slab.SlabPropagator(grid, torch.from_numpy(np.ascontiguousarray(v[lay.x_slice])).cuda(), m, 1e-6,
                                   phase_tables=0, transport="fused")
        with open(f"{out}.{rank}.txt", "w") as fh:
            fh.write(f"{prop.transport}\n{prop.transport_fallback}\n{prop.send.numel()}")
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [0, 1])
def test_fused_transport_falls_back_on_every_rank(tmp_path, fail_rank):
    """One rank cannot map its peer's buffers: every rank (not just that one)
    agrees on the NCCL all-to-all transport, so no rank is left waiting in a
    collective the others never reach; the reason names the failing rank."""
    out = str(tmp_path / "tr")
    mp.spawn(_fallback_worker, args=(2, _port(), out, fail_rank), nprocs=2, join=True)
    for r in range(2):
        transport, why, n = open(f"{out}.{r}.txt").read().split("\n")
        assert transport == "nccl"
        assert int(n) == 16 * 16 * 32
        if r == fail_rank:
            assert "peer mapping refused" in why and f"rank {fail_rank}" in why
        else:
            assert why != "None"
