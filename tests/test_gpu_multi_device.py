"""The slab and pencil decompositions on REAL separate GPUs over NCCL
(skipped unless the box has >= 2 devices; the leases this project runs on
have one, where tests/test_gpu_slab_virtual.py, test_gpu_pencil_virtual.py
and test_gpu_slab_ipc.py cover the same kernels and schedules).

One process per GPU: the NCCL transport serial and by z chunks (two
streams), the fused transport with its default stream-ordered NCCL barrier
and CUDA-IPC peer mappings, and a 1 x 2 pencil grid; each must be bitwise
equal to the single-GPU propagation.  ADVICE r01: the fused transport's real
cross-GPU path had never run.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                                 reason="needs >= 2 GPUs")]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(n):
    from paper_1309_2451_b200 import qgrid
    from paper_1309_2451_b200.constants import muB, species_mass

    m = species_mass("li6")
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(31)
    a0 = rng.standard_normal(grid.n) + 1j * rng.standard_normal(grid.n)
    return grid, v, a0, m


def _worker(rank, world, port, mode, n, steps, out):
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_1309_2451_b200 import pencil, slab

        grid, v, a0, m = _case(n)
        if mode == "pencil":
            lay = pencil.PencilLayout(grid.n, 1, world, rank)
            rg, cg = pencil.make_groups(1, world)
            vb = torch.from_numpy(np.ascontiguousarray(v[lay.x_slice, lay.y_slice])).cuda()
            prop = pencil.PencilPropagator(grid, vb, m, 1e-6, 1, world, rg, cg)
            psi = torch.from_numpy(np.ascontiguousarray(a0[lay.x_slice, lay.y_slice])).cuda()
        else:
            lay = slab.SlabLayout(grid.n, world, rank)
            transport, chunks = {"nccl": ("nccl", 1), "nccl_chunked": ("nccl", 4), "fused": ("fused", 1)}[mode]
            prop = slab.SlabPropagator(grid, torch.from_numpy(np.ascontiguousarray(v[lay.x_slice])).cuda(), m,
                                       1e-6, transport=transport, chunks=chunks)
            if mode == "fused":
                assert prop.transport == "fused", prop.transport_fallback
            psi = torch.from_numpy(np.ascontiguousarray(a0[lay.x_slice])).cuda()
        prop.advance(psi, steps)
        torch.cuda.synchronize()
        np.save(f"{out}.{rank}.npy", psi.cpu().numpy())
        if hasattr(prop, "close"):
            prop.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["nccl", "nccl_chunked", "fused", "pencil"])
def test_two_gpus_bitwise_equal_one(tmp_path, mode):
    from paper_1309_2451_b200 import propagator, qgrid

    world, n, steps = 2, (64, 32, 64), 6
    out = str(tmp_path / "psi")
    mp.spawn(_worker, args=(world, _port(), mode, n, steps, out), nprocs=world, join=True)
    grid, v, a0, m = _case(n)
    ref, _ = propagator.evolve_real(qgrid.Wavefunction(a0.copy(), grid), propagator.make_plan(grid, v, m, 1e-6),
                                    steps)
    ref = ref.amplitudes
    if mode == "pencil":
        got = np.concatenate([np.load(f"{out}.{r}.npy") for r in range(world)], axis=1)
    else:
        got = np.concatenate([np.load(f"{out}.{r}.npy") for r in range(world)], axis=0)
    assert np.array_equal(got, ref)
