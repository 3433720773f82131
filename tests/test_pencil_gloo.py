"""Pencil decomposition on CPU: Pr x Pc = 2 x 2 and 1 x 2 ranks over gloo.

The real schedule (paper_1309_2451_b200.pencil.pencil_schedule), the real
row / column sub-communicators (make_groups) and the all-to-all convention
(torch.distributed.all_to_all_single on the exchange buffers) run as on the
GPUs; only the pass kernels are emulated in numpy (tests/pencil_emulator.py).
The result must equal the single-process oracle.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import split_step as orc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    m = orc.MASSES["li6"]
    g = orc.Grid((16, 8, 32), (20e-6, 4e-6, 250e-6), (-10e-6, 0.25e-6, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = g.meshgrid()
    v = orc.MUB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                        + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(8)
    a0 = rng.standard_normal(g.n) + 1j * rng.standard_normal(g.n)
    return g, v, m, a0


def _worker(rank, Pr, Pc, port, steps, out):
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=Pr * Pc)
    try:
        from paper_1309_2451_b200 import pencil
        from pencil_emulator import EmulatedPencilRank

        g, v, m, a0 = _case()
        f = orc.make_factors(g, v, m, 1e-6)
        lay = pencil.PencilLayout(g.n, Pr, Pc, rank)
        row, col = pencil.make_groups(Pr, Pc)
        emu = EmulatedPencilRank(lay, f)
        bufs = {k: np.zeros(lay.points, complex) for k in ("zc", "yb", "xp", "xr")}
        bufs["psi"] = a0[lay.x_slice, lay.y_slice].reshape(-1).copy()
        for op in pencil.pencil_schedule(steps):
            if op[0] == "pass":
                emu.run_pass(op[1], bufs[op[2]], bufs[op[3]])
            else:
                _, which, s, d = op
                src = torch.view_as_real(torch.from_numpy(bufs[s])).contiguous()
                dst = torch.empty_like(src)
                dist.all_to_all_single(dst, src, group=row if which == "row" else col)
                bufs[d][:] = torch.view_as_complex(dst).numpy()
        blocks = [torch.empty(lay.points * 2, dtype=torch.float64) for _ in range(Pr * Pc)]
        dist.all_gather(blocks, torch.view_as_real(torch.from_numpy(bufs["psi"])).reshape(-1).clone())
        if rank == 0:
            full = np.empty(g.n, complex)
            for r, b in enumerate(blocks):
                lr = pencil.PencilLayout(g.n, Pr, Pc, r)
                full[lr.x_slice, lr.y_slice] = torch.view_as_complex(b.reshape(-1, 2)).numpy().reshape(lr.block_shape)
            np.save(out, full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Pr,Pc", [(2, 2), (1, 2)])
def test_pencil_schedule_matches_oracle(tmp_path, Pr, Pc):
    steps = 4
    out = str(tmp_path / "psi.npy")
    mp.spawn(_worker, args=(Pr, Pc, _free_port(), steps, out), nprocs=Pr * Pc, join=True)
    got = np.load(out)
    g, v, m, a0 = _case()
    ref = orc.advance(a0.copy(), orc.make_factors(g, v, m, 1e-6), steps)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13


def test_pencil_layout_and_schedule():
    from paper_1309_2451_b200 import _lib
    from paper_1309_2451_b200.pencil import PencilLayout, pencil_schedule

    lay = PencilLayout((1024, 1024, 512), 2, 4, 6)   # config 5 on a 2 x 4 grid
    assert (lay.a, lay.b) == (1, 2)
    assert lay.block_shape == (512, 256, 512)
    assert (lay.yd, lay.zc) == (512, 128)
    assert lay.row_ranks() == [4, 5, 6, 7] and lay.col_ranks() == [2, 6]
    # 2 row + 2 column transposes
    pts = 512 * 256 * 512
    assert lay.a2a_bytes_per_step() == 2 * (3 * pts // 4 + pts // 2) * 16
    with pytest.raises(ValueError, match="does not split"):
        PencilLayout((16, 16, 16), 2, 4, 0)        # nz < 8 Pc
    with pytest.raises(ValueError, match="out of range"):
        PencilLayout((16, 16, 32), 2, 2, 4)
    assert list(pencil_schedule(0)) == []
    ops = list(pencil_schedule(3))
    assert ops[0] == ("pass", _lib.PASS_PZ_FIRST, "psi", "zc")
    assert ops[-1] == ("pass", _lib.PASS_PZ_LAST, "zc", "psi")
    assert sum(1 for o in ops if o[0] == "a2a") == 12
    assert sum(1 for o in ops if o[0] == "pass" and o[1] == _lib.PASS_PZ_MID) == 2
