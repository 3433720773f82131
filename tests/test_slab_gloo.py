"""Multi-rank slab decomposition on CPU: world_size 2 and 4 over gloo.

The real schedule (paper_1309_2451_b200.slab.segment_schedule), the real
all-to-all convention (torch.distributed.all_to_all_single on the peer-major
buffers) and the rank-ordered observer reduction run exactly as on the GPUs;
only the pass kernels are emulated in numpy (tests/slab_emulator.py).  The
result must equal the single-process oracle.
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
    g = orc.Grid((16, 8, 16), (20e-6, 4e-6, 250e-6), (-10e-6, 0.25e-6, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = g.meshgrid()
    v = orc.MUB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                        + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(5)
    a0 = rng.standard_normal(g.n) + 1j * rng.standard_normal(g.n)
    return g, v, m, a0


def _worker(rank, world, port, steps, out):
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_2451_b200 import slab
        from slab_emulator import EmulatedRank

        g, v, m, a0 = _case()
        f = orc.make_factors(g, v, m, 1e-6)
        lay = slab.SlabLayout(g.n, world, rank)
        emu = EmulatedRank(lay, f)
        bufs = {"psi": a0[lay.x_slice].reshape(-1).copy(),
                "send": np.zeros(lay.points, complex), "recv": np.zeros(lay.points, complex)}
        for op in slab.segment_schedule(steps):
            if op[0] == "pass":
                emu.run_pass(op[1], bufs[op[2]], bufs[op[3]])
            else:
                src = torch.view_as_real(torch.from_numpy(bufs[op[1]]))
                dst = torch.empty_like(src)
                dist.all_to_all_single(dst, src.contiguous())
                bufs[op[2]][:] = torch.view_as_complex(dst).numpy()
        # rank-ordered reduction of a per-rank partial
        part = torch.tensor([float(np.sum(np.abs(bufs["psi"]) ** 2)), float(rank)], dtype=torch.float64)
        tot = slab.combine_in_rank_order(part)
        slabs = [torch.empty(lay.points * 2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(slabs, torch.view_as_real(torch.from_numpy(bufs["psi"])).reshape(-1).clone())
        if rank == 0:
            full = np.concatenate([torch.view_as_complex(s.reshape(-1, 2)).numpy() for s in slabs])
            np.save(out, full.reshape(g.n))
            np.save(out + ".sum.npy", tot.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_slab_schedule_matches_oracle(tmp_path, world):
    steps = 5
    out = str(tmp_path / "psi.npy")
    mp.spawn(_worker, args=(world, _free_port(), steps, out), nprocs=world, join=True)
    got = np.load(out)
    g, v, m, a0 = _case()
    ref = orc.advance(a0.copy(), orc.make_factors(g, v, m, 1e-6), steps)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13
    tot = np.load(out + ".sum.npy")
    assert tot[1] == sum(range(world))
    assert tot[0] == pytest.approx(float(np.sum(np.abs(ref) ** 2)), rel=1e-12)


def test_layout_validation():
    from paper_1309_2451_b200.slab import SlabLayout

    with pytest.raises(ValueError, match="divisible"):
        SlabLayout((24, 16, 8), 16, 0)
    with pytest.raises(ValueError, match="out of range"):
        SlabLayout((16, 16, 8), 2, 2)
    lay = SlabLayout((512, 512, 512), 8, 3)
    assert lay.x_slice == slice(192, 256)
    assert lay.slab_shape == (64, 512, 512)
    assert lay.yslab_shape == (512, 64, 512)
    # 2 transposes of (P-1)/P of the 16 B/pt slab
    assert lay.a2a_bytes_per_step() == 2 * 7 * (64 * 512 * 512) // 8 * 16


def test_schedule_shape():
    from paper_1309_2451_b200 import _lib
    from paper_1309_2451_b200.slab import segment_schedule

    assert list(segment_schedule(0)) == []
    ops = list(segment_schedule(3))
    assert ops[0] == ("pass", _lib.PASS_Z_FIRST, "psi", "psi")
    assert ops[-1] == ("pass", _lib.PASS_Z_LAST, "psi", "psi")
    assert sum(1 for o in ops if o[0] == "a2a") == 6
    assert sum(1 for o in ops if o[0] == "pass" and o[1] == _lib.PASS_Z_MID) == 2


def test_fused_schedule_shape():
    from paper_1309_2451_b200 import _lib
    from paper_1309_2451_b200.slab import segment_schedule_fused

    assert list(segment_schedule_fused(0)) == []
    ops = list(segment_schedule_fused(2))
    kinds = [o[1] if o[0] == "pass" else "barrier" for o in ops]
    assert kinds == [_lib.PASS_Z_FIRST,
                     _lib.PASS_Y_FWD_TO_PEERS, "barrier", _lib.PASS_X_KIN_TO_PEERS, "barrier",
                     _lib.PASS_Y_INV_FROM_PEER, _lib.PASS_Z_MID,
                     _lib.PASS_Y_FWD_TO_PEERS, "barrier", _lib.PASS_X_KIN_TO_PEERS, "barrier",
                     _lib.PASS_Y_INV_FROM_PEER, _lib.PASS_Z_LAST]


def test_chunked_schedule_shape_and_dependencies():
    """segment_schedule_chunked: per step K y passes, K exchanges, K kinetic
    passes, K exchanges, K y^-1 passes; every chunk's exchange comes after its
    own producer pass and before its consumer pass (the event order the two
    streams of SlabPropagator._advance_chunked follow)."""
    from paper_1309_2451_b200 import _lib
    from paper_1309_2451_b200.slab import segment_schedule_chunked

    K, steps = 4, 2
    ops = list(segment_schedule_chunked(steps, K))
    assert ops[0] == ("pass", _lib.PASS_Z_FIRST, "psi", "psi") and ops[-1][1] == _lib.PASS_Z_LAST
    assert sum(1 for o in ops if o[0] == "a2a") == 2 * K * steps
    assert sum(1 for o in ops if o[0] == "cpass") == 3 * K * steps
    done = set()
    for o in ops:
        if o[0] == "cpass":
            _, kind, src, dst, c = o
            if src != "psi":
                assert (src, c) in done, o
            done.add((dst, c))
        elif o[0] == "a2a":
            assert (o[1], o[3]) in done, o
            done.add((o[2], o[3]))
