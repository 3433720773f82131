"""Replica-parallel current sweep (runner.run_sweep) on CPU:
world_size 1, 2 and 3 over gloo with a stand-in for the per-point run.  The
gathered rows must be the reference's order (orderings outer, currents
inner, runner.py:238-242) whatever the number of replicas, and rank 0 alone
writes sweep.csv."""

import dataclasses
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


@dataclasses.dataclass(frozen=True)
class FakeCfg:
    ordering: str = "counter_intuitive"

    def sweep_values(self):
        return np.array([0.010, 0.012, 0.014, 0.016, 0.018])


def fake_point(cfg, i_m):
    # deterministic stand-in for evolve_point(...)["final_p_r"]
    return i_m * 1e3 + (0.5 if cfg.ordering == "intuitive" else 0.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, result_dir):
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_2451_b200 import runner
        from test_sweep_gloo import FakeCfg, fake_point

        ran = []

        def point(cfg, i_m):
            ran.append((cfg.ordering, i_m))
            return fake_point(cfg, i_m)

        rows = runner.run_sweep(FakeCfg(), out_dir, run_point=point)
        np.save(os.path.join(result_dir, f"rows_{rank}.npy"), np.array([r[2] for r in rows]))
        np.save(os.path.join(result_dir, f"ran_{rank}.npy"), np.array([i for _, i in ran]))
    finally:
        dist.destroy_process_group()


def test_sweep_points_and_shares():
    from paper_1309_2451_b200 import runner

    pts = runner.sweep_points([1.0, 2.0])
    assert pts == [("counter_intuitive", 1.0), ("counter_intuitive", 2.0), ("intuitive", 1.0), ("intuitive", 2.0)]
    for world in (1, 2, 3, 8):
        shares = [runner.rank_share(10, r, world) for r in range(world)]
        assert sorted(sum(shares, [])) == list(range(10))


@pytest.mark.parametrize("world", [2, 3])
def test_replica_sweep_gloo(tmp_path, world):
    from paper_1309_2451_b200 import runner

    seq = runner.run_sweep(FakeCfg(), None, run_point=fake_point)
    out = tmp_path / "sweep"
    mp.spawn(_worker, args=(world, _free_port(), str(out), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert np.array_equal(np.load(tmp_path / f"rows_{r}.npy"), np.array([row[2] for row in seq]))
        assert len(np.load(tmp_path / f"ran_{r}.npy")) == len(runner.rank_share(len(seq), r, world))
    lines = (out / "sweep.csv").read_text().splitlines()
    assert lines[0] == "i_m,ordering,final_p_r" and len(lines) == 1 + len(seq)
    assert lines[1].split(",")[1] == "counter_intuitive" and lines[-1].split(",")[1] == "intuitive"


class PlainCfg:
    """Not a dataclass: run_sweep must still give each point its ordering
    (reference runner.py:238-242 builds a config per ordering)."""

    def __init__(self):
        self.ordering = "counter_intuitive"

    def sweep_values(self):
        return np.array([0.010, 0.012])


def test_sweep_plain_config_gets_each_ordering():
    from paper_1309_2451_b200 import runner

    cfg = PlainCfg()
    seen = []
    rows = runner.run_sweep(cfg, None, run_point=lambda c, i: seen.append(c.ordering) or fake_point(c, i))
    assert seen == ["counter_intuitive", "counter_intuitive", "intuitive", "intuitive"]
    assert [r[1] for r in rows] == seen
    assert rows[-1][2] == fake_point(FakeCfg(ordering="intuitive"), 0.012)
    assert cfg.ordering == "counter_intuitive"   # the caller's object is untouched
