"""Host-side logic of the drop-in (no GPU needed): data model, validation,
event schedule, trace/snapshot formats, and the no-CPU-fallback rule."""

import numpy as np
import pytest
import torch

from oracle import split_step as orc
from paper_1309_2451_b200 import observables as obs
from paper_1309_2451_b200 import propagator as prop
from paper_1309_2451_b200 import qgrid
from paper_1309_2451_b200.constants import species_mass

M = species_mass("li6")


def test_units_match_oracle():
    u = qgrid.UnitSystem(1e-6, M)
    assert u.time == orc.unit_time(M)
    assert u.energy == orc.unit_energy(M)


def test_grid_axes_and_k_match_oracle_bitwise():
    g = qgrid.make_grid(16, 8, 32, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 0.25e-6, 0.0))
    og = orc.as_grid(g)
    for i in range(3):
        assert np.array_equal(g.axis(i), og.axis(i))
        assert np.array_equal(g.k_axis(i), og.k_axis(i))
    assert np.array_equal(g.k_squared(), og.k_squared())
    assert g.dvol == og.dvol
    # k convention of the reference (qgrid.py:3-7, test_qgrid.py): |k|max = pi n / L
    assert abs(np.abs(g.kx).max() - np.pi * 16 / 20e-6) < 1e-6


@pytest.mark.parametrize("n", [4, 12, 0, 7])
def test_make_grid_rejects_non_pow2(n):
    with pytest.raises(ValueError, match="powers of two"):
        qgrid.make_grid(n, 8, 8, (1e-5,) * 3)


def test_make_grid_rejects_nonpositive_extent():
    with pytest.raises(ValueError, match="extents must be positive"):
        qgrid.make_grid(8, 8, 8, (1e-5, 0.0, 1e-5))


def test_wavefunction_shape_check_and_host_copy():
    g = qgrid.make_grid(8, 8, 8, (1e-5,) * 3)
    with pytest.raises(ValueError, match="amplitude shape"):
        qgrid.Wavefunction(np.zeros((8, 8, 4), complex), g)
    a = np.arange(512, dtype=complex).reshape(8, 8, 8)
    w = qgrid.Wavefunction(a, g, time=1.5)
    c = w.copy()
    c.amplitudes[0, 0, 0] = 99
    assert w.amplitudes[0, 0, 0] == 0 and c.time == 1.5
    assert np.array_equal(w.density(), np.abs(a) ** 2)


def test_gaussian_packet_boundary_and_width_guards():
    g = qgrid.make_grid(16, 16, 16, (10e-6,) * 3, origin=(-5e-6,) * 3)
    with pytest.raises(ValueError, match="widths must be positive"):
        qgrid.gaussian_packet(g, (0, 0, 0), (1e-6, 0, 1e-6))
    with pytest.raises(ValueError, match="too close to boundary along axis 1"):
        qgrid.gaussian_packet(g, (0, 4e-6, 0), (0.5e-6,) * 3)


def test_same_grid_is_by_value():
    a = qgrid.make_grid(8, 8, 8, (1e-5,) * 3)
    b = qgrid.SimGrid((8, 8, 8), (1e-5, 1e-5, 1e-5), (0.0, 0.0, 0.0))
    assert qgrid.same_grid(a, b)
    assert qgrid.same_grid(a, orc.as_grid(a))
    assert not qgrid.same_grid(a, qgrid.make_grid(8, 8, 16, (1e-5,) * 3))


def test_event_schedule_matches_reference_contract():
    class O:
        def __init__(self, s):
            self.stride = s

    assert prop.event_schedule(20, [O(7)]) == [0, 7, 14, 20]
    assert prop.event_schedule(10, [O(5), O(3)]) == [0, 3, 5, 6, 9, 10]
    assert prop.event_schedule(0, [O(4)]) == [0]
    assert prop.event_schedule(10, []) == orc.event_schedule(10, [])
    with pytest.raises(ValueError, match="stride must be positive"):
        prop.event_schedule(10, [O(0)])


def test_make_plan_validation_before_device_work():
    g = qgrid.make_grid(8, 8, 8, (1e-5,) * 3)
    with pytest.raises(ValueError, match="unknown mode"):
        prop.make_plan(g, np.zeros(g.n), M, 1e-6, mode="sideways")
    with pytest.raises(ValueError, match="shape does not match"):
        prop.make_plan(g, np.zeros((8, 8, 4)), M, 1e-6)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    g = qgrid.make_grid(8, 8, 8, (1e-5,) * 3)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        prop.make_plan(g, np.zeros(g.n), M, 1e-6)
    w = qgrid.Wavefunction(np.ones(g.n, complex), g)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        w.norm()


def test_trace_csv_roundtrip_and_fidelity(tmp_path):
    tr = obs.PopulationTrace()
    for k in range(5):
        tr.append(k * 1e-6, 0.9 - 0.2 * k, 0.05, 0.05 + 0.2 * k, 1.0, 1e-9 * k)
    path = tmp_path / "trace.csv"
    tr.to_csv(path)
    assert path.read_text().splitlines()[0] == "t,p_l,p_m,p_r,norm,edge"
    back = obs.PopulationTrace.from_csv(path)
    assert np.array_equal(back.as_array(), tr.as_array())
    assert obs.transfer_fidelity(tr) == tr.p_r[-1]
    assert tr.max_middle() == 0.05
    with pytest.raises(ValueError, match="empty population trace"):
        obs.transfer_fidelity(obs.PopulationTrace())


def test_qwf1_snapshot_roundtrip(tmp_path):
    g = qgrid.make_grid(8, 8, 16, (1e-5, 2e-5, 3e-5), origin=(-1e-6, 0.5e-6, 0.0))
    rng = np.random.default_rng(1)
    a = rng.standard_normal(g.n) + 1j * rng.standard_normal(g.n)
    p = tmp_path / "psi.qwf"
    qgrid.write_snapshot(p, a, g, time=2.5e-6)
    b, g2, t = qgrid.read_snapshot(p)
    assert np.array_equal(a, b) and t == 2.5e-6
    assert g2.n == g.n and np.allclose(g2.extents, g.extents) and g2.origin == g.origin
    raw = p.read_bytes()
    assert raw[:4] == b"QWF1" and len(raw) == 4 + 88 + 16 * a.size
    r = rng.standard_normal(g.n)
    qgrid.write_snapshot(p, r, g)
    assert np.array_equal(qgrid.read_snapshot(p)[0], r)
    p.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="bad magic"):
        qgrid.read_snapshot(p)


def test_symmetric_partition():
    g = qgrid.make_grid(16, 8, 32, (20e-6, 4e-6, 40e-6))
    part = obs.symmetric_partition(g, 3.5e-6)
    assert part.xb1.shape == (32,) and np.all(part.xb1 == -3.5e-6) and np.all(part.xb2 == 3.5e-6)
    assert not part.merged.any() and part.grid_ref is g


def test_unknown_precision_rejected():
    g = qgrid.make_grid(8, 8, 8, (1e-5,) * 3)
    with pytest.raises((ValueError, RuntimeError)):
        prop.make_plan(g, np.zeros(g.n), M, 1e-6, precision="complex32")


def test_bench_thread_counts_matches_reference_rule():
    """runner.bench_thread_counts (runner.py:260-268): powers of two below the
    host thread count, plus the count."""
    from paper_1309_2451_b200.runner import bench_thread_counts

    assert bench_thread_counts(1) == [1]
    assert bench_thread_counts(6) == [1, 2, 4, 6]
    assert bench_thread_counts(8) == [1, 2, 4, 8]
    assert bench_thread_counts(16) == [1, 2, 4, 8, 16]


def test_bench_grid_parsing_and_identical_arm_configs():
    """bench.py: --grid parsing, and both arms report the same config dict
    (the driver compares the arms' configs)."""
    import argparse

    import bench

    assert bench.parse_grid("512x512x512") == (512, 512, 512)
    assert bench.parse_grid("1024,1024,512") == (1024, 1024, 512)
    with pytest.raises(argparse.ArgumentTypeError):
        bench.parse_grid("64x64")
    c = bench._config((512, 512, 512))
    assert c == bench._config([512, 512, 512])
    assert "BASELINE config 4" in c["workload"] and c["grid"] == [512, 512, 512]
    assert "BASELINE config 5" in bench._config((1024, 1024, 512))["workload"]
