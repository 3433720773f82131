"""The evolve pipeline on the device (runner.py:114-229 of the reference):
partition, transverse spectrum, transverse ground state, initial state and a
short CTAP run, against tests/golden/runner_scaled_64x32x64.npz made by the
reference's own runner on the same 64x32x64 scaled-chip grid."""

import dataclasses

import numpy as np
import pytest

from conftest import load_golden
from paper_1309_2451_b200 import magfield, observables, propagator, qgrid, runner

pytestmark = pytest.mark.gpu


@dataclasses.dataclass(frozen=True, eq=False)
class TableLayout(magfield.ChipSegments):
    """Chip segments plus the wire x positions per z slice (the part of a
    reference ChipLayout that build_partition needs)."""

    wire_table: np.ndarray = None
    zs: np.ndarray = None

    def wire_positions_at(self, z):
        k = int(np.argmin(np.abs(self.zs - z)))
        return dict(zip(("left", "middle", "right"), self.wire_table[k]))


@dataclasses.dataclass(frozen=True)
class StubConfig:
    grid: object
    layout: object
    z_start_eff: float
    sigma_z_eff: float
    gs_tau: float
    gs_tol: float
    mass: float
    dt: float
    n_steps: int = 200
    trace_stride: int = 50
    edge_stride: int = 50
    edge_margin_cells: int = 2
    edge_threshold: float = 1.0
    i_middle: float = 0.014
    ordering: str = "counter_intuitive"

    def to_grid(self):
        return self.grid

    def to_layout(self, i_middle=None):
        if i_middle is None or i_middle == self.i_middle:
            return self.layout
        cur = self.layout.seg_cur.copy()
        cur[np.isclose(cur, self.i_middle)] = i_middle
        return dataclasses.replace(self.layout, seg_cur=cur)

    def sweep_values(self):
        return np.array([self.i_middle, 0.9 * self.i_middle])


def _setup():
    d = load_golden("runner_scaled_64x32x64.npz")
    grid = qgrid.SimGrid(tuple(int(v) for v in d["n"]), tuple(float(v) for v in d["extents"]),
                         tuple(float(v) for v in d["origin"]))
    chip = magfield.ChipSegments.from_arrays(load_golden("segments_scaled.npz"))
    lay = TableLayout(**{f.name: getattr(chip, f.name) for f in dataclasses.fields(chip)},
                      wire_table=d["wire_pos"], zs=np.asarray(grid.z))
    cfg = StubConfig(grid, lay, float(d["z_start"]), float(d["sigma_z"]), float(d["gs_tau"]),
                     float(d["gs_tol"]), float(d["mass"]), float(d["dt"]))
    return d, cfg


def test_prepare_potential_and_spectrum_match_reference():
    d, cfg = _setup()
    _, grid, pot, part = runner.prepare_potential(cfg)
    assert np.array_equal(part.xb1, d["xb1"]) and np.array_equal(part.xb2, d["xb2"])
    assert np.array_equal(part.merged, d["merged"])
    s = runner.transverse_spectrum(pot, int(d["iz0"]), 0)
    assert np.array_equal(np.array([s.omega_x, s.omega_y, s.v_min, *s.energies]), d["spectrum"])


def test_transverse_ground_state_and_initial_state():
    d, cfg = _setup()
    _, grid, pot, part = runner.prepare_potential(cfg)
    phi = runner.transverse_ground_state(pot, part, int(d["iz0"]), 0, tau=cfg.gs_tau, tol=cfg.gs_tol)
    assert np.linalg.norm(phi - d["phi"]) / np.linalg.norm(d["phi"]) < 1e-9
    psi = runner.initial_state(cfg, pot, part)
    a = psi.amplitudes
    ref = d["psi0_center"]
    assert np.linalg.norm(a[:, :, int(d["iz0"])] - ref) / np.linalg.norm(ref) < 1e-9
    assert psi.norm() == pytest.approx(1.0, abs=1e-12)


def test_evolve_point_trace_matches_reference():
    d, cfg = _setup()
    res = runner.evolve_point(cfg)
    got = res["trace"].as_array()
    assert got.shape == d["trace"].shape
    assert np.array_equal(got[:, 0], d["trace"][:, 0])
    assert np.abs(got[:, 1:4] - d["trace"][:, 1:4]).max() < 1e-9
    assert res["final_p_r"] == got[-1, 3]


def test_run_sweep_single_replica(tmp_path):
    d, cfg = _setup()
    cfg = dataclasses.replace(cfg, n_steps=100)
    rows = runner.run_sweep(cfg, str(tmp_path))
    assert [(r[1], r[0]) for r in rows] == runner.sweep_points(cfg.sweep_values())
    direct = runner.evolve_point(cfg, i_middle=float(cfg.sweep_values()[1]))["final_p_r"]
    assert rows[1][2] == direct
    assert (tmp_path / "sweep.csv").exists()


@dataclasses.dataclass(frozen=True)
class BenchConfig:
    """The fields of ExperimentConfig that run_bench reads (defaults of the
    reference config: 64^3 over 20 x 4 x 1000 um, f_z = 5 Hz, dt = 1 us)."""

    mass: float
    omega_z: float = 2 * np.pi * 5.0
    dt: float = 1e-6
    bench_warm_steps: int = 100
    bench_timed_steps: int = 300

    def to_grid(self):
        return qgrid.make_grid(64, 64, 64, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / 128, 0.0))


def test_run_bench_reports_and_files(tmp_path):
    """runner.run_bench (runner.py:271-325): median/min/max chunk rates per
    thread count, bench.csv and bench.txt in the reference's format."""
    from paper_1309_2451_b200.constants import species_mass

    cfg = BenchConfig(mass=species_mass("li6"))
    rep = runner.run_bench(cfg, str(tmp_path), thread_counts=[1, 2], warm_steps=20, timed_steps=100, chunks=5)
    assert rep["grid"] == (64, 64, 64) and set(rep["rates"]) == {1, 2}
    for r in rep["rates"].values():
        assert 0 < r["min"] <= r["median"] <= r["max"]
    lines = open(rep["csv"]).read().splitlines()
    assert lines[0] == "threads,steps_per_sec" and len(lines) == 3
    assert float(lines[1].split(",")[1]) == rep["rates"][1]["median"]
    txt = open(rep["txt"]).read()
    assert "warm 20 steps discarded, 100 timed steps in 5 chunks" in txt and "threads=2: median" in txt
