"""Parity of the CUDA path (through libctap.so) with the CPU oracle and the
reference's golden vectors.

Gates (BASELINE.json north_star): complex128 wavefunction relative L2 error
<= 1e-10 and guide populations within 1e-9 after N steps; potential bitwise.
"""

import numpy as np
import pytest
import torch

from conftest import load_golden, oracle_grid, product_grid
from oracle import potential as opot
from oracle import split_step as orc
from paper_1309_2451_b200 import _lib, magfield, observables, propagator, qgrid
from paper_1309_2451_b200.constants import species_mass

pytestmark = pytest.mark.gpu

REL_L2 = 1e-10
POP_TOL = 1e-9
M = species_mass("li6")


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def partition_of(d, grid):
    return observables.GuidePartition(xb1=d["xb1"], xb2=d["xb2"], grid_ref=grid)


@pytest.mark.parametrize("name", ["ioffe_32x16x32.npz", "ctap_scaled_32x16x32.npz"])
def test_golden_evolution_with_trace(name):
    d = load_golden(name)
    grid = product_grid(d)
    psi = qgrid.Wavefunction(d["psi0"].copy(), grid)
    plan = propagator.make_plan(grid, d["V"], float(d["mass"]), float(d["dt"]))
    rec = observables.PopulationRecorder(partition_of(d, grid), stride=int(d["stride"]))
    psi, stats = propagator.evolve_real(psi, plan, int(d["steps"]), [rec])
    assert stats.n_steps == int(d["steps"])
    assert rel_l2(psi.amplitudes, d["psi"]) <= REL_L2
    got = rec.trace.as_array()
    assert got.shape == d["trace"].shape
    assert np.array_equal(got[:, 0], d["trace"][:, 0])          # time stamps exact
    assert np.abs(got[:, 1:4] - d["trace"][:, 1:4]).max() <= POP_TOL
    assert np.abs(got[:, 4] - d["trace"][:, 4]).max() <= 1e-12   # norm
    assert np.abs(got[:, 5] - d["trace"][:, 5]).max() <= 1e-12   # edge mass


def test_golden_harmonic():
    d = load_golden("harmonic_16x16x32.npz")
    grid = product_grid(d)
    psi = qgrid.Wavefunction(d["psi0"].copy(), grid)
    plan = propagator.make_plan(grid, d["V"], float(d["mass"]), float(d["dt"]))
    psi, _ = propagator.evolve_real(psi, plan, int(d["steps"]))
    assert rel_l2(psi.amplitudes, d["psi"]) <= REL_L2


def test_device_potential_bitwise_golden():
    d = load_golden("ctap_scaled_32x16x32.npz")
    chip = magfield.ChipSegments.from_arrays(load_golden("segments_scaled.npz"))
    grid = product_grid(d)
    v = magfield.potential_values(chip, grid).cpu().numpy()
    assert np.array_equal(v, d["V"])


def test_phase_fields_match_reference_plan():
    d = load_golden("ctap_scaled_32x16x32.npz")
    grid = product_grid(d)
    plan = propagator.make_plan(grid, d["V"], float(d["mass"]), float(d["dt"]))
    # same phase bit for bit; cos/sin may differ from glibc by an ulp
    for name in ("exp_v_half", "exp_v_full", "exp_k"):
        got, ref = getattr(plan, name), d[name]
        assert np.abs(got - ref).max() <= 4.5e-16, name
    assert np.abs(np.abs(plan.exp_v_half) - 1).max() < 1e-14
    assert np.abs(np.abs(plan.exp_k) - 1).max() < 1e-14


def test_observables_golden():
    d = load_golden("observables_16x8x8.npz")
    grid = product_grid(d)
    psi = qgrid.Wavefunction(d["amps"].copy(), grid)
    part = observables.GuidePartition(xb1=d["xb1"], xb2=d["xb2"], grid_ref=grid)
    pops = observables.populations(psi, part)
    assert np.allclose(pops, d["pops"], rtol=1e-13, atol=0)
    for m, e in zip(d["margins"], d["edges"]):
        assert observables.edge_density(psi, int(m)) == pytest.approx(float(e), rel=1e-13)
    assert psi.norm() == pytest.approx(float(d["norm"]), rel=1e-13)
    assert np.allclose(observables.density_xz(psi), d["density_xz"], rtol=1e-13, atol=0)


def test_energies_and_ground_state_golden():
    d = load_golden("imag_16.npz")
    grid = product_grid(d)
    m = float(d["mass"])
    seed = qgrid.Wavefunction(d["seed"].copy(), grid)
    assert propagator.kinetic_expectation(seed, m) == pytest.approx(float(d["e_seed_t"]), rel=1e-12)
    assert propagator.potential_expectation(seed, d["V"]) == pytest.approx(float(d["e_seed_v"]), rel=1e-12)
    gs = propagator.ground_state_imaginary(grid, d["V"], seed, tol=float(d["tol"]),
                                           tau=float(d["tau"]), mass=m)
    # imaginary time is contracting: tiny per-step differences (exp ulps, FFT
    # round-off) shrink, so the converged state matches closely
    assert rel_l2(gs.amplitudes, d["gs"]) <= 1e-8
    assert propagator.energy_expectation(gs, d["V"], m) == pytest.approx(float(d["e_gs"]), rel=1e-10)
    assert abs(gs.norm() - 1) < 1e-12


def test_config1_harmonic_64cube_1000_steps():
    """BASELINE config 1: run_bench's synthetic trap on the default 64^3 grid."""
    og = orc.Grid((64, 64, 64), (20e-6, 4e-6, 1000e-6), (-10e-6, 4e-6 / 128, 0.0))
    v = orc.bench_potential(og, M, 5.0)
    c = [og.origin[i] + og.extents[i] / 2 for i in range(3)]
    a0 = orc.gaussian_packet(og, c, [e / 16 for e in og.extents])
    f = orc.make_factors(og, v, M, 1e-6)
    part = observables.GuidePartition(xb1=np.full(64, -3.5e-6), xb2=np.full(64, 3.5e-6))
    ref, rows = orc.evolve_with_trace(a0.copy(), og, f, 1000, 50, part.xb1, part.xb2)
    grid = qgrid.SimGrid(og.n, og.extents, og.origin)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    rec = observables.PopulationRecorder(part, stride=50)
    psi, _ = propagator.evolve_real(psi, propagator.make_plan(grid, v, M, 1e-6), 1000, [rec])
    assert rel_l2(psi.amplitudes, ref) <= REL_L2
    assert np.abs(rec.trace.as_array()[:, 1:4] - rows[:, 1:4]).max() <= POP_TOL


def test_ctap_scaled_chip_64cube_1000_steps():
    """Phase-sensitive CTAP case (|phi_V| >= 1312 rad per step): device V bitwise
    equal to the oracle's, then 1000 steps within 1e-10."""
    chip_d = load_golden("segments_scaled.npz")
    chip = magfield.ChipSegments.from_arrays(chip_d)
    ny = 64
    og = orc.Grid((64, ny, 64), (20e-6, 4e-6, 250e-6), (-10e-6, 4e-6 / ny / 2, 0.0))
    grid = qgrid.SimGrid(og.n, og.extents, og.origin)
    v_dev = magfield.potential_values(chip, grid)
    v = opot.potential_from_chip(chip_d, og.axis(0), og.axis(1), og.axis(2))
    assert np.array_equal(v_dev.cpu().numpy(), v)
    phi_full = (-1.0 * (v / orc.unit_energy(M))) * (1e-6 / orc.unit_time(M))
    assert phi_full.max() < -1300.0   # Ioffe floor: large phases every step
    a0 = orc.gaussian_packet(og, (-3.5e-6, 2e-6, 60e-6), (0.5e-6, 0.3e-6, 10e-6))
    f = orc.make_factors(og, v, M, 1e-6)
    xb = np.full(64, 1.75e-6)
    ref, rows = orc.evolve_with_trace(a0.copy(), og, f, 1000, 100, -xb, xb)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    part = observables.GuidePartition(xb1=-xb, xb2=xb, grid_ref=grid)
    rec = observables.PopulationRecorder(part, stride=100)
    psi, _ = propagator.evolve_real(psi, propagator.make_plan(grid, v_dev, M, 1e-6), 1000, [rec])
    assert rel_l2(psi.amplitudes, ref) <= REL_L2
    assert np.abs(rec.trace.as_array()[:, 1:4] - rows[:, 1:4]).max() <= POP_TOL


@pytest.mark.parametrize("n", [(8, 8, 8), (16, 32, 8), (128, 8, 16), (8, 256, 32), (1024, 8, 8),
                               (8, 1024, 8), (8, 8, 1024), (32, 512, 16)])
def test_fft_every_axis_length(n):
    """Axis lengths 8..1024 on every axis against numpy's FFT."""
    rng = np.random.default_rng(sum(n))
    a = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    grid = qgrid.SimGrid(n, (1e-5,) * 3, (0.0,) * 3)
    plan = propagator._aux_plan(grid)
    d = torch.from_numpy(a.copy()).cuda()
    plan.fft3d(d, -1)
    ref = np.fft.fftn(a)
    assert rel_l2(d.cpu().numpy(), ref) <= 1e-14
    plan.fft3d(d, +1)
    assert rel_l2(d.cpu().numpy() / a.size, a) <= 1e-14


def test_determinism_bitwise():
    d = load_golden("ioffe_32x16x32.npz")
    grid = product_grid(d)

    def run():
        psi = qgrid.Wavefunction(d["psi0"].copy(), grid)
        plan = propagator.make_plan(grid, d["V"], M, 1e-6)
        rec = observables.PopulationRecorder(partition_of(d, grid), stride=10)
        psi, _ = propagator.evolve_real(psi, plan, 50, [rec])
        return psi.amplitudes, rec.trace.as_array()

    a1, t1 = run()
    a2, t2 = run()
    assert np.array_equal(a1, a2)
    assert np.array_equal(t1, t2)


@pytest.mark.parametrize("steps", [300])
def test_complex64_mode_within_1e4(steps):
    """Optional complex64 mode (north_star): exact FP64 phases, complex64
    storage and transforms, held to <= 1e-4 against the complex128 oracle."""
    d = load_golden("ioffe_32x16x32.npz")
    grid = product_grid(d)
    psi = qgrid.Wavefunction(d["psi0"].copy(), grid)
    plan = propagator.make_plan(grid, d["V"], float(d["mass"]), float(d["dt"]), precision="complex64")
    rec = observables.PopulationRecorder(partition_of(d, grid), stride=int(d["stride"]))
    psi, _ = propagator.evolve_real(psi, plan, steps, [rec])
    got = psi.amplitudes
    assert got.dtype == np.complex64
    assert rel_l2(got.astype(np.complex128), d["psi"]) <= 1e-4
    assert np.abs(rec.trace.as_array()[:, 1:4] - d["trace"][:, 1:4]).max() <= 1e-4


def test_complex64_fft_and_reductions():
    rng = np.random.default_rng(4)
    n = (16, 64, 32)
    a = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    grid = qgrid.SimGrid(n, (1e-5,) * 3, (0.0,) * 3)
    plan = propagator._aux_plan(grid, torch.complex64)
    d = torch.from_numpy(a.copy()).cuda()
    plan.fft3d(d, -1)
    assert rel_l2(d.cpu().numpy(), np.fft.fftn(a.astype(np.complex128))) <= 1e-6
    w = qgrid.Wavefunction(a.copy(), grid)
    assert w.norm() == pytest.approx(float(np.sum(np.abs(a.astype(np.complex128)) ** 2) * grid.dvol), rel=1e-6)


@pytest.mark.parametrize("precision", ["complex128", "complex64"])
def test_regenerated_k2_matches_table_loads(monkeypatch, precision):
    """The x pass regenerates kx^2, ky^2, kz^2 in registers once the plan has
    verified numpy's (2 pi fftfreq)^2 tables bit for bit; forcing the table
    loads (CTAP_KGEN=0) must give the identical wavefunction."""
    n = (128, 64, 32)
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    x, y, z = grid.x, grid.y, grid.z
    v = 0.5 * M * ((2 * np.pi * 2e3) ** 2 * x[:, None, None] ** 2 + (2 * np.pi * 2e4) ** 2
                   * (y[None, :, None] - 2e-6) ** 2 + (2 * np.pi * 20) ** 2 * (z[None, None, :] - 125e-6) ** 2)
    psi0 = qgrid.gaussian_packet(grid, (-2e-6, 2e-6, 125e-6), (1e-6, 0.3e-6, 10e-6)).amplitudes

    def run(kgen):
        monkeypatch.setenv("CTAP_KGEN", kgen)
        plan = propagator.make_plan(grid, v, M, 1e-6, precision=precision)
        psi = qgrid.Wavefunction(psi0.copy(), grid)
        psi, _ = propagator.evolve_real(psi, plan, 20)
        return psi.amplitudes

    assert np.array_equal(run("1"), run("0"))


@pytest.mark.parametrize("precision", ["complex128", "complex64"])
def test_zchunked_kinetic_block_bitwise(monkeypatch, precision):
    """CTAP_ZCHUNK runs y, [x K x^-1], y^-1 per z chunk on two forked streams
    (an experiment kept behind a switch); the result must not change."""
    n = (64, 32, 64)
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    rng = np.random.default_rng(3)
    v = 1e-30 * (1.0 + rng.random(n))
    a0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)

    def run(w):
        monkeypatch.setenv("CTAP_ZCHUNK", w)
        plan = propagator.make_plan(grid, v, M, 1e-6, precision=precision)
        psi = qgrid.Wavefunction(a0.copy(), grid)
        psi, _ = propagator.evolve_real(psi, plan, 40)
        return psi.amplitudes

    ref = run("0")
    assert np.array_equal(run("16"), ref)
    assert np.array_equal(run("32"), ref)


@pytest.mark.parametrize("n,tables", [((1024, 16, 32), 0), ((64, 32, 64), 2), ((64, 32, 64), 3)])
def test_zchunked_kinetic_block_other_paths(monkeypatch, n, tables):
    """The z-chunked kinetic block also through the 1024-point x pass (4-column
    tiles) and with the exp(-ik^2 dt/2) table (indexed at the chunk's absolute
    z): unchanged results (both paths used to mis-address chunks)."""
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    rng = np.random.default_rng(5)
    v = 1e-30 * (1.0 + rng.random(n))
    a0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)

    def run(w):
        monkeypatch.setenv("CTAP_ZCHUNK", w)
        plan = propagator.make_plan(grid, v, M, 1e-6, phase_tables=tables)
        psi = qgrid.Wavefunction(a0.copy(), grid)
        psi, _ = propagator.evolve_real(psi, plan, 12)
        return psi.amplitudes

    ref = run("0")
    assert np.array_equal(run("8"), ref)
    assert np.array_equal(run("16"), ref)


def test_complex64_has_no_systematic_rounding_drift():
    """complex64 applies no rounded constant to the data (float-float
    twiddles and sqrt(1/2), FP64 phase products): a rounded factor would
    repeat at every point every step and the norm would drift linearly
    (-5e-5 after 1000 steps with the radix-8 constant rounded to float)."""
    n = (64, 64, 128)
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 125e-6) ** 2)
    a0 = qgrid.gaussian_packet(grid, (-2e-6, 2e-6, 125e-6), np.sqrt(1.0545718e-34 / (M * om))).amplitudes
    out = {}
    for prec in ("complex128", "complex64"):
        plan = propagator.make_plan(grid, v, M, 1e-6, precision=prec)
        psi = qgrid.Wavefunction(a0.copy(), grid)
        n0 = psi.norm()
        psi, _ = propagator.evolve_real(psi, plan, 1000)
        out[prec] = (psi.amplitudes.astype(np.complex128), psi.norm() / n0 - 1.0)
    assert abs(out["complex64"][1]) < 5e-6
    assert rel_l2(out["complex64"][0], out["complex128"][0]) < 5e-5


@pytest.mark.parametrize("n", [(512, 16, 32), (256, 32, 16), (1024, 8, 16), (16, 1024, 16)])
def test_wline_bitwise_equals_tile_kernel(monkeypatch, n):
    """The warp-per-line x-pass kernels (CTAP_WLINE=1 TMA ring, 2 one tile per
    CTA) use the same radix plan, twiddles and exact kinetic phase as
    tile_kernel (CTAP_WLINE=0), also with two warps per column (3): 30 steps
    must agree bit for bit, in real and
    imaginary time."""
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    rng = np.random.default_rng(7)
    v = 1e-30 * (1.0 + rng.random(n))
    a0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)

    def run(mode, kind):
        monkeypatch.setenv("CTAP_WLINE", mode)
        plan = propagator.make_plan(grid, v, M, 1e-6, mode=kind)
        psi = qgrid.Wavefunction(a0.copy(), grid)
        if kind == "real_time":
            psi, _ = propagator.evolve_real(psi, plan, 30)
        else:
            for _ in range(5):
                psi = propagator.step(psi, plan)
        return psi.amplitudes

    modes = ("1", "2", "3") if n[0] == 512 or n[1] == 1024 else ("4", "5", "6")  # 4-6: forced ring (nx 256/1024)
    for kind in ("real_time", "imaginary_time"):
        ref = run("0", kind)
        for mode in modes:
            assert np.array_equal(run(mode, kind), ref)


def test_1024_line_tiles_bitwise(tmp_path):
    """1024-point y and x lines run in 4-column tiles by default
    (CTAP_W1024=4, two 64 KB tiles per SM); the transform is the same, so the
    8-column tiles (CTAP_W1024=8) give identical bits.  CTAP_W1024 is read once
    per process, so each variant runs in its own subprocess."""
    import os
    import subprocess
    import sys

    code = (
        "import sys, numpy as np\n"
        "from paper_1309_2451_b200 import propagator, qgrid\n"
        "from paper_1309_2451_b200.constants import species_mass\n"
        "n = (1024, 16, 32)\n"
        "g = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 1.25e-7, 0.0))\n"
        "r = np.random.default_rng(2)\n"
        "v = 1e-30 * (1 + r.random(n))\n"
        "w = qgrid.Wavefunction(r.standard_normal(n) + 1j * r.standard_normal(n), g)\n"
        "w, _ = propagator.evolve_real(w, propagator.make_plan(g, v, species_mass('li6'), 1e-6), 10)\n"
        "np.save(sys.argv[1], w.amplitudes)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for w in ("4", "8"):
        path = str(tmp_path / f"w{w}.npy")
        subprocess.run([sys.executable, "-c", code, path], check=True, cwd=root,
                       env=dict(os.environ, CTAP_W1024=w, PYTHONPATH=root))
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("n", [(16, 16, 64), (8, 8, 512), (8, 8, 1024)])
def test_two_stage_z_fft_option(monkeypatch, n):
    """CTAP_Z2=1 (ctap_zline2.cu: the two-stage 32 x L/32 z transform, opt-in
    because it measured slower at 512^3) against the oracle and the default
    radix-8 z passes."""
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    rng = np.random.default_rng(17)
    x, y, z = grid.meshgrid()
    v = 0.5 * M * ((2 * np.pi * 2e3) ** 2 * x ** 2 + (2 * np.pi * 20.0) ** 2 * (z - 125e-6) ** 2) + 1e-28
    a0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    og = orc.as_grid(grid)
    ref = orc.advance(a0.copy(), orc.make_factors(og, v, M, 1e-6), 10)

    def run(z2):
        monkeypatch.setenv("CTAP_Z2", z2)
        psi = qgrid.Wavefunction(a0.copy(), grid)
        psi, _ = propagator.evolve_real(psi, propagator.make_plan(grid, v, M, 1e-6), 10)
        return psi.amplitudes

    got2, got1 = run("1"), run("0")
    assert rel_l2(got2, ref) <= REL_L2
    assert rel_l2(got2, got1) <= 1e-13
    d = torch.from_numpy(a0.copy()).cuda()
    monkeypatch.setenv("CTAP_Z2", "1")
    plan = propagator.make_plan(grid, v, M, 1e-6).native
    plan.run_pass(_lib.PASS_Z_FWD, d, d)
    assert rel_l2(d.cpu().numpy(), np.fft.fft(a0, axis=2)) <= 1e-14
