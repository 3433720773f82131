"""Pin the CPU oracle against vectors produced by the reference itself
(tests/golden/make_golden.py ran ctapsim in the build container)."""

import numpy as np
import pytest

from conftest import load_golden, oracle_grid
from oracle import potential as opot
from oracle import split_step as orc


def test_units_match_reference_repr():
    # measured repr of the reference's Li-6 units
    m = orc.MASSES["li6"]
    assert orc.unit_time(m) == 9.471427012239201e-05
    assert orc.unit_energy(m) == 1.1134244251509448e-30
    assert 1e-6 / orc.unit_time(m) == 0.01055807111967158


def test_plan_factors_bitwise():
    d = load_golden("ctap_scaled_32x16x32.npz")
    g = oracle_grid(d)
    f = orc.make_factors(g, d["V"], float(d["mass"]), float(d["dt"]))
    assert np.array_equal(f.exp_v_half, d["exp_v_half"])
    assert np.array_equal(f.exp_v_full, d["exp_v_full"])
    assert np.array_equal(f.exp_k, d["exp_k"])


@pytest.mark.parametrize("name", ["ctap_scaled_32x16x32.npz", "ioffe_32x16x32.npz"])
def test_evolution_and_trace_bitwise(name):
    d = load_golden(name)
    g = oracle_grid(d)
    f = orc.make_factors(g, d["V"], float(d["mass"]), float(d["dt"]))
    amps, rows = orc.evolve_with_trace(d["psi0"].copy(), g, f, int(d["steps"]), int(d["stride"]),
                                       d["xb1"], d["xb2"])
    assert np.array_equal(amps, d["psi"])
    assert np.array_equal(rows, d["trace"])


def test_harmonic_bitwise():
    d = load_golden("harmonic_16x16x32.npz")
    g = oracle_grid(d)
    f = orc.make_factors(g, d["V"], float(d["mass"]), float(d["dt"]))
    amps = orc.evolve(d["psi0"].copy(), f, int(d["steps"]))
    assert np.array_equal(amps, d["psi"])


def test_gaussian_and_bench_potential():
    d = load_golden("harmonic_16x16x32.npz")
    g = oracle_grid(d)
    c = [g.origin[i] + g.extents[i] / 2 for i in range(3)]
    assert np.array_equal(orc.gaussian_packet(g, c, [e / 16 for e in g.extents]), d["psi0"])
    assert np.array_equal(orc.bench_potential(g, float(d["mass"]), 5.0), d["V"])
    d = load_golden("gaussian_8x8x16.npz")
    g = oracle_grid(d)
    a = orc.gaussian_packet(g, (0.1e-6, -0.2e-6, 0.3e-6), (0.6e-6, 0.5e-6, 1.1e-6),
                            momentum=(1e6, -2e6, 3e5))
    assert np.array_equal(a, d["amps"])


def test_observables_bitwise():
    d = load_golden("observables_16x8x8.npz")
    g = oracle_grid(d)
    assert orc.populations(d["amps"], g, d["xb1"], d["xb2"]) == tuple(d["pops"])
    for m, e in zip(d["margins"], d["edges"]):
        assert orc.edge_density(d["amps"], g, int(m)) == e
    assert orc.norm(d["amps"], g) == float(d["norm"])
    assert np.array_equal(orc.density_xz(d["amps"], g), d["density_xz"])


def test_energies_and_ground_state():
    d = load_golden("imag_16.npz")
    g = oracle_grid(d)
    m = float(d["mass"])
    assert orc.kinetic_expectation(d["seed"], g, m) == float(d["e_seed_t"])
    assert orc.potential_expectation(d["seed"], d["V"]) == float(d["e_seed_v"])
    gs, _ = orc.ground_state_imaginary(g, d["V"], d["seed"], tol=float(d["tol"]),
                                       tau=float(d["tau"]), mass=m)
    assert np.array_equal(gs, d["gs"])
    assert orc.energy_expectation(gs, g, d["V"], m) == float(d["e_gs"])


def test_potential_oracle_bitwise():
    d = load_golden("ctap_scaled_32x16x32.npz")
    chip = load_golden("segments_scaled.npz")
    g = oracle_grid(d)
    v = opot.potential_from_chip(chip, g.axis(0), g.axis(1), g.axis(2))
    assert np.array_equal(v, d["V"])
