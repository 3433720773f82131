"""Generate the golden fixtures by running the REFERENCE itself (ctapsim).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every array here comes out of the reference's own public functions
(make_grid, make_plan, evolve_real, PopulationRecorder, assemble_potential,
build_partition, ground_state_imaginary, energy_expectation, ...).  The
fixtures pin the oracle (tests/test_oracle_golden.py) and, through it, the
GPU path.  Reference paths: /root/reference/pkg/src/ctapsim/.
"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from ctapsim import chipgeom, config, magfield, observables, propagator, qgrid  # noqa: E402
from ctapsim.constants import hbar, muB, species_mass  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CFG = "/root/reference/pkg/configs"
M = species_mass("li6")


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path) / 1024:.0f} KiB")


def grid_arrays(g):
    return dict(n=np.array(g.n), extents=np.array(g.extents), origin=np.array(g.origin))


def chip_fixture(cfg_name):
    """Segment arrays exactly as assemble_potential concatenates them
    (magfield.py:229-235)."""
    cfg = config.load_config(os.path.join(CFG, cfg_name))
    layout = cfg.to_layout()
    segs = magfield.layout_segments(layout)
    seg_a = np.concatenate([s.a for s in segs])
    seg_b = np.concatenate([s.b for s in segs])
    seg_cur = np.concatenate([np.full(len(s), s.current) for s in segs])
    e = np.asarray(layout.bias_direction, float)
    e = e / np.linalg.norm(e)
    b0 = layout.b_bias * e + np.array([0.0, 0.0, layout.b_ioffe])
    wires = {w.value: layout.wire(w).x_of_z(np.array([0.0]))[0] for w in chipgeom.WireId}
    return cfg, layout, dict(seg_a=seg_a, seg_b=seg_b, seg_cur=seg_cur, b0=b0,
                             mu_eff=layout.mu_eff, mass=layout.mass, omega_z=layout.omega_z,
                             z_center=layout.z_max / 2.0, z_max=layout.z_max,
                             x_span=layout.x_span, pref=magfield.MU0_4PI,
                             wire_x0=np.array([wires["left"], wires["middle"], wires["right"]]))


def main():
    # 1. chip segment arrays (scaled desk chip and the paper chip)
    cfg_s, layout_s, chip_s = chip_fixture("scaled.cfg")
    save("segments_scaled.npz", **chip_s)
    cfg_p, layout_p, chip_p = chip_fixture("paper.cfg")
    save("segments_paper.npz", **chip_p)

    # 2. CTAP potential + partition on a small scaled-chip grid (numba kernel)
    cfg_small = dataclasses.replace(cfg_s, n_x=32, n_y=16, n_z=32)
    grid = cfg_small.to_grid()
    pot = magfield.assemble_potential(layout_s, grid)
    part = observables.build_partition(pot)
    # 3. CTAP propagation: Gaussian in the left guide, 200 steps, trace every 25
    x_l = float(part.xb1[0]) - 3.5e-6
    psi = qgrid.gaussian_packet(grid, (-7e-6, 2e-6, 125e-6), (0.45e-6, 0.3e-6, 12e-6))
    psi0 = psi.amplitudes.copy()
    plan = propagator.make_plan(grid, pot.values, M, 1e-6)
    rec = observables.PopulationRecorder(part, stride=25, margin_cells=2)
    psi, _ = propagator.evolve_real(psi, plan, 200, [rec])
    save("ctap_scaled_32x16x32.npz", **grid_arrays(grid), V=pot.values, xb1=part.xb1,
         xb2=part.xb2, psi0=psi0, psi=psi.amplitudes, trace=rec.trace.as_array(),
         steps=200, stride=25, dt=1e-6, mass=M, x_l=x_l,
         exp_v_half=plan.exp_v_half, exp_v_full=plan.exp_v_full, exp_k=plan.exp_k)

    # 4. population-moving Ioffe-floor harmonic case (SURVEY config 2b, shrunk)
    g2 = qgrid.make_grid(32, 16, 32, (20e-6, 4e-6, 250e-6),
                         origin=(-10e-6, 4e-6 / 16 / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = g2.meshgrid()
    v2 = muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                     + om[2] ** 2 * (z - 125e-6) ** 2)
    widths = np.sqrt(hbar / (M * om))
    psi = qgrid.gaussian_packet(g2, (-4.4e-6, 2e-6, 125e-6), widths)
    psi0 = psi.amplitudes.copy()
    part2 = observables.GuidePartition(xb1=np.full(32, -3.5e-6), xb2=np.full(32, 3.5e-6),
                                       merged=np.zeros(32, bool), grid_ref=g2)
    plan = propagator.make_plan(g2, v2, M, 1e-6)
    rec = observables.PopulationRecorder(part2, stride=25)
    psi, _ = propagator.evolve_real(psi, plan, 300, [rec])
    save("ioffe_32x16x32.npz", **grid_arrays(g2), V=v2, psi0=psi0, psi=psi.amplitudes,
         xb1=part2.xb1, xb2=part2.xb2, trace=rec.trace.as_array(), steps=300, stride=25,
         dt=1e-6, mass=M, widths=widths)

    # 5. harmonic bench-style grid (run_bench synthetic V), 100 steps
    g3 = qgrid.make_grid(16, 16, 32, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / 32, 0.0))
    c = [o + e / 2 for o, e in zip(g3.origin, g3.extents)]
    x, y, z = g3.meshgrid()
    omz = 2 * np.pi * 5.0
    v3 = 0.5 * M * omz ** 2 * ((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
    psi = qgrid.gaussian_packet(g3, c, [e / 16 for e in g3.extents])
    psi0 = psi.amplitudes.copy()
    plan = propagator.make_plan(g3, v3, M, 1e-6)
    psi, _ = propagator.evolve_real(psi, plan, 100)
    save("harmonic_16x16x32.npz", **grid_arrays(g3), V=v3, psi0=psi0, psi=psi.amplitudes,
         steps=100, dt=1e-6, mass=M)

    # 6. imaginary-time ground state + energies (anisotropic HO, small)
    omegas = 2 * np.pi * np.array([3e3, 4e3, 5e3])
    ax = np.sqrt(hbar / (M * omegas[0]))
    g4 = qgrid.make_grid(16, 16, 16, (14 * ax,) * 3, origin=(-7 * ax,) * 3)
    x, y, z = g4.meshgrid()
    v4 = 0.5 * M * (omegas[0] ** 2 * x ** 2 + omegas[1] ** 2 * y ** 2 + omegas[2] ** 2 * z ** 2)
    seed = qgrid.gaussian_packet(g4, (0.3 * ax, -0.2 * ax, 0.1 * ax), (0.9 * ax,) * 3)
    seed_amps = seed.amplitudes.copy()
    e_seed_t = propagator.kinetic_expectation(seed, M)
    e_seed_v = propagator.potential_expectation(seed, v4)
    gs = propagator.ground_state_imaginary(g4, v4, seed.copy(), tol=1e-9, tau=1e-6, mass=M)
    e_gs = propagator.energy_expectation(gs, v4, M)
    save("imag_16.npz", **grid_arrays(g4), V=v4, seed=seed_amps, gs=gs.amplitudes, e_gs=e_gs,
         e_seed_t=e_seed_t, e_seed_v=e_seed_v, tol=1e-9, tau=1e-6, mass=M)

    # 7. observables on a random state (edge margins, populations)
    g5 = qgrid.make_grid(16, 8, 8, (20e-6, 4e-6, 40e-6), origin=(-10e-6, 0.25e-6, 0.0))
    rng = np.random.default_rng(7)
    amps = rng.standard_normal(g5.n) + 1j * rng.standard_normal(g5.n)
    w5 = qgrid.Wavefunction(amps.copy(), g5)
    xb1 = rng.uniform(-6e-6, -1e-6, 8)
    xb2 = rng.uniform(1e-6, 6e-6, 8)
    part5 = observables.GuidePartition(xb1=xb1, xb2=xb2, merged=np.zeros(8, bool), grid_ref=g5)
    pops = observables.populations(w5, part5)
    edges = [observables.edge_density(w5, m) for m in (1, 2, 3, 5)]
    save("observables_16x8x8.npz", **grid_arrays(g5), amps=amps, xb1=xb1, xb2=xb2,
         pops=np.array(pops), edges=np.array(edges), margins=np.array([1, 2, 3, 5]),
         norm=w5.norm(), density_xz=observables.density_xz(w5))

    # 8. gaussian packet with momentum
    g6 = qgrid.make_grid(8, 8, 16, (8e-6, 8e-6, 16e-6), origin=(-4e-6, -4e-6, -8e-6))
    gp = qgrid.gaussian_packet(g6, (0.1e-6, -0.2e-6, 0.3e-6), (0.6e-6, 0.5e-6, 1.1e-6),
                               momentum=(1e6, -2e6, 3e5))
    save("gaussian_8x8x16.npz", **grid_arrays(g6), amps=gp.amplitudes)



def minima_fixtures():
    """Per-slice transverse minima (magfield._find_slice_minima through
    assemble_potential) and build_partition, from the reference."""

    def pack(pot, part=None, wires=None):
        m = pot.minima
        d = dict(V=pot.values, mx=np.array([s.x for s in m]), my=np.array([s.y for s in m]),
                 mv=np.array([s.value for s in m]), mn=np.array([s.n_guides for s in m]))
        if part is not None:
            d.update(xb1=part.xb1, xb2=part.xb2, merged=part.merged, wire_pos=wires)
        return d

    out = {}
    for cfg_name, n, tag in (("scaled.cfg", (64, 32, 64), "scaled"), ("paper.cfg", (64, 32, 64), "paper")):
        cfg = config.load_config(os.path.join(CFG, cfg_name))
        cfg = dataclasses.replace(cfg, n_x=n[0], n_y=n[1], n_z=n[2])
        layout = cfg.to_layout()
        grid = cfg.to_grid()
        pot = magfield.assemble_potential(layout, grid)
        part = observables.build_partition(pot)
        wires = np.array([sorted(layout.wire_positions_at(float(z)).values()) for z in grid.z])
        for k, v in pack(pot, part, wires).items():
            out[f"{tag}_{k}"] = v
        out[f"{tag}_n"] = np.array(grid.n)
        out[f"{tag}_extents"] = np.array(grid.extents)
        out[f"{tag}_origin"] = np.array(grid.origin)
        print(tag, "slices with >=3 minima:", int((pot.minima and sum(s.n_guides >= 3 for s in pot.minima))),
              "merged:", int(part.merged.sum()))
    # synthetic slices: (a) small integer-valued slices full of exact ties
    # (the < / <= pattern), redrawn until a slice has <= 3 minima so the
    # reference's value argsort (whose tie order is numpy-build specific) is
    # not involved, (b) continuous random slices with many minima
    rng = np.random.default_rng(21)
    ties = np.empty((8, 8, 64))
    for k in range(ties.shape[2]):
        while True:
            s = rng.integers(0, 3, size=(8, 8)).astype(float)
            c = s[1:-1, 1:-1]
            cnt = int(((c < s[:-2, 1:-1]) & (c <= s[2:, 1:-1]) & (c < s[1:-1, :-2]) & (c <= s[1:-1, 2:])).sum())
            if cnt <= 3:
                break
        ties[:, :, k] = s
    smooth = rng.standard_normal((64, 32, 16))
    for tag, v in (("ties", ties), ("many", smooth)):
        g = qgrid.make_grid(v.shape[0], v.shape[1], v.shape[2],
                            (20e-6, 4e-6, 100e-6), origin=(-10e-6, 0.1e-6, 0.0))
        pot = magfield.PotentialGrid(values=v, grid=g, layout=None,
                                     minima=tuple(magfield._find_slice_minima(v[:, :, k], g.x, g.y)
                                                  for k in range(v.shape[2])))
        for k, a in pack(pot).items():
            out[f"{tag}_{k}"] = a
        out[f"{tag}_n"] = np.array(g.n)
        out[f"{tag}_extents"] = np.array(g.extents)
        out[f"{tag}_origin"] = np.array(g.origin)
        print(tag, "max minima per slice:", int(out[f"{tag}_mn"].max()))
    save("minima.npz", **out)


def runner_fixtures():
    """transverse_ground_state / initial_state of the evolve pipeline
    (runner.py:114-181) on a 64x32x64 scaled-chip grid, and a short
    evolution from that initial state."""
    from ctapsim import runner

    cfg = config.load_config(os.path.join(CFG, "scaled.cfg"))
    cfg = dataclasses.replace(cfg, n_x=64, n_y=32, n_z=64)
    layout, grid, pot, part = runner.prepare_potential(cfg)
    iz0 = int(np.argmin(np.abs(grid.z - cfg.z_start_eff)))
    spec = magfield.transverse_spectrum(pot, iz0, 0)
    phi = runner.transverse_ground_state(pot, part, iz0, 0, tau=cfg.gs_tau, tol=cfg.gs_tol)
    psi = runner.initial_state(cfg, pot, part)
    psi0 = psi.amplitudes.copy()
    plan = propagator.make_plan(grid, pot.values, cfg.mass, cfg.dt)
    rec = observables.PopulationRecorder(part, stride=50, margin_cells=cfg.edge_margin_cells)
    psi, _ = propagator.evolve_real(psi, plan, 200, [rec])
    wires = np.array([[layout.wire_positions_at(float(z))[k] for k in ("left", "middle", "right")]
                      for z in grid.z])
    save("runner_scaled_64x32x64.npz", **grid_arrays(grid), xb1=part.xb1, xb2=part.xb2,
         merged=part.merged, wire_pos=wires, iz0=iz0, phi=phi, psi0_norm=float(np.sum(np.abs(psi0) ** 2)),
         psi0_center=psi0[:, :, iz0],
         trace=rec.trace.as_array(), spectrum=np.array([spec.omega_x, spec.omega_y, spec.v_min,
                                                         *spec.energies]),
         z_start=cfg.z_start_eff, sigma_z=cfg.sigma_z_eff, gs_tau=cfg.gs_tau, gs_tol=cfg.gs_tol,
         mass=cfg.mass, dt=cfg.dt, edge_margin=cfg.edge_margin_cells)


if __name__ == "__main__":
    if sys.argv[1:] == ["minima"]:
        minima_fixtures()
    elif sys.argv[1:] == ["runner"]:
        runner_fixtures()
    else:
        main()
        minima_fixtures()
        runner_fixtures()
