"""Small propagation that touches every kernel family (z passes, y/x tile
passes, the warp-per-line ring x pass, reductions, 3D FFT) for
compute-sanitizer runs:

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python scripts/sanitize_case.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_1309_2451_b200 import observables, propagator, qgrid
from paper_1309_2451_b200.constants import species_mass

M = species_mass("li6")
for n in ((512, 8, 16), (256, 16, 16), (32, 16, 64)):
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    rng = np.random.default_rng(1)
    v = 1e-30 * (1.0 + rng.random(n))
    psi = qgrid.Wavefunction(rng.standard_normal(n) + 1j * rng.standard_normal(n), grid)
    plan = propagator.make_plan(grid, v, M, 1e-6)
    rec = observables.PopulationRecorder(observables.symmetric_partition(grid, 3.5e-6), stride=2)
    psi, _ = propagator.evolve_real(psi, plan, 3, [rec])
    e = propagator.kinetic_expectation(psi, M)
    print(n, "ok", len(rec.trace), f"{e:.3e}", flush=True)
