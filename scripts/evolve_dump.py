"""Run a short propagation on fixed inputs and save psi (for comparing two
builds bit for bit).  usage: python scripts/evolve_dump.py NX NY NZ STEPS OUT.npy [complex64]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_1309_2451_b200 import propagator, qgrid
from paper_1309_2451_b200.constants import species_mass

nx, ny, nz, steps = (int(v) for v in sys.argv[1:5])
prec = sys.argv[6] if len(sys.argv) > 6 else "complex128"
g = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
r = np.random.default_rng(4)
v = 3e-27 * (1 + r.random((nx, ny, nz)))
w = qgrid.Wavefunction(r.standard_normal((nx, ny, nz)) + 1j * r.standard_normal((nx, ny, nz)), g)
w, _ = propagator.evolve_real(w, propagator.make_plan(g, v, species_mass("li6"), 1e-6, precision=prec), steps)
np.save(sys.argv[5], w.amplitudes)
print("saved", sys.argv[5])
