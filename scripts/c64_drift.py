"""Norm drift and deviation of complex64 against complex128 over many steps
(diagnostic for the c64 rounding design).  usage: python scripts/c64_drift.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1309_2451_b200 import propagator, qgrid
from paper_1309_2451_b200.constants import hbar, muB, species_mass

M = species_mass("li6")
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
grid = qgrid.make_grid(128, 128, 256, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / 256, 0.0))
om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
x, y, z = grid.meshgrid()
v = muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 125e-6) ** 2)
a0 = qgrid.gaussian_packet(grid, (-4.4e-6, 2e-6, 125e-6), np.sqrt(hbar / (M * om))).amplitudes
res = {}
for prec in ("complex128", "complex64"):
    plan = propagator.make_plan(grid, v, M, 1e-6, precision=prec)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    n0 = psi.norm()
    psi, _ = propagator.evolve_real(psi, plan, steps)
    res[prec] = psi.amplitudes.astype(np.complex128)
    print(prec, "norm drift", psi.norm() / n0 - 1.0, flush=True)
d = res["complex64"] - res["complex128"]
print("c64 vs c128 rel L2", np.linalg.norm(d) / np.linalg.norm(res["complex128"]),
      "tma", os.environ.get("CTAP_TMA", "default"))
