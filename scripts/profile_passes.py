"""Launch each split-step pass kind twice (warm-up + profiled) for ncu.

usage: python scripts/profile_passes.py NX NY NZ
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

nx, ny, nz = (int(v) for v in sys.argv[1:4])
grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
# Ioffe floor + an anisotropic harmonic trap (config-2b shape): phases vary
# from point to point like the CTAP potential's (a flat V would make every
# sincos-table gather hit one line)
m = species_mass("li6")
x, y, z = (torch.as_tensor(a, device="cuda") for a in grid.meshgrid())
om = 2 * 3.141592653589793 * torch.tensor([2e3, 2e4, 20.0], dtype=torch.float64)
v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 500e-6) ** 2)
plan = propagator.make_plan(grid, v, m, 1e-6)
psi = torch.randn(nx, ny, nz, dtype=torch.complex128, device="cuda")
kinds = [int(k) if k.isdigit() else getattr(_lib, 'PASS_' + k) for k in (sys.argv[4].split(',') if len(sys.argv) > 4 else ['Z_MID', 'Y_FWD', 'X_KIN', 'Z_FWD', 'Z_FIRST'])]
for kind in kinds:
    for _ in range(2):
        plan.native.run_pass(kind, psi, psi)
torch.cuda.synchronize()
print("ok")
