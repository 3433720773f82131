"""Launch the segment-end z pass plain and with the fused observer sums (for ncu).

usage: python scripts/profile_obs.py N
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1309_2451_b200 import _device, _lib, observables, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
grid = qgrid.make_grid(n, n, n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n / 2, 0.0))
m = species_mass("li6")
x, y, z = (torch.as_tensor(a, device="cuda") for a in grid.meshgrid())
om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 5e-4) ** 2)
del x, y, z
plan = propagator.make_plan(grid, v, m, 1e-6).native
psi = (torch.randn(n, n, n, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
part = observables.symmetric_partition(grid, 3.5e-6)
xs = _device.to_device_f64(grid.x)
b1, b2 = _device.to_device_f64(part.xb1), _device.to_device_f64(part.xb2)
for _ in range(2):
    plan.run_pass(_lib.PASS_Z_LAST, psi, psi)
    plan.advance_observe(psi, 1, xs, b1, b2, 2)
torch.cuda.synchronize()
print("ok")
