"""ms per step of plan.advance(psi, K) at a grid size (CUDA events), to compare
switches such as CTAP_GRAPHS=0/1.  usage: python scripts/advance_timing.py NX NY NZ K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

nx, ny, nz, K = (int(v) for v in sys.argv[1:5])
grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
v = torch.full((nx, ny, nz), muB / 2 * 0.03, dtype=torch.float64, device="cuda") + 1e-31
plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6)
psi = (torch.randn(nx, ny, nz, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
for _ in range(2):
    plan.native.advance(psi, K)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
plan.native.advance(psi, K)
b.record()
torch.cuda.synchronize()
print(f"{nx}x{ny}x{nz} K={K} graphs={os.environ.get('CTAP_GRAPHS', '1')}: {a.elapsed_time(b) / K:.4f} ms/step")
