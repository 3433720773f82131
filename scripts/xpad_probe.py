"""Diagnostic: x-pass time against the x pitch (plane stride) padding.

usage: CTAP_XPAD=P python scripts/xpad_probe.py NX NY NZ
Times the copy-only and kinetic x pass (diagnostic kinds 63/64) on a buffer
whose x planes are ny*nz + P points apart."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

nx, ny, nz = (int(v) for v in sys.argv[1:4])
pad = int(os.environ.get("CTAP_XPAD", "0"))
grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
v = torch.full((nx, ny, nz), muB / 2 * 0.03, dtype=torch.float64, device="cuda")
plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6)
buf = torch.randn(nx * (ny * nz + pad), dtype=torch.complex128, device="cuda")
for kind, name in ((63, "XP_COPY"), (64, "XP_KIN")):
    for _ in range(3):
        plan.native.run_pass(kind, buf, buf)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(20):
        plan.native.run_pass(kind, buf, buf)
    e.record()
    torch.cuda.synchronize()
    print(f"pad={pad:6d} {name}: {s.elapsed_time(e) / 20:.3f} ms", flush=True)
