"""Device time of observed evolve_real segments (A/B of step schedules).

usage: python scripts/segment_timing.py N STEPS STRIDE
Runs evolve_real on an N^3 harmonic case with a PopulationRecorder every
STRIDE steps, psi resident on the device, and prints ms per step (CUDA
events), after one untimed warm-up run of the same length.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1309_2451_b200 import observables, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass


def main():
    n, steps, stride = (int(v) for v in sys.argv[1:4])
    m = species_mass("li6")
    grid = qgrid.make_grid(n, n, n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n / 2, 0.0))
    x, y, z = (torch.as_tensor(a, device="cuda") for a in grid.meshgrid())
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 5e-4) ** 2)
    del x, y, z
    plan = propagator.make_plan(grid, v, m, 1e-6)
    part = observables.symmetric_partition(grid, 3.5e-6)
    psi = qgrid.gaussian_packet(grid, (-3.5e-6, 2e-6, 5e-4), (0.3e-6, 0.3e-6, 40e-6))
    for timed in (False, True):
        rec = observables.PopulationRecorder(part, stride=stride)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        psi, _ = propagator.evolve_real(psi, plan, steps, [rec])
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    print(f"{n}^3 {steps} steps, observer every {stride}: {ms:.4f} ms/step = {1000 / ms:.1f} steps/s; "
          f"last row {rec.trace.as_array()[-1].tolist()}")


if __name__ == "__main__":
    main()
