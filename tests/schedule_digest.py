"""Helper of tests/test_gpu_pblock.py (run in a subprocess, the step
schedule is chosen from the environment at plan time): evolve a seeded
256^3 case through evolve_real with a PopulationRecorder and print a JSON
digest of the final psi and of the trace rows."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1309_2451_b200 import observables, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass


def main():
    n, steps, stride = (int(v) for v in sys.argv[1:4])
    precision = sys.argv[4] if len(sys.argv) > 4 else "complex128"
    m = species_mass("li6")
    grid = qgrid.make_grid(n, n, n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n / 2, 0.0))
    x, y, z = grid.meshgrid()
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 5e-4) ** 2)
    plan = propagator.make_plan(grid, v, m, 1e-6, precision=precision)
    part = observables.symmetric_partition(grid, 3.5e-6)
    psi = qgrid.gaussian_packet(grid, (-3.5e-6, 2e-6, 5e-4), (0.3e-6, 0.3e-6, 40e-6))
    rec = observables.PopulationRecorder(part, stride=stride)
    psi, _ = propagator.evolve_real(psi, plan, steps, [rec])
    d = psi.device_amplitudes(None)
    r = torch.view_as_real(d).contiguous()
    bits = int((r.view(torch.int64) if r.dtype == torch.float64 else r.view(torch.int32).to(torch.int64)).sum().item())
    rows = rec.trace.as_array()
    print(json.dumps({"psi_bits": bits, "rows": rows.tolist()}))


if __name__ == "__main__":
    main()
