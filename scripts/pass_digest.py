"""Bitwise digest of one pass on a seeded random psi (A/B of kernel variants).

usage: python scripts/pass_digest.py NX NY NZ PASS [PASS ...]   (PASS: a pass name or ADVANCE<n>)
Prints, per pass name (pass_timing.py's names), an int64 sum of the output's
bit patterns: two kernels are bitwise interchangeable iff their digests match.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass


def main():
    nx, ny, nz = (int(v) for v in sys.argv[1:4])
    m = species_mass("li6")
    grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    x, y, z = (torch.as_tensor(a, device="cuda") for a in grid.meshgrid())
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 5e-4) ** 2)
    del x, y, z
    plan = propagator.make_plan(grid, v, m, 1e-6)
    gen = torch.Generator(device="cuda").manual_seed(7)
    for name in sys.argv[4:]:
        psi = torch.randn(nx, ny, nz, dtype=torch.complex128, device="cuda", generator=gen) * 1e-3
        if name.startswith("ADVANCE"):
            plan.native.advance(psi, int(name[7:] or 20))
        else:
            plan.native.run_pass(getattr(_lib, "PASS_" + name), psi, psi)
        torch.cuda.synchronize()
        d = int(torch.view_as_real(psi).contiguous().view(torch.int64).sum().item())
        print(f"{name} digest {d}")


if __name__ == "__main__":
    main()
