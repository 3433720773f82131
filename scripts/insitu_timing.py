"""Per-pass device time IN SEQUENCE (z_mid, y, x_kin, y^-1 repeated, events
between the launches) next to the same passes timed in isolation.

usage: python scripts/insitu_timing.py NX NY NZ [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass


def main():
    nx, ny, nz = (int(v) for v in sys.argv[1:4])
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    v = torch.full((nx, ny, nz), muB / 2 * 0.03, dtype=torch.float64, device="cuda")
    v += torch.rand_like(v) * 1e-29
    plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6)
    psi = (torch.randn(nx, ny, nz, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
    seq = [("Z_MID", _lib.PASS_Z_MID), ("Y_FWD", _lib.PASS_Y_FWD), ("X_KIN", _lib.PASS_X_KIN),
           ("Y_INV", _lib.PASS_Y_INV)]
    for _ in range(3):
        for _, k in seq:
            plan.native.run_pass(k, psi, psi)
    def time_advance(label):
        for _ in range(2):
            plan.native.advance(psi, steps)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s0.record()
        plan.native.advance(psi, steps)
        s1.record()
        torch.cuda.synchronize()
        print(label, round(s0.elapsed_time(s1) / steps, 4), "ms/step")

    if os.environ.get("INSITU_ADVANCE_FIRST"):
        time_advance("advance first:")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4 * steps + 1)]
    torch.cuda.synchronize()
    ev[0].record()
    i = 1
    for _ in range(steps):
        for _, k in seq:
            plan.native.run_pass(k, psi, psi)
            ev[i].record()
            i += 1
    torch.cuda.synchronize()
    tot = {n: 0.0 for n, _ in seq}
    for s in range(steps):
        for j, (n, _) in enumerate(seq):
            a = 4 * s + j
            tot[n] += ev[a].elapsed_time(ev[a + 1])
    print("in sequence  :", {n: round(t / steps, 4) for n, t in tot.items()},
          "sum", round(sum(tot.values()) / steps, 4))
    iso = {}
    for n, k in seq:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(steps):
            plan.native.run_pass(k, psi, psi)
        s1.record()
        torch.cuda.synchronize()
        iso[n] = s0.elapsed_time(s1) / steps
    print("in isolation :", {n: round(t, 4) for n, t in iso.items()}, "sum", round(sum(iso.values()), 4))
    time_advance("advance      :")


if __name__ == "__main__":
    main()
