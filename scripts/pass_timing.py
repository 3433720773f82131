"""Per-pass device timing (CUDA events) of the split-step passes on one GPU.

usage: python scripts/pass_timing.py NX NY NZ [reps]
Prints ms per pass and the achieved GB/s against 32 B/pt (+8 B/pt V for z
passes with a potential phase).
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
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    m = species_mass("li6")
    grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    n = nx * ny * nz
    # Ioffe floor + anisotropic harmonic trap: point-to-point varying phases
    # like the CTAP potential's (a flat V makes every sincos gather hit one line)
    x, y, z = (torch.as_tensor(a, device="cuda") for a in grid.meshgrid())
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2 + om[2] ** 2 * (z - 5e-4) ** 2)
    del x, y, z
    prec = os.environ.get('CTAP_PRECISION', 'complex128')
    plan = propagator.make_plan(grid, v, m, 1e-6, phase_tables=int(os.environ.get('CTAP_PHASE_TABLES', '0')), precision=prec)
    psi = (torch.randn(nx, ny, nz, dtype=propagator.PRECISIONS[prec], device="cuda") * 1e-3).contiguous()
    P = _lib
    passes = [("Z_MID", P.PASS_Z_MID, 40), ("Y_FWD", P.PASS_Y_FWD, 32), ("X_KIN", P.PASS_X_KIN, 32),
              ("Y_INV", P.PASS_Y_INV, 32), ("Z_FIRST", P.PASS_Z_FIRST, 40), ("Z_LAST", P.PASS_Z_LAST, 40),
              ("Z_FWD", P.PASS_Z_FWD, 32), ("X_FWD", P.PASS_X_FWD, 32), ("X_INV", P.PASS_X_INV, 32)]
    kbuf = torch.empty_like(psi)
    passes += [("Y_COPY", 60, 32), ("X_COPY", 61, 32), ("XB_COPY", 62, 32), ("WX_COPY", 65, 32), ("WY_COPY", 66, 32), ("WY_FWD", 67, 32)]
    io = {P.PASS_Y_FWD_BLK: (psi, kbuf), P.PASS_X_KIN_BLK: (kbuf, kbuf), P.PASS_Y_INV_BLK: (kbuf, psi)}
    total = 0.0
    for name, kind, bpp in passes:
        src, dst = io.get(kind, (psi, psi))
        try:
            for _ in range(3):
                plan.native.run_pass(kind, src, dst)
        except Exception as e:  # diagnostic kinds not built for this size / precision
            print(f"{name:8s} n/a ({e.__class__.__name__})")
            continue
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            plan.native.run_pass(kind, src, dst)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        gbs = bpp * (0.5 if prec == "complex64" and bpp % 16 == 0 else 1.0) * n / (ms * 1e-3) / 1e9
        if name in ("Z_MID", "Y_FWD", "X_KIN", "Y_INV"):
            total += ms
        print(f"{name:8s} {ms:8.3f} ms  {gbs:8.1f} GB/s")
    # full steps
    for _ in range(2):
        plan.native.advance(psi, reps)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    plan.native.advance(psi, reps)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"sum of 4 passes {total:.3f} ms; advance {ms:.3f} ms/step = {1000 / ms:.1f} steps/s; "
          f"{136 * n / (ms * 1e-3) / 1e9:.1f} GB/s algorithmic (136 B/pt)")


if __name__ == "__main__":
    main()
