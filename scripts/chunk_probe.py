"""Probe: does running the position block (y^-1, [z^-1 V z], y) per x-plane
chunk, with the chunk L2-resident between its three passes, beat the three
full-volume passes?  Uses one plan for an (W, ny, nz) chunk and nx/W separate
chunk buffers (together the full 2 GiB wavefunction), optionally spread over
several streams.

usage: python scripts/chunk_probe.py NX NY NZ W [streams]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass


def main():
    nx, ny, nz, W = (int(v) for v in sys.argv[1:5])
    ns = int(sys.argv[5]) if len(sys.argv) > 5 else 1
    m = species_mass("li6")
    full = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    sub = qgrid.make_grid(W, ny, nz, (20e-6 * W / nx, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    v = torch.full((W, ny, nz), muB / 2 * 0.03, dtype=torch.float64, device="cuda") + 1e-31
    plan = propagator.make_plan(sub, v, m, 1e-6)
    vf = torch.full((nx, ny, nz), muB / 2 * 0.03, dtype=torch.float64, device="cuda") + 1e-31
    planf = propagator.make_plan(full, vf, m, 1e-6)
    psi = (torch.randn(nx, ny, nz, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
    chunks = [psi[c * W:(c + 1) * W] for c in range(nx // W)]
    P = _lib
    streams = [torch.cuda.Stream() for _ in range(ns)]

    def chunked():
        ev0 = torch.cuda.Event()
        ev0.record()
        for i, ch in enumerate(chunks):
            s = streams[i % ns]
            s.wait_event(ev0)
            with torch.cuda.stream(s):
                for k in (P.PASS_Y_INV, P.PASS_Z_MID, P.PASS_Y_FWD):
                    plan.native.run_pass(k, ch, ch)
        cur = torch.cuda.current_stream()
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            cur.wait_event(e)

    def whole():
        for k in (P.PASS_Y_INV, P.PASS_Z_MID, P.PASS_Y_FWD):
            planf.native.run_pass(k, psi, psi)

    for name, fn in (("whole", whole), ("chunked", chunked)):
        for _ in range(3):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{name:8s} W={W:4d} streams={ns}: {a.elapsed_time(b) / 10:.3f} ms per position block")


if __name__ == "__main__":
    main()
