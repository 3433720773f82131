"""Probe: the TMA-ring x pass and an LSU y pass running concurrently on two
streams on different buffers (does the ring leave HBM bandwidth and SMs a
y pass can use?).  usage: CTAP_RING_SMS=n python scripts/overlap_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

n = 512
grid = qgrid.make_grid(n, n, n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n / 2, 0.0))
v = torch.full((n, n, n), muB / 2 * 0.03, dtype=torch.float64, device="cuda")
plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6).native
a = (torch.randn(n, n, n, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
b = (torch.randn(n, n, n, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def x_only():
    plan.run_pass(_lib.PASS_X_KIN, a, a)


def y_only():
    plan.run_pass(_lib.PASS_Y_FWD, b, b)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        plan.run_pass(_lib.PASS_X_KIN, a, a)
    with torch.cuda.stream(s2):
        plan.run_pass(_lib.PASS_Y_FWD, b, b)
        plan.run_pass(_lib.PASS_Y_INV, b, b)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


def seq():
    plan.run_pass(_lib.PASS_X_KIN, a, a)
    plan.run_pass(_lib.PASS_Y_FWD, b, b)
    plan.run_pass(_lib.PASS_Y_INV, b, b)


print(f"ring SMs {os.environ.get('CTAP_RING_SMS', 'all')}: x {timed(x_only):.3f}  y {timed(y_only):.3f}  "
      f"x + 2y sequential {timed(seq):.3f}  concurrent {timed(both):.3f} ms")
