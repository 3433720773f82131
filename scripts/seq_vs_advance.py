"""Same kernels, two launch paths: a Python loop of the four step passes
(ctap_pass) vs ctap_advance (graph-captured chunks), K steps each, CUDA
events around the whole loop only.  usage: python scripts/seq_vs_advance.py K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n = 512
grid = qgrid.make_grid(n, n, n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n / 2, 0.0))
v = torch.full((n, n, n), muB / 2 * 0.03, dtype=torch.float64, device="cuda") + 1e-31
plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6)
psi = (torch.randn(n, n, n, dtype=torch.complex128, device="cuda") * 1e-3).contiguous()
seq = [_lib.PASS_Y_FWD, _lib.PASS_X_KIN, _lib.PASS_Y_INV, _lib.PASS_Z_MID]


def manual():
    for _ in range(K):
        for k in seq:
            plan.native.run_pass(k, psi, psi)


def adv():
    plan.native.advance(psi, K)


for rep in range(2):
    for name, fn in (("manual", manual), ("advance", adv)):
        fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{name:8s} {a.elapsed_time(b) / K:.4f} ms/step", flush=True)
