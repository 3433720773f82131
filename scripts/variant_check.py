"""Cross-check of pass variants selected by environment switches.

usage: CTAP_WPC=1 python scripts/variant_check.py NX NY NZ OUT.pt
Runs X_FWD, X_INV, X_KIN, Y_FWD, Y_INV on the same seeded field and saves the
results; compare two runs with --compare A.pt B.pt (max rel L2 printed).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch


def run(nx, ny, nz, out):
    from paper_1309_2451_b200 import _lib, propagator, qgrid
    from paper_1309_2451_b200.constants import muB, species_mass
    grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    prec = os.environ.get("CTAP_PRECISION", "complex128")
    g = torch.Generator(device="cpu").manual_seed(7)
    v = (muB / 2 * 0.03 * (1 + torch.rand(nx, ny, nz, generator=g, dtype=torch.float64))).cuda()
    plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6, phase_tables=0, precision=prec)
    psi0 = torch.complex(torch.randn(nx, ny, nz, generator=g, dtype=torch.float64),
                         torch.randn(nx, ny, nz, generator=g, dtype=torch.float64))
    psi0 = psi0.to(propagator.PRECISIONS[prec]).cuda()
    res = {}
    for name in ("X_FWD", "X_INV", "X_KIN", "Y_FWD", "Y_INV"):
        psi = psi0.clone()
        plan.native.run_pass(getattr(_lib, "PASS_" + name), psi, psi)
        res[name] = psi.cpu()
    # torch FFT references for the pure transforms
    ref = {"X_FWD": torch.fft.fft(psi0, dim=0), "Y_FWD": torch.fft.fft(psi0, dim=1),
           "X_INV": torch.fft.ifft(psi0, dim=0) * nx, "Y_INV": torch.fft.ifft(psi0, dim=1) * ny}
    for k, r in ref.items():
        r = r.cpu()
        print(f"{k}: rel L2 vs torch.fft = {float((res[k] - r).norm() / r.norm()):.3e}")
    torch.save(res, out)


def compare(a, b):
    A, B = torch.load(a), torch.load(b)
    worst = 0.0
    for k in A:
        rel = float((A[k] - B[k]).norm() / B[k].norm())
        worst = max(worst, rel)
        print(f"{k}: rel L2 = {rel:.3e}  bitwise={bool(torch.equal(A[k], B[k]))}")
    print(f"worst {worst:.3e}")


if __name__ == "__main__":
    if sys.argv[1] == "--compare":
        compare(sys.argv[2], sys.argv[3])
    else:
        run(*(int(x) for x in sys.argv[1:4]), sys.argv[4])
