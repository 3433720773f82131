"""Time and fingerprint plan.advance under the current environment switches.

usage: CTAP_ZCHUNK=16 python scripts/advance_variant.py NX NY NZ [steps]
Prints ms/step (CUDA events, after a warm-up of the same length) and a hash
of psi after `steps` steps from a seeded state, so runs with different
switches can be checked for bitwise equality.
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1309_2451_b200 import propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass


def main():
    nx, ny, nz = (int(v) for v in sys.argv[1:4])
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    prec = os.environ.get("CTAP_PRECISION", "complex128")
    grid = qgrid.make_grid(nx, ny, nz, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / ny / 2, 0.0))
    g = torch.Generator(device="cuda").manual_seed(5)
    v = muB / 2 * 0.03 * (1 + 0.01 * torch.rand(nx, ny, nz, generator=g, device="cuda", dtype=torch.float64))
    plan = propagator.make_plan(grid, v, species_mass("li6"), 1e-6, precision=prec)
    psi0 = torch.complex(torch.randn(nx, ny, nz, generator=g, device="cuda", dtype=torch.float64),
                         torch.randn(nx, ny, nz, generator=g, device="cuda", dtype=torch.float64))
    psi = psi0.to(propagator.PRECISIONS[prec]).contiguous()
    ref = psi.clone()
    plan.native.advance(ref, steps)
    torch.cuda.synchronize()
    h = hashlib.sha256(ref.cpu().numpy().tobytes()).hexdigest()[:16]
    plan.native.advance(psi, steps)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    plan.native.advance(psi, steps)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    print(f"{prec} {nx}x{ny}x{nz} zchunk={os.environ.get('CTAP_ZCHUNK', '0')}: {ms:.3f} ms/step "
          f"({1e3 / ms:.1f} steps/s) hash {h}")


if __name__ == "__main__":
    main()
