"""Config 5 of SURVEY §8(d): (nx, ny, nz) = (1024, 1024, 512), harmonic trap
of runner.run_bench (runner.py:284-292), on one B200.

    python scripts/config5.py [--steps 40] [--parity-steps 4] [--shape 1024 1024 512]
        [--out gpurun_out/config5.json]

* Throughput: device-timed steps/s of the single-GPU propagator (CUDA events
  around plan.advance, K steps after warm-up), against the 136 B/pt roofline.
* Self-parity: the slab decomposition with P = 2 and 8 virtual ranks on the
  same GPU (peer-major y passes, y-slab x pass, the all-to-all emulated by
  device copies, ranks run one after another) must equal P = 1 bit for bit
  (SURVEY gate: <= 1e-12).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_1309_2451_b200 import propagator, qgrid
from paper_1309_2451_b200.constants import species_mass
from paper_1309_2451_b200.propagator import NativePlan
from paper_1309_2451_b200.slab import SlabLayout, segment_schedule

M = species_mass("li6")
HBM_PEAK = 6544.0


def harmonic_on_device(grid, omega_z):
    """0.5 m wz^2 |r - c|^2 (runner.run_bench) evaluated on the device."""
    ax = [torch.from_numpy(np.asarray(grid.axis(i))).cuda() for i in range(3)]
    c = [o + e / 2 for o, e in zip(grid.origin, grid.extents)]
    dx = (ax[0] - c[0])[:, None, None] ** 2
    dy = (ax[1] - c[1])[None, :, None] ** 2
    dz = (ax[2] - c[2])[None, None, :] ** 2
    return (0.5 * M * omega_z ** 2) * ((dx + dy) + dz)


def packet_on_device(grid):
    """Separable normalized Gaussian at the box centre, widths extents/16."""
    c = [o + e / 2 for o, e in zip(grid.origin, grid.extents)]
    f = []
    for i in range(3):
        s = grid.extents[i] / 16
        a = torch.from_numpy(np.asarray(grid.axis(i))).cuda()
        f.append(torch.exp(-((a - c[i]) ** 2) / (4 * s * s)).to(torch.complex128))
    psi = f[0][:, None, None] * f[1][None, :, None] * f[2][None, None, :]
    psi /= torch.sqrt(torch.sum(torch.abs(psi) ** 2) * grid.dvol)
    return psi.contiguous()


def run_virtual(grid, v, a0, P, steps):
    lays = [SlabLayout(grid.n, P, r) for r in range(P)]
    plans = [NativePlan(grid, v[l.x_slice].contiguous(), M, 1e-6, slab_p=P, slab_r=r)
             for r, l in enumerate(lays)]
    bufs = [{"psi": a0[l.x_slice].clone().reshape(-1),  # (a slab view would alias a0)
             "send": torch.empty(l.points, dtype=torch.complex128, device="cuda"),
             "recv": torch.empty(l.points, dtype=torch.complex128, device="cuda")} for l in lays]
    chunk = lays[0].points // P
    for op in segment_schedule(steps):
        if op[0] == "pass":
            for r in range(P):
                plans[r].run_pass(op[1], bufs[r][op[2]], bufs[r][op[3]])
        else:
            src, dst = op[1], op[2]
            for q in range(P):
                for p in range(P):
                    bufs[q][dst][p * chunk:(p + 1) * chunk].copy_(bufs[p][src][q * chunk:(q + 1) * chunk])
    torch.cuda.synchronize()
    out = torch.cat([b["psi"] for b in bufs]).reshape(grid.n)
    del plans, bufs
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", type=int, nargs=3, default=[1024, 1024, 512])
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--parity-steps", type=int, default=4)
    ap.add_argument("--ranks", type=int, nargs="*", default=[2, 8])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "config5.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    n = tuple(args.shape)
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    v = harmonic_on_device(grid, 2 * np.pi * 5.0)
    a0 = packet_on_device(grid)
    N = grid.size
    res = {"shape": list(n), "points": N, "psi_gib": N * 16 / 2 ** 30}

    # single-GPU throughput (device time, CUDA events)
    plan = propagator.make_plan(grid, v, M, 1e-6)
    psi = a0.clone()
    plan.native.advance(psi, 5)
    plan.native.advance(psi, args.steps)  # graph capture happens on first use of this count
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    plan.native.advance(psi, args.steps)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    res["ms_per_step"] = ms
    res["steps_per_s"] = 1e3 / ms
    res["hbm_fraction_136B"] = 136.0 * N / (ms * 1e-3) / (HBM_PEAK * 1e9)
    print(json.dumps(res), flush=True)
    del psi

    # self-parity: P virtual slab ranks vs P = 1, bit for bit
    ref = a0.clone()
    plan.native.advance(ref, args.parity_steps)
    torch.cuda.synchronize()
    del plan
    torch.cuda.empty_cache()
    res["parity_steps"] = args.parity_steps
    res["self_parity"] = {}
    for P in args.ranks:
        t0 = time.perf_counter()
        got = run_virtual(grid, v, a0, P, args.parity_steps)
        rel = float(torch.linalg.vector_norm(got - ref) / torch.linalg.vector_norm(ref))
        res["self_parity"][str(P)] = {"bitwise_equal": bool(torch.equal(got, ref)), "rel_l2": rel,
                                      "seconds": time.perf_counter() - t0}
        del got
        torch.cuda.empty_cache()
        print(json.dumps({"P": P, **res["self_parity"][str(P)]}), flush=True)
    res["pass"] = all(r["rel_l2"] <= 1e-12 for r in res["self_parity"].values())
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
