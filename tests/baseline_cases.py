"""BASELINE.json's configurations as parity cases (TEST INFRASTRUCTURE ONLY).

Each case builds the inputs of one configuration, runs the
CUDA path through the package's public API (make_plan, evolve_real,
PopulationRecorder) and the CPU oracle (oracle/split_step.py, the reference's
algorithm restated and pinned to the reference's own outputs) on the same
inputs, and reports the north_star gates:

    psi relative L2 <= 1e-10, every trace row's p_l, p_m, p_r within 1e-9
    (complex64: 1e-4 against the complex128 oracle).

Used by tests/test_gpu_baseline_configs.py (driver-run `-m gpu`, bounded step
counts) and scripts/parity_run.py (the long runs, e.g. config 2's 25,000
steps).  Reference: /root/reference/pkg/src/ctapsim/propagator.py:134-173
(evolve_real), runner.py:182-229 (run_evolve), configs/*.cfg.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from oracle import potential as opot
from oracle import split_step as orc
from paper_1309_2451_b200 import chip, magfield, observables, propagator, qgrid
from paper_1309_2451_b200.constants import hbar, muB, species_mass

M = species_mass("li6")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GATES = {"complex128": (1e-10, 1e-9), "complex64": (1e-4, 1e-4)}


def _grid(n, z_max):
    og = orc.Grid(tuple(n), (20e-6, 4e-6, z_max), (-10e-6, 4e-6 / n[1] / 2, 0.0))
    return og, qgrid.SimGrid(og.n, og.extents, og.origin)


def chip_potential(grid, og, name, every: int | None):
    """V from the device Biot-Savart kernel on the product-side chip geometry,
    checked bit for bit against the oracle's C restatement of the numba
    kernel (all points, or every `every`-th point along each axis)."""
    v = magfield.potential_values(chip.chip_segments(name), grid)
    ch = dict(np.load(os.path.join(GOLDEN, f"segments_{name}.npz")))
    if every is None:
        ref = opot.potential_from_chip(ch, og.axis(0), og.axis(1), og.axis(2))
        got = v.cpu().numpy()
    else:
        sl = slice(every // 2, None, every)
        ref = opot.potential_from_chip(ch, og.axis(0)[sl], og.axis(1)[sl], og.axis(2)[sl])
        got = v[sl, sl, sl].cpu().numpy()
    return v, {"points": int(ref.size), "bitwise_equal": bool(np.array_equal(got, ref)),
               "sampled": "all" if every is None else f"every {every}th"}


def cfg1():
    og, grid = _grid((64, 64, 64), 1000e-6)
    v = orc.bench_potential(og, M, 5.0)
    c = [og.origin[i] + og.extents[i] / 2 for i in range(3)]
    a0 = orc.gaussian_packet(og, c, [e / 16 for e in og.extents])
    return dict(name="cfg1 64^3 harmonic", grid=grid, og=og, v=v, a0=a0, stride=50, half_gap=3.5e-6)


def cfg2b():
    og, grid = _grid((128, 128, 256), 250e-6)
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = og.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    a0 = orc.gaussian_packet(og, (-4.4e-6, 2e-6, 125e-6), np.sqrt(hbar / (M * om)))
    return dict(name="cfg2b 128x128x256 Ioffe harmonic (population-moving)", grid=grid, og=og, v=v, a0=a0,
                stride=25, half_gap=3.5e-6)


def cfg2(every=None):
    og, grid = _grid((128, 128, 256), 250e-6)
    v, check = chip_potential(grid, og, "scaled", every)
    a0 = orc.gaussian_packet(og, (-7e-6, 2e-6, 60e-6), (0.3e-6, 0.3e-6, 9.2e-6))
    return dict(name="cfg2 128x128x256 scaled-chip CTAP", grid=grid, og=og, v=v, a0=a0, stride=50,
                half_gap=3.5e-6, v_check=check)


def cfg3(every=8):
    og, grid = _grid((256, 256, 256), 1000e-6)
    v, check = chip_potential(grid, og, "paper", every)
    a0 = orc.gaussian_packet(og, (-7e-6, 1.43e-6, 200e-6), (0.25e-6, 0.12e-6, 15e-6))
    return dict(name="cfg3 256^3 paper-chip CTAP", grid=grid, og=og, v=v, a0=a0, stride=100, half_gap=3.5e-6,
                v_check=check)


def cfg4(every=16):
    og, grid = _grid((512, 512, 512), 1000e-6)
    v, check = chip_potential(grid, og, "paper", every)
    a0 = orc.gaussian_packet(og, (-7e-6, 1.43e-6, 200e-6), (0.25e-6, 0.12e-6, 15e-6))
    return dict(name="cfg4 512^3 paper-chip CTAP", grid=grid, og=og, v=v, a0=a0, stride=50, half_gap=3.5e-6,
                v_check=check)


def cfg5():
    """BASELINE config 5 grid (1024 x 1024 x 512) with run_bench's harmonic
    trap ("harmonic synthetic"), a Gaussian packet; ~50 GB of
    host RAM on the oracle side, so a few steps only."""
    og, grid = _grid((1024, 1024, 512), 1000e-6)
    v = orc.bench_potential(og, M, 5.0)
    a0 = orc.gaussian_packet(og, (-2e-6, 2e-6, 500e-6), (1e-6, 0.3e-6, 40e-6))
    return dict(name="cfg5 1024x1024x512 harmonic", grid=grid, og=og, v=v, a0=a0, stride=5, half_gap=3.5e-6)


def run_case(case, steps: int, stride: int | None = None, precision: str = "complex128") -> dict:
    """GPU (public API, host psi in / out) then the oracle on the same inputs."""
    grid, og, v, a0 = case["grid"], case["og"], case["v"], case["a0"]
    stride = stride or case["stride"]
    part = observables.symmetric_partition(grid, case["half_gap"])
    psi = qgrid.Wavefunction(a0.copy(), grid)
    plan = propagator.make_plan(grid, v, M, 1e-6, precision=precision)
    rec = observables.PopulationRecorder(part, stride=stride)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    psi, stats = propagator.evolve_real(psi, plan, steps, [rec])
    got = psi.amplitudes.astype(np.complex128)
    t_gpu = time.perf_counter() - t0
    rows_gpu = rec.trace.as_array()
    del plan, psi
    torch.cuda.empty_cache()
    v_host = v.cpu().numpy() if isinstance(v, torch.Tensor) else v
    t0 = time.perf_counter()
    f = orc.make_factors(og, v_host, M, 1e-6)
    t_plan = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref, rows = orc.evolve_with_trace(a0.copy(), og, f, steps, stride, part.xb1, part.xb2)
    t_cpu = time.perf_counter() - t0
    del f
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    dpop = float(np.abs(rows_gpu[:, 1:4] - rows[:, 1:4]).max())
    gate_psi, gate_pop = GATES[precision]
    out = {
        "case": case["name"], "grid": list(grid.n), "steps": steps, "stride": stride, "precision": precision,
        "rel_l2": rel, "max_population_diff": dpop,
        "max_norm_diff": float(np.abs(rows_gpu[:, 4] - rows[:, 4]).max()),
        "max_edge_diff": float(np.abs(rows_gpu[:, 5] - rows[:, 5]).max()),
        "times_equal": bool(np.array_equal(rows_gpu[:, 0], rows[:, 0])),
        "trace_rows": int(len(rows)), "rows_match": bool(rows_gpu.shape == rows.shape),
        "final_populations_gpu": rows_gpu[-1, 1:4].tolist(),
        "final_populations_cpu": rows[-1, 1:4].tolist(),
        "population_range_p_l": [float(rows[:, 1].min()), float(rows[:, 1].max())],
        "gpu_seconds": t_gpu, "gpu_steps_per_s": steps / t_gpu,
        "cpu_seconds": t_cpu, "cpu_steps_per_s": steps / t_cpu, "cpu_plan_seconds": t_plan,
        "cpu_threads": os.cpu_count(), "gates": [gate_psi, gate_pop],
        "pass": bool(rel <= gate_psi and dpop <= gate_pop and np.array_equal(rows_gpu[:, 0], rows[:, 0])),
    }
    if "v_check" in case:
        out["potential_check"] = case["v_check"]
        out["pass"] = out["pass"] and case["v_check"]["bitwise_equal"]
    return out
