"""Observer sums fused into the segment-end pass (ctap_advance_observe).

evolve_real asks the last [z^-1 . Vh] pass of each observed segment for the
event's [sum rho, left, middle, right, edge]:
the wavefunction must be bitwise the one ctap_advance leaves, the sums equal
to the standalone reduction's (ctap_observe, a different fixed summation
order) to rounding, and bitwise reproducible run to run.  Reference:
/root/reference/pkg/src/ctapsim/observables.py:74-110, propagator.py:160-168.
"""

import numpy as np
import pytest
import torch

from paper_1309_2451_b200 import _device, observables, propagator, qgrid
from paper_1309_2451_b200.constants import muB, species_mass

pytestmark = pytest.mark.gpu
M = species_mass("li6")


def _case(n, precision="complex128"):
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    rng = np.random.default_rng(11)
    a0 = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    plan = propagator.make_plan(grid, v, M, 1e-6, precision=precision)
    return grid, plan, a0


@pytest.mark.parametrize("n,precision,with_part", [((64, 32, 64), "complex128", True),
                                                   ((32, 16, 512), "complex128", True),
                                                   ((64, 32, 64), "complex128", False),
                                                   ((64, 32, 128), "complex64", True)])
def test_fused_sums_match_standalone(n, precision, with_part):
    grid, plan, a0 = _case(n, precision)
    nat = plan.native
    dt = nat.torch_dtype
    part = observables.symmetric_partition(grid, 1.5e-6)
    xs = _device.to_device_f64(grid.x)
    xb1, xb2 = (_device.to_device_f64(part.xb1), _device.to_device_f64(part.xb2)) if with_part else (None, None)
    ref = torch.from_numpy(a0).to("cuda", dt)
    got = ref.clone()
    nat.advance(ref, 20)
    want = nat.observe(ref, xs, xb1, xb2, 2).cpu().numpy()
    s1 = nat.advance_observe(got, 20, xs, xb1, xb2, 2).cpu().numpy()
    assert torch.equal(got, ref)                  # same wavefunction, bit for bit
    tol = 1e-13 if precision == "complex128" else 1e-6
    assert np.all(np.abs(s1 - want) <= tol * abs(want[0])), (s1, want)
    assert s1[0] > 0 and (not with_part or min(s1[1:4]) > 0)
    # deterministic run to run
    got2 = torch.from_numpy(a0).to("cuda", dt)
    s2 = nat.advance_observe(got2, 20, xs, xb1, xb2, 2).cpu().numpy()
    assert np.array_equal(s1, s2)


def test_evolve_real_uses_fused_sums_and_matches_standalone_trace():
    """A PopulationRecorder trace from evolve_real (fused sums) against the
    same run observed by the standalone reduction after each segment."""
    grid, plan, a0 = _case((64, 32, 64))
    part = observables.symmetric_partition(grid, 1.5e-6)
    rec = observables.PopulationRecorder(part, stride=7)
    edge = observables.EdgeMonitor(stride=5, threshold=1.0)
    psi = qgrid.Wavefunction(a0.copy(), grid)
    psi, _ = propagator.evolve_real(psi, plan, 30, [rec, edge])
    got = rec.trace.as_array()
    # standalone: advance segment by segment and reduce separately
    w = qgrid.Wavefunction(a0.copy(), grid)
    rows, cur = [], 0
    for ev in propagator.event_schedule(30, [rec, edge]):
        if ev > cur:
            plan.native.advance(w.device_amplitudes(), ev - cur)
            w.time += (ev - cur) * plan.dt
            w.invalidate_norm()
            cur = ev
        if ev % 7 == 0 or ev == 30:
            p = observables.populations(w, part)
            rows.append((w.time, *p))
    rows = np.array(rows)
    assert np.array_equal(got[:, 0], rows[:, 0])
    assert np.abs(got[:, 1:4] - rows[:, 1:4]).max() <= 1e-14 * got[:, 4].max()
    assert np.array_equal(psi.amplitudes, w.amplitudes)
