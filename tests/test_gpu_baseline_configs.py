"""Driver-run parity at BASELINE.json's own sizes.

* configs 4, 3, 2 and 2b (512^3 and 256^3 paper chip, 128x128x256 scaled chip
  and the population-moving Ioffe trap) against the CPU oracle on identical
  inputs, with a PopulationRecorder: psi rel L2 <= 1e-10, populations <= 1e-9,
  trace time stamps bitwise, device V bitwise equal to the oracle's on the
  sampled points (tests/baseline_cases.py);
* the 512-point z and x transforms of the benched kernels directly against
  numpy;
* config 5 (1024 x 1024 x 512): the 2 x 4 pencil decomposition (virtual
  ranks on one GPU, tests/test_gpu_pencil_virtual.py's exchange emulation)
  bitwise equal to the single-GPU propagation over 4 steps;
* qgrid.gaussian_packet (device normalisation) against the reference's
  vector (/root/reference/pkg/src/ctapsim/qgrid.py:171-196).
Step counts are bounded so the oracle side finishes in ~30 s per case; the
long runs (config 2's 25,000 steps) go through scripts/parity_run.py.
"""

import numpy as np
import pytest
import torch

import baseline_cases as bc
from conftest import load_golden
from oracle import split_step as orc
from paper_1309_2451_b200 import _lib, propagator, qgrid
from paper_1309_2451_b200.constants import muB
from paper_1309_2451_b200.pencil import PencilLayout, pencil_schedule
from paper_1309_2451_b200.propagator import NativePlan

pytestmark = pytest.mark.gpu
M = bc.M


@pytest.mark.parametrize("cfg,steps,stride", [
    ("cfg4", 20, 10),      # 512^3 paper chip: the metric's configuration
    ("cfg3", 200, 50),     # 256^3 paper chip
    ("cfg2b", 1000, 25),   # 128x128x256, populations swing O(1)
    ("cfg2", 1000, 50),    # 128x128x256 scaled chip (full run: scripts/parity_run.py cfg2)
])
def test_baseline_config_parity(cfg, steps, stride):
    case = {"cfg4": lambda: bc.cfg4(every=16), "cfg3": lambda: bc.cfg3(every=8),
            "cfg2": lambda: bc.cfg2(every=4), "cfg2b": bc.cfg2b}[cfg]()
    r = bc.run_case(case, steps, stride)
    print(r)
    assert r["times_equal"] and r["rows_match"]
    assert r["rel_l2"] <= 1e-10, r
    assert r["max_population_diff"] <= 1e-9, r
    assert r["max_norm_diff"] <= 1e-12, r
    if "potential_check" in r:
        assert r["potential_check"]["bitwise_equal"], r["potential_check"]
    if cfg == "cfg2b":   # the case exists because its populations move
        assert r["population_range_p_l"][0] < 0.5 < r["population_range_p_l"][1]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_z_and_x_transforms_at_512_direct_numpy():
    """The 512-point line transforms of the benched passes against numpy:
    [z] forward (zline_kernel), [z^-1 V z] with the oracle's exp_v_full, and
    the warp-per-column ring's [x K x^-1] with the oracle's exp_k."""
    n = (512, 8, 512)
    og = orc.Grid(n, (20e-6, 4e-6, 1000e-6), (-10e-6, 4e-6 / 16, 0.0))
    grid = qgrid.SimGrid(og.n, og.extents, og.origin)
    rng = np.random.default_rng(512)
    a = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x, y, z = og.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * M * ((2 * np.pi * 2e3) ** 2 * x ** 2 + (2 * np.pi * 20.0) ** 2 * (z - 5e-4) ** 2)
    f = orc.make_factors(og, v, M, 1e-6)
    plan = propagator.make_plan(grid, v, M, 1e-6).native

    def rel(got, ref):
        return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))

    d = _dev(a)
    plan.run_pass(_lib.PASS_Z_FWD, d, d)
    assert rel(d.cpu().numpy(), np.fft.fft(a, axis=2)) <= 1e-14
    d = _dev(a)
    plan.run_pass(_lib.PASS_Z_MID, d, d)
    ref = np.fft.fft(f.exp_v_full * (n[2] * np.fft.ifft(a, axis=2)), axis=2)
    assert rel(d.cpu().numpy(), ref) <= 1e-13
    d = _dev(a)
    plan.run_pass(_lib.PASS_X_KIN, d, d)   # ring kernel at nx = 512 (ctap_wline.cu)
    ref = np.fft.ifft(f.exp_k * np.fft.fft(a, axis=0), axis=0) / (n[1] * n[2])
    assert rel(d.cpu().numpy(), ref) <= 1e-13


def test_config5_pencil_2x4_equals_single_gpu():
    """BASELINE config 5 (1024 x 1024 x 512, pencil 2 x 4) self-parity: the 8
    virtual ranks' pencil passes + emulated row/column all-to-alls give
    bitwise the single-GPU psi after 4 steps.  Inputs are built on the device
    (8 GiB psi)."""
    n, Pr, Pc, steps = (1024, 1024, 512), 2, 4, 4
    grid = qgrid.make_grid(*n, (20e-6, 4e-6, 1000e-6), origin=(-10e-6, 4e-6 / n[1] / 2, 0.0))
    ax = [torch.from_numpy(grid.axis(i)).cuda() for i in range(3)]
    om = 2 * np.pi * np.array([2e3, 2e4, 5.0])
    v = (muB / 2 * 0.03 + 0.5 * M * (om[0] ** 2 * ax[0][:, None, None] ** 2
                                     + om[1] ** 2 * (ax[1][None, :, None] - 2e-6) ** 2
                                     + om[2] ** 2 * (ax[2][None, None, :] - 5e-4) ** 2)).contiguous()
    g = torch.Generator(device="cuda").manual_seed(5)
    a0 = torch.complex(torch.randn(n, dtype=torch.float64, device="cuda", generator=g),
                       torch.randn(n, dtype=torch.float64, device="cuda", generator=g))
    # single GPU
    ref = a0.clone()
    one = NativePlan(grid, v, M, 1e-6)
    one.advance(ref, steps)
    torch.cuda.synchronize()
    del one
    # 2 x 4 virtual pencil ranks
    P = Pr * Pc
    lays = [PencilLayout(grid.n, Pr, Pc, r) for r in range(P)]
    plans, bufs = [], []
    for lay in lays:
        plans.append(NativePlan(grid, v[lay.x_slice, lay.y_slice].contiguous(), M, 1e-6, slab_p=P,
                                slab_r=lay.rank, pencil_c=Pc))
        b = {k: torch.empty(lay.points, dtype=torch.complex128, device="cuda") for k in ("zc", "yb", "xp", "xr")}
        b["psi"] = a0[lay.x_slice, lay.y_slice].contiguous().reshape(-1)
        bufs.append(b)
    del a0, v
    for op in pencil_schedule(steps):
        if op[0] == "pass":
            for r in range(P):
                plans[r].run_pass(op[1], bufs[r][op[2]], bufs[r][op[3]])
            continue
        _, which, src, dst = op
        groups = ([PencilLayout(grid.n, Pr, Pc, a * Pc).row_ranks() for a in range(Pr)] if which == "row"
                  else [PencilLayout(grid.n, Pr, Pc, b).col_ranks() for b in range(Pc)])
        for members in groups:
            chunk = lays[0].points // len(members)
            for qi, q in enumerate(members):
                for pi, p in enumerate(members):
                    bufs[q][dst][pi * chunk:(pi + 1) * chunk].copy_(bufs[p][src][qi * chunk:(qi + 1) * chunk])
    for lay, b in zip(lays, bufs):
        assert torch.equal(b["psi"].reshape(lay.block_shape), ref[lay.x_slice, lay.y_slice]), lay.rank


def test_gaussian_packet_device_golden():
    """qgrid.gaussian_packet (host expressions, device normalisation) against
    the vector the reference produced (tests/golden/gaussian_8x8x16.npz)."""
    d = load_golden("gaussian_8x8x16.npz")
    grid = qgrid.SimGrid(tuple(int(v) for v in d["n"]), tuple(d["extents"]), tuple(d["origin"]))
    psi = qgrid.gaussian_packet(grid, (0.1e-6, -0.2e-6, 0.3e-6), (0.6e-6, 0.5e-6, 1.1e-6),
                                momentum=(1e6, -2e6, 3e5))
    got = psi.amplitudes
    assert float(np.abs(got - d["amps"]).max() / np.abs(d["amps"]).max()) <= 1e-15
    assert abs(psi.norm() - 1.0) <= 1e-14
