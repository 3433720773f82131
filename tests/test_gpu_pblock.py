"""The x-slab position-block schedule of ctap_advance (the passes between
two x passes, [y^-1, z^-1 V z, y], run slab by slab on three streams so a
slab stays in L2) is bitwise equal to the plane-order schedule: psi and every
trace row of an observed evolve_real, eager steps, graph-captured steps and
the fused observer segment end included.  The schedule is chosen from
CTAP_PBLOCK when the plan is made, so each variant runs in its own process."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(env_extra, precision="complex128", n=256, steps=45, stride=20):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(HERE, "schedule_digest.py"), str(n), str(steps), str(stride),
                          precision],
                         env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
@pytest.mark.parametrize("precision", ["complex128", "complex64"])
def test_position_block_schedule_bitwise_equal(precision):
    ref = _digest({"CTAP_PBLOCK": "0"}, precision)
    assert len(ref["rows"]) == 4  # t = 0, 20, 40 and the final step; 20-step segments use the step graphs
    variants = (("16", "3"), ("8", "1"), ("32", "2")) if precision == "complex128" else (("16", "3"),)
    for planes, streams in variants:
        got = _digest({"CTAP_PBLOCK": planes, "CTAP_PBLOCK_STREAMS": streams}, precision)
        assert got == ref, (planes, streams)
    if precision == "complex128":
        # with the exp(-iV dt) plan table (offset per slab like v_i); the table
        # holds the on-the-fly recipe's factors, so psi is the same bit for bit
        got = _digest({"CTAP_PBLOCK": "16", "CTAP_PHASE_TABLES": "1"}, precision)
        assert got == ref


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_schedule_choice_and_launch_count():
    """ctap_step_schedule reports the automatic choice: x-slabs for a
    complex128 grid whose psi + v_i exceed the L2 (4 planes at 512^3 on
    three streams, 16 at 256^3), plane order for complex64 and small grids."""
    import numpy as np

    from paper_1309_2451_b200 import propagator, qgrid

    if os.environ.get("CTAP_PBLOCK"):
        pytest.skip("CTAP_PBLOCK overrides the automatic choice")
    for n, precision, want in ((256, "complex128", (16, 3)), (256, "complex64", (0, 1)), (64, "complex128", (0, 1))):
        grid = qgrid.make_grid(n, n, n, (20e-6, 4e-6, 1000e-6))
        plan = propagator.make_plan(grid, np.zeros(grid.n), 1.0e-26, 1e-6, precision=precision)
        assert plan.native.step_schedule() == want, (n, precision)
        planes = want[0]
        assert plan.native.launches(20) == (4 * 20 + 1 if planes == 0 else
                                            2 * (n // planes) + 19 * (1 + 3 * (n // planes)) + 1 + 2 * (n // planes))
