"""The CPU restatement of the transverse-minima scan and build_partition
(oracle/minima.py) against the reference's own outputs (tests/golden/minima.npz,
made by tests/golden/make_golden.py from ctapsim.magfield / observables)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import minima as om
from oracle import split_step as orc


def _grid(d, tag):
    return orc.Grid(tuple(int(v) for v in d[f"{tag}_n"]), tuple(float(v) for v in d[f"{tag}_extents"]),
                    tuple(float(v) for v in d[f"{tag}_origin"]))


@pytest.mark.parametrize("tag", ["scaled", "paper", "ties", "many"])
def test_slice_minima_bitwise(tag):
    d = load_golden("minima.npz")
    g = _grid(d, tag)
    got = om.all_slice_minima(d[f"{tag}_V"], g.axis(0), g.axis(1))
    assert np.array_equal(np.array([m.x for m in got]), d[f"{tag}_mx"], equal_nan=True)
    assert np.array_equal(np.array([m.y for m in got]), d[f"{tag}_my"], equal_nan=True)
    assert np.array_equal(np.array([m.value for m in got]), d[f"{tag}_mv"], equal_nan=True)
    assert np.array_equal(np.array([m.n_guides for m in got]), d[f"{tag}_mn"])


@pytest.mark.parametrize("tag", ["scaled", "paper"])
def test_partition_bitwise(tag):
    d = load_golden("minima.npz")
    g = _grid(d, tag)
    v = d[f"{tag}_V"]
    mins = om.all_slice_minima(v, g.axis(0), g.axis(1))
    xb1, xb2, merged = om.build_partition(v, mins, g.axis(0), d[f"{tag}_wire_pos"])
    assert np.array_equal(xb1, d[f"{tag}_xb1"])
    assert np.array_equal(xb2, d[f"{tag}_xb2"])
    assert np.array_equal(merged, d[f"{tag}_merged"])
