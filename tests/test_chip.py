"""The product-side chip geometry (paper_1309_2451_b200/chip.py) reproduces
the segment arrays the reference itself produced (tests/golden/segments_*.npz,
made by tests/golden/make_golden.py from ctapsim's config + chipgeom +
magfield.layout_segments) bit for bit -- the bench's potential input does not
depend on a test fixture or on the reference being importable."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1309_2451_b200 import chip


@pytest.mark.parametrize("name", ["paper", "scaled"])
def test_chip_segments_bitwise_reference(name):
    got = chip.chip_segments(name)
    ref = load_golden(f"segments_{name}.npz")
    for k in ("seg_a", "seg_b", "seg_cur", "b0"):
        assert np.array_equal(getattr(got, k), ref[k]), k
    for k in ("mu_eff", "mass", "omega_z", "z_max", "x_span"):
        assert getattr(got, k) == float(ref[k]), k


def test_chip_segments_validation():
    with pytest.raises(ValueError, match="unknown chip"):
        chip.chip_segments("desk")
    with pytest.raises(ValueError, match="unknown ordering"):
        chip.chip_segments("paper", ordering="sideways")
    a = chip.chip_segments("paper", ordering="intuitive")
    b = chip.chip_segments("paper")
    assert a.seg_a.shape == b.seg_a.shape and not np.array_equal(a.seg_a, b.seg_a)
