"""Device transverse-minima scan (ctap_slice_minima) and build_partition
against the reference's outputs (tests/golden/minima.npz) and the oracle."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import minima as om
from paper_1309_2451_b200 import magfield, observables, qgrid

pytestmark = pytest.mark.gpu


def _grid(d, tag):
    return qgrid.SimGrid(tuple(int(v) for v in d[f"{tag}_n"]), tuple(float(v) for v in d[f"{tag}_extents"]),
                         tuple(float(v) for v in d[f"{tag}_origin"]))


def _check(got, mx, my, mv, mn):
    assert np.array_equal(np.array([m.x for m in got]), mx, equal_nan=True)
    assert np.array_equal(np.array([m.y for m in got]), my, equal_nan=True)
    assert np.array_equal(np.array([m.value for m in got]), mv, equal_nan=True)
    assert np.array_equal(np.array([m.n_guides for m in got]), mn)


@pytest.mark.parametrize("tag", ["scaled", "paper", "ties", "many"])
def test_slice_minima_match_reference(tag):
    d = load_golden("minima.npz")
    got = magfield.slice_minima(torch.from_numpy(d[f"{tag}_V"]).cuda(), _grid(d, tag))
    _check(got, d[f"{tag}_mx"], d[f"{tag}_my"], d[f"{tag}_mv"], d[f"{tag}_mn"])


@pytest.mark.parametrize("tag", ["scaled", "paper"])
def test_partition_matches_reference(tag):
    d = load_golden("minima.npz")
    g = _grid(d, tag)
    pot = magfield.PotentialGrid(values=torch.from_numpy(d[f"{tag}_V"]).cuda(), grid=g, layout=None)
    part = observables.build_partition(pot, wire_positions=d[f"{tag}_wire_pos"])
    assert np.array_equal(part.xb1, d[f"{tag}_xb1"])
    assert np.array_equal(part.xb2, d[f"{tag}_xb2"])
    assert np.array_equal(part.merged, d[f"{tag}_merged"])


@pytest.mark.parametrize("tag", ["scaled", "paper"])
def test_assemble_potential_minima_from_segments(tag):
    d = load_golden("minima.npz")
    g = _grid(d, tag)
    chip = magfield.ChipSegments.from_arrays(load_golden(f"segments_{tag}.npz"))
    pot = magfield.assemble_potential(chip, g)
    assert np.array_equal(pot.host_values(), d[f"{tag}_V"])
    _check(pot.minima, d[f"{tag}_mx"], d[f"{tag}_my"], d[f"{tag}_mv"], d[f"{tag}_mn"])
    m = pot.minima[int(np.argmax(d[f"{tag}_mn"]))]
    assert pot.guide_minimum(int(np.argmax(d[f"{tag}_mn"])), 0) == (m.x[0], m.y[0], m.value[0])
    lone = np.nonzero(d[f"{tag}_mn"] < 3)[0]
    if lone.size:
        with pytest.raises(magfield.MinimumAbsentError, match="absent"):
            pot.guide_minimum(int(lone[0]), 2)


@pytest.mark.parametrize("shape,seed,kind", [((128, 64, 64), 1, "smooth"), ((256, 32, 32), 2, "smooth"),
                                             ((8, 8, 256), 3, "ties"), ((16, 16, 8), 4, "flat")])
def test_slice_minima_match_oracle_random(shape, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "smooth":  # many minima per slice, unique values
        v = rng.standard_normal(shape)
    elif kind == "ties":  # exact ties everywhere; slices with <= 3 minima (no value sort)
        v = rng.integers(0, 3, size=shape).astype(float)
        for k in range(shape[2]):
            while len(om.minima_indices(v[:, :, k])[0]) > 3:
                v[:, :, k] = rng.integers(0, 3, size=shape[:2])
    else:  # constant slices: no point is strictly below its neighbours
        v = np.ones(shape)
    g = qgrid.make_grid(*shape, (20e-6, 4e-6, 100e-6), origin=(-10e-6, 0.1e-6, 0.0))
    ref = om.all_slice_minima(v, np.asarray(g.x), np.asarray(g.y))
    got = magfield.slice_minima(torch.from_numpy(v).cuda(), g)
    _check(got, np.array([m.x for m in ref]), np.array([m.y for m in ref]),
           np.array([m.value for m in ref]), np.array([m.n_guides for m in ref]))
