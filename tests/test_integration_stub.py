"""The reference-side binding documented in INTEGRATION.md is executed here.

The stub is extracted verbatim from INTEGRATION.md's ```python block, so the
document and the tested code cannot drift apart:
  * CPU: its PlanDesc is ctap_plan_desc field for field (names, ctypes types,
    offsets, total size) as _lib.CtapPlanDesc and include/ctap.h declare it;
  * GPU: DevicePlan(plan).advance runs a 32^3 Ioffe-floor trap through
    libctap.so and matches the oracle (rel L2 <= 1e-10), the hook the stub
    proposes for /root/reference/pkg/src/ctapsim/propagator.py:98-107.
"""

import ctypes
import importlib
import os
import re
import sys
import types

import numpy as np
import pytest

from conftest import ROOT
from paper_1309_2451_b200 import _lib


def stub_source() -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    assert len(blocks) == 1, "INTEGRATION.md must hold exactly one python block (the stub)"
    return blocks[0]


def load_stub(tmpdir):
    """Install the stub as `<pkg>._ctap` inside a throwaway package whose
    `qgrid` provides UnitSystem (as ctapsim.qgrid does)."""
    pkg = f"ctapsim_stub_{os.getpid()}"
    d = os.path.join(str(tmpdir), pkg)
    os.makedirs(d, exist_ok=True)
    open(os.path.join(d, "__init__.py"), "w").close()
    with open(os.path.join(d, "qgrid.py"), "w") as fh:
        fh.write("from paper_1309_2451_b200.qgrid import UnitSystem  # noqa: F401\n")
    with open(os.path.join(d, "_ctap.py"), "w") as fh:
        fh.write(stub_source())
    os.environ["CTAP_LIBRARY"] = _lib.LIB_PATH
    sys.path.insert(0, str(tmpdir))
    try:
        return importlib.import_module(f"{pkg}._ctap")
    finally:
        sys.path.remove(str(tmpdir))


def header_desc_fields():
    text = open(os.path.join(ROOT, "include", "ctap.h")).read()
    body = re.search(r"typedef struct ctap_plan_desc \{(.*?)\} ctap_plan_desc;", text, flags=re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    return re.findall(r"(int64_t|int32_t|double)\s+(\w+)", body)


def test_stub_plandesc_matches_abi(tmp_path):
    stub = load_stub(tmp_path)
    ours, theirs = _lib.CtapPlanDesc, stub.PlanDesc
    assert [f[0] for f in theirs._fields_] == [f[0] for f in ours._fields_]
    for (name, t_a), (_, t_b) in zip(theirs._fields_, ours._fields_):
        assert ctypes.sizeof(t_a) == ctypes.sizeof(t_b), name
        assert getattr(theirs, name).offset == getattr(ours, name).offset, name
    assert ctypes.sizeof(theirs) == ctypes.sizeof(ours) == 80
    # and both follow include/ctap.h
    assert [n for _, n in header_desc_fields()] == [f[0] for f in ours._fields_]


def test_stub_defaults_are_the_library_defaults():
    src = stub_source()
    assert "d.phase_tables = 0" in src
    assert "d.dtype, d.pencil_c = 0, 0" in src


@pytest.mark.gpu
def test_stub_device_plan_advance_matches_oracle(tmp_path):
    from oracle import split_step as orc
    from paper_1309_2451_b200 import qgrid
    from paper_1309_2451_b200.constants import hbar, muB, species_mass

    stub = load_stub(tmp_path)
    m = species_mass("li6")
    grid = qgrid.make_grid(32, 32, 32, (20e-6, 4e-6, 250e-6), origin=(-10e-6, 4e-6 / 64, 0.0))
    om = 2 * np.pi * np.array([2e3, 2e4, 20.0])
    x, y, z = grid.meshgrid()
    v = muB / 2 * 0.03 + 0.5 * m * (om[0] ** 2 * x ** 2 + om[1] ** 2 * (y - 2e-6) ** 2
                                    + om[2] ** 2 * (z - 125e-6) ** 2)
    og = orc.as_grid(grid)
    amps0 = orc.gaussian_packet(og, (-4.4e-6, 2e-6, 125e-6), np.sqrt(hbar / (m * om)))
    # what make_plan returns in the reference (propagator.py:37-52), minus the factors
    plan = types.SimpleNamespace(grid=grid, dt=1e-6, mode="real_time", mass=m, potential=v)
    dev = stub.DevicePlan(plan)
    got = dev.advance(amps0.copy(), 40)
    ref = orc.advance(amps0.copy(), orc.make_factors(og, v, m, 1e-6), 40)
    rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    assert rel <= 1e-10, rel
