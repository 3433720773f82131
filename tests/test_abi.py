"""C ABI: libctap.so loads without a GPU and exports every declared symbol;
argument validation happens before any CUDA call."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1309_2451_b200 import _lib


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ctap.h")).read()
    return sorted(set(re.findall(r"CTAP_API\s+[\w\s\*]+?\b(ctap_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.ctap_version()


def test_nm_exports_only_the_abi():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert exported == declared_symbols()


def _desc(n=(16, 16, 16), mode=0, p=1, r=0, pc=0):
    d = _lib.CtapPlanDesc()
    for i in range(3):
        d.n[i] = n[i]
    d.e0, d.dt_i, d.len2, d.v_shift = 1.0, 1.0, 1e-12, 0.0
    d.mode, d.slab_p, d.slab_r, d.pencil_c = mode, p, r, pc
    return d


@pytest.mark.parametrize("kw,code,msg", [
    (dict(n=(12, 16, 16)), _lib.CTAP_EUNSUPPORTED, "powers of two"),
    (dict(n=(2048, 16, 16)), _lib.CTAP_EUNSUPPORTED, "powers of two"),
    (dict(mode=7), _lib.CTAP_EINVAL, "unknown mode"),
    (dict(p=3), _lib.CTAP_EINVAL, "divisible"),
    (dict(p=2, r=2), _lib.CTAP_EINVAL, "out of range"),
    (dict(p=6, pc=4), _lib.CTAP_EINVAL, "do not form a pencil grid"),
    (dict(p=8, pc=4, n=(16, 16, 16)), _lib.CTAP_EINVAL, "pencil grid 2 x 4"),   # nz < 8 Pc
    (dict(p=4, pc=2, r=4, n=(16, 16, 16)), _lib.CTAP_EINVAL, "out of range"),
])
def test_plan_create_validation(kw, code, msg):
    import numpy as np

    lib = _lib.load()
    k2 = np.zeros(2048)
    h = ctypes.c_void_p()
    st = lib.ctap_plan_create(ctypes.byref(_desc(**kw)), k2.ctypes.data, k2.ctypes.data,
                              k2.ctypes.data, 8, ctypes.byref(h))
    assert st == code
    assert msg in lib.ctap_last_error().decode()
    with pytest.raises((ValueError, NotImplementedError), match=msg):
        _lib.check(st)


def test_null_arguments_rejected():
    lib = _lib.load()
    assert lib.ctap_advance(None, None, 1, None) == _lib.CTAP_EINVAL
    assert lib.ctap_advance_observe(None, None, 1, None, None, None, 2, None, None) == _lib.CTAP_EINVAL
    assert lib.ctap_set_peer_buffers(None, 0, None, 0) == _lib.CTAP_EINVAL
    assert lib.ctap_observe(None, None, None, None, None, 2, None, None) == _lib.CTAP_EINVAL
    assert lib.ctap_potential(None, 1, None, 1, None, 1, None, None, None, 0,
                              0., 0., 0., 0., 0., 0., 0., 0., None, None) == _lib.CTAP_EINVAL
    assert lib.ctap_step_schedule(None, None, None) == _lib.CTAP_EINVAL
