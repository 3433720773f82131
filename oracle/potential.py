"""ctypes wrapper of oracle/potential.c (TEST ORACLE ONLY).

Restates magfield._potential_kernel (magfield.py:107-144) and the segment
assembly of assemble_potential (magfield.py:229-238); built by oracle/Makefile.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle_potential.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        lib = ctypes.CDLL(_LIB)
        d, i64, p = ctypes.c_double, ctypes.c_int64, ctypes.c_void_p
        lib.oracle_potential.argtypes = [p, i64, p, i64, p, i64, p, p, p, i64,
                                         d, d, d, d, d, d, d, d, p, ctypes.c_int]
        lib.oracle_potential.restype = None
        _lib = lib
    return _lib


def potential(xs, ys, zs, seg_a, seg_b, seg_cur, b0, mu_eff, mass, omega_z, z_center,
              pref, threads: int | None = None) -> np.ndarray:
    """V on the grid (nx, ny, nz), float64, bit-identical to the numba kernel."""
    lib = _load()
    xs, ys, zs = (np.ascontiguousarray(a, dtype=np.float64) for a in (xs, ys, zs))
    seg_a = np.ascontiguousarray(seg_a, dtype=np.float64)
    seg_b = np.ascontiguousarray(seg_b, dtype=np.float64)
    seg_cur = np.ascontiguousarray(seg_cur, dtype=np.float64)
    out = np.empty((xs.size, ys.size, zs.size))
    lib.oracle_potential(xs.ctypes.data, xs.size, ys.ctypes.data, ys.size, zs.ctypes.data, zs.size,
                         seg_a.ctypes.data, seg_b.ctypes.data, seg_cur.ctypes.data, seg_cur.size,
                         float(b0[0]), float(b0[1]), float(b0[2]), float(mu_eff), float(mass),
                         float(omega_z), float(z_center), float(pref), out.ctypes.data,
                         int(threads or os.cpu_count() or 1))
    return out


def potential_from_chip(chip: dict, xs, ys, zs, threads=None) -> np.ndarray:
    """V from a chip fixture dict (keys of tests/golden/segments_*.npz)."""
    return potential(xs, ys, zs, chip["seg_a"], chip["seg_b"], chip["seg_cur"], chip["b0"],
                     float(chip["mu_eff"]), float(chip["mass"]), float(chip["omega_z"]),
                     float(chip["z_center"]), float(chip["pref"]), threads)
