"""ctypes binding of libctap.so (include/ctap.h).

The library is built in-tree by __graft_entry__.build() (nvcc, sm_100a).
There is no fallback: if the library is missing or no CUDA device is present,
every propagation call raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CTAP_LIBRARY overrides the in-tree build (used for A/B kernel experiments)
LIB_PATH = os.environ.get("CTAP_LIBRARY") or os.path.join(_HERE, "lib", "libctap.so")

CTAP_OK = 0
CTAP_EINVAL = 1
CTAP_ECUDA = 2
CTAP_EUNSUPPORTED = 3

REAL_TIME_MODE = 0
IMAGINARY_TIME_MODE = 1

DTYPE_C128 = 0
DTYPE_C64 = 1

# ctap_pass_kind
PASS_Z_FWD, PASS_Z_INV, PASS_Z_FIRST, PASS_Z_MID, PASS_Z_LAST = range(5)
PASS_Y_FWD, PASS_Y_INV, PASS_Y_FWD_TO_PEER, PASS_Y_INV_FROM_PEER = range(5, 9)
PASS_X_KIN, PASS_X_FWD, PASS_X_INV = range(9, 12)
PASS_Y_FWD_BLK, PASS_X_KIN_BLK, PASS_Y_INV_BLK = range(12, 15)
PASS_Y_FWD_TO_PEERS, PASS_X_KIN_TO_PEERS = 15, 16
PASS_PZ_FIRST, PASS_PZ_MID, PASS_PZ_LAST, PASS_PY_FWD, PASS_PY_INV, PASS_PX_KIN = range(17, 23)

# every symbol include/ctap.h declares
EXPORTS = (
    "ctap_plan_create", "ctap_plan_destroy", "ctap_advance", "ctap_advance_observe", "ctap_pass", "ctap_pass_zchunk", "ctap_observe",
    "ctap_density_xz", "ctap_k2_sums", "ctap_v_sums", "ctap_v_sums_with", "ctap_phase_field", "ctap_scale",
    "ctap_fft3d", "ctap_potential", "ctap_last_error", "ctap_version",
    "ctap_set_peer_buffers", "ctap_ipc_handle", "ctap_ipc_open", "ctap_ipc_close",
    "ctap_device_alloc", "ctap_device_free", "ctap_slice_minima", "ctap_flag_barrier", "ctap_step_schedule",
)


class CtapPlanDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64 * 3),
        ("e0", ctypes.c_double),
        ("dt_i", ctypes.c_double),
        ("len2", ctypes.c_double),
        ("v_shift", ctypes.c_double),
        ("mode", ctypes.c_int32),
        ("slab_p", ctypes.c_int32),
        ("slab_r", ctypes.c_int32),
        ("phase_tables", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("pencil_c", ctypes.c_int32),
    ]


class CtapError(RuntimeError):
    """A CUDA-side failure inside libctap."""


_lib = None


def load():
    """Load libctap.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(LIB_PATH)
    p, i32, i64, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "ctap_plan_create": [ctypes.POINTER(CtapPlanDesc), p, p, p, p, ctypes.POINTER(p)],
        "ctap_plan_destroy": [p],
        "ctap_advance": [p, p, i64, p],
        "ctap_advance_observe": [p, p, i64, p, p, p, i32, p, p],
        "ctap_pass": [p, i32, p, p, p],
        "ctap_pass_zchunk": [p, i32, p, p, i64, i64, p],
        "ctap_observe": [p, p, p, p, p, i32, p, p],
        "ctap_density_xz": [p, p, p, p],
        "ctap_k2_sums": [p, p, p, p],
        "ctap_v_sums": [p, p, p, p],
        "ctap_v_sums_with": [p, p, p, p, p],
        "ctap_phase_field": [p, i32, p, p],
        "ctap_scale": [p, p, d, p],
        "ctap_fft3d": [p, p, i32, p],
        "ctap_potential": [p, i64, p, i64, p, i64, p, p, p, i64, d, d, d, d, d, d, d, d, p, p],
        "ctap_set_peer_buffers": [p, i32, ctypes.POINTER(p), i32],
        "ctap_ipc_handle": [p, p],
        "ctap_ipc_open": [p, ctypes.POINTER(p)],
        "ctap_ipc_close": [p],
        "ctap_device_alloc": [i64, ctypes.POINTER(p)],
        "ctap_device_free": [p],
        "ctap_slice_minima": [p, i64, i64, i64, p, p, p],
        "ctap_flag_barrier": [ctypes.POINTER(p), p, i32, i32, ctypes.c_uint32, p],
        "ctap_step_schedule": [p, ctypes.POINTER(i64), ctypes.POINTER(i32)],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.ctap_last_error.argtypes = []
    lib.ctap_last_error.restype = ctypes.c_char_p
    lib.ctap_version.argtypes = []
    lib.ctap_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def check(status: int):
    """Map a ctap_status to the reference's exception types."""
    if status == CTAP_OK:
        return
    msg = load().ctap_last_error().decode(errors="replace")
    if status == CTAP_EINVAL:
        raise ValueError(msg)
    if status == CTAP_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise CtapError(msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args))
