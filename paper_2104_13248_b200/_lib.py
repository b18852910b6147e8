"""ctypes binding of libconebp_b200.so (include/conebp_b200.h).

The library is the only compute path: there is no CPU fallback.  Importing
this module does not touch the GPU; ``lib()`` loads the shared object and
raises ``RuntimeError`` if it is missing (build it with
``python -m paper_2104_13248_b200.build``).
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_char_p, c_float, c_int, c_int64, c_uint, c_void_p
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("CBP_LIB_PATH", str(Path(__file__).resolve().parent / "libconebp_b200.so")))

CBP_OK = 0
CBP_EINVAL = -1
CBP_ECUDA = -2
CBP_ENOMEM = -3
CBP_EBAND = -4
CBP_ENODEV = -5

NATURAL = 0
TRANSPOSED = 1

FLAG_NAIVE = 1
FLAG_NO_SMEM = 2
FLAG_FMA_LERP = 4
FLAG_CHECK = 8

_f32p = POINTER(c_float)
_i64p = POINTER(c_int64)

# name -> (restype, argtypes); every symbol declared in include/conebp_b200.h
SIGNATURES = {
    "cbp_version": (c_int, []),
    "cbp_last_error": (c_char_p, []),
    "cbp_device_count": (c_int, []),
    "cbp_staged_pitch": (c_int64, [c_int64]),
    "cbp_stage_projections": (
        c_int,
        [c_void_p, c_int, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p],
    ),
    "cbp_backproject_f32": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int, _f32p, c_void_p, c_int64, c_int64, c_int64, c_int, c_int,
         c_uint, c_void_p],
    ),
    "cbp_backproject_staged": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, _f32p, c_void_p, c_int, c_int64, c_int64,
         c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_uint, c_void_p],
    ),
    "cbp_backproject_host_f32": (
        c_int,
        [_f32p, c_int64, c_int64, c_int64, c_int, _f32p, _f32p, c_int64, c_int64, c_int64, c_int, c_int, c_uint],
    ),
    "cbp_sync_status": (c_int, [c_void_p, _i64p]),
    "cbp_count_ops": (
        c_int,
        [_f32p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int64, _i64p, c_void_p],
    ),
    "cbp_slab_plan": (
        c_int,
        [_f32p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int64, c_int64, _i64p, _i64p],
    ),
    "cbp_slab_band": (
        c_int,
        [_f32p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int64, c_int64, _i64p, _i64p],
    ),
    "cbp_forward_project_f32": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, ctypes.c_double, POINTER(ctypes.c_double), c_int64, c_int64, c_int64,
         ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, c_void_p, c_void_p],
    ),
    "cbp_fdk_filter_f32": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
         ctypes.c_double, ctypes.c_double, c_void_p, c_int64, c_void_p],
    ),
    "cbp_backproject_window": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, _f32p, c_void_p, c_int,
         c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_uint, c_void_p],
    ),
    "cbp_backproject_multi": (
        c_int,
        [c_void_p, c_int64, c_int64, c_int64, _f32p, POINTER(c_void_p), c_int64, c_int64, c_int64, _i64p, c_int,
         POINTER(c_int), c_int, c_uint, c_int64, _i64p],
    ),
    "cbp_copy_band": (
        c_int,
        [c_void_p, c_int, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p],
    ),
    "cbp_ipc_export": (c_int, [c_void_p, c_void_p, _i64p]),
    "cbp_ipc_open": (c_int, [c_void_p, c_int64, POINTER(c_void_p)]),
    "cbp_ipc_close": (c_int, [c_void_p, c_int64]),
    "cbp_selftest_rcp": (c_int, [ctypes.c_uint32, ctypes.c_uint32, POINTER(ctypes.c_uint64), POINTER(ctypes.c_uint32)]),
    "cbp_release": (c_int, []),
    "cbp_last_plan": (c_int, [_i64p]),
}

_lib = None


class CbpError(RuntimeError):
    """A libconebp_b200 call failed (the message is cbp_last_error())."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"libconebp_b200 error {code}: {msg}")
        self.code = code


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: the CUDA back-projection library must be built "
                "(python -m paper_2104_13248_b200.build); there is no CPU fallback"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(code: int) -> None:
    if code != CBP_OK:
        msg = lib().cbp_last_error().decode(errors="replace")
        if code == CBP_EINVAL:
            raise ValueError(msg)
        raise CbpError(code, msg)


def f32ptr(arr):
    """ctypes float* of a C-contiguous float32 numpy array."""
    return arr.ctypes.data_as(_f32p)


def i64ptr(arr):
    return arr.ctypes.data_as(_i64p)
