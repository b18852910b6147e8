"""CPU ORACLE -- test infrastructure only.

Python front end of the C restatement in oracle/bp_oracle.c plus an
independent vectorised numpy restatement of the reference baseline kernel.
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module; the product library never does.

* ``baseline(img, mats, vol, ...)``   -- /root/reference/pkg/src/conebp/_kernels.py:29-61
* ``rung(variant, img_t, mats, vol_t, nb)`` -- _kernels.py:64-369 (transposed rungs)
* ``voxels(img, mats, idx, vals)``    -- baseline on a global-index voxel list
* ``numpy_baseline(img, mats, vol)``  -- vectorised restatement, same float32 op order
  (the reference's own test oracle idea, pkg/tests/helpers.py:61-87)

Parity status: pinned.  tests/test_oracle_golden.py checks both restatements
bit for bit against golden vectors written by tests/golden/make_golden.py from
the live reference package.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_float, c_int, c_int64
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_f32p = POINTER(c_float)
_i64p = POINTER(c_int64)
_lib = None


def build(force: bool = False) -> Path:
    src = HERE / "bp_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "-B" if force else "liboracle.so"], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        lib.oracle_baseline.restype = c_int64
        lib.oracle_baseline.argtypes = [_f32p, c_int64, c_int64, c_int64, c_int64, c_int64, _f32p, _f32p, c_int64,
                                        c_int64, c_int64, c_int64, c_int]
        lib.oracle_rung.restype = c_int
        lib.oracle_rung.argtypes = [c_int, _f32p, c_int64, c_int64, c_int64, _f32p, _f32p, c_int64, c_int64, c_int64,
                                    c_int64, c_int]
        lib.oracle_voxels.restype = None
        lib.oracle_voxels.argtypes = [_f32p, c_int64, c_int64, c_int64, _f32p, _i64p, c_int64, _f32p, c_int]
        _lib = lib
    return _lib


def _f(a):
    return a.ctypes.data_as(_f32p)


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))


def baseline(img: np.ndarray, mats: np.ndarray, vol: np.ndarray, threads: int | None = None, *, nh: int | None = None,
             v0: int = 0, k_lo: int = 0) -> int:
    """Accumulate the reference baseline into ``vol`` in place.

    img: [np][rows][nw] float32 holding detector rows [v0, v0+rows) of an nh-row
    detector (default: the full detector); vol: [nz_slab][ny][nx] holding global
    slices [k_lo, k_lo+nz_slab).  Returns the number of samples that needed a row
    outside the band (0 for a full detector).
    """
    img = np.ascontiguousarray(img, dtype=np.float32)
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    assert vol.dtype == np.float32 and vol.flags.c_contiguous
    n_proj, rows, nw = img.shape
    nzs, ny, nx = vol.shape
    nh = rows if nh is None else nh
    return int(_load().oracle_baseline(_f(img), n_proj, nh, nw, v0, rows, _f(mats), _f(vol), nx, ny, k_lo,
                                       k_lo + nzs, threads or default_threads()))


def rung(variant: int, img_t: np.ndarray, mats: np.ndarray, vol_t: np.ndarray, nb: int,
         threads: int | None = None) -> None:
    """Optimized rung ``variant`` (1..5) on TRANSPOSED layouts, in place."""
    img_t = np.ascontiguousarray(img_t, dtype=np.float32)
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    assert vol_t.dtype == np.float32 and vol_t.flags.c_contiguous
    n_proj, nw, nh = img_t.shape
    nx, ny, nz = vol_t.shape
    rc = _load().oracle_rung(int(variant), _f(img_t), n_proj, nh, nw, _f(mats), _f(vol_t), nx, ny, nz, nb,
                             threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_rung: invalid variant / nb / nz")


def voxels(img: np.ndarray, mats: np.ndarray, idx: np.ndarray, vals: np.ndarray | None = None,
           threads: int | None = None) -> np.ndarray:
    """Baseline value of each voxel idx[q] = (i, j, k) (global indices), added to vals."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 3)
    out = np.zeros(len(idx), np.float32) if vals is None else np.ascontiguousarray(vals, dtype=np.float32).copy()
    n_proj, nh, nw = img.shape
    _load().oracle_voxels(_f(img), n_proj, nh, nw, _f(mats), idx.ctypes.data_as(_i64p), len(idx), _f(out),
                          threads or default_threads())
    return out


def numpy_baseline(img: np.ndarray, mats: np.ndarray, vol: np.ndarray) -> np.ndarray:
    """Vectorised restatement of _kernels.baseline (float32, reference op order)."""
    n_proj, nh, nw = img.shape
    nz, ny, nx = vol.shape
    one = np.float32(1.0)
    fi = np.arange(nx, dtype=np.float32)[None, None, :]
    fj = np.arange(ny, dtype=np.float32)[None, :, None]
    fk = np.arange(nz, dtype=np.float32)[:, None, None]
    umax, vmax = np.float32(nw - 1), np.float32(nh - 1)
    for s in range(n_proj):
        m = mats[s].astype(np.float32)
        z = ((m[2, 0] * fi + m[2, 1] * fj) + m[2, 2] * fk) + m[2, 3]
        f = one / z
        x = (((m[0, 0] * fi + m[0, 1] * fj) + m[0, 2] * fk) + m[0, 3]) * f
        y = (((m[1, 0] * fi + m[1, 1] * fj) + m[1, 2] * fk) + m[1, 3]) * f
        take = (x >= 0) & (x < umax) & (y >= 0) & (y < vmax)
        ix = np.where(take, x, 0).astype(np.int64)
        iy = np.where(take, y, 0).astype(np.int64)
        ax = x - ix.astype(np.float32)
        ay = y - iy.astype(np.float32)
        p = img[s]
        s0 = p[iy, ix] * (one - ax) + p[iy, ix + 1] * ax
        s1 = p[iy + 1, ix] * (one - ax) + p[iy + 1, ix + 1] * ax
        upd = (s0 * (one - ay) + s1 * ay) * (f * f)
        vol[take] = vol[take] + upd[take]  # immediate += only where sampled (_kernels.py:52,61)
    return vol
