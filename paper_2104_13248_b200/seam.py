"""The reference package's kernel seam, served by libconebp_b200.

``conebp`` has no plugin registry: its entry points call the numba kernels in
``conebp._kernels`` directly (``backprojector.py:159`` for BASELINE, the
dispatch dict at ``:199-206`` for the optimized rungs).  ``install(conebp)``
replaces those six module attributes with functions that take exactly the
numba kernels' arguments -- ``baseline(img, mats, vol)`` and
``<rung>(img_t, mats, vol_t, ij, nb)`` on C-contiguous float32 numpy arrays --
and accumulate into ``vol`` in place through ``cbp_backproject_host_f32``.
Nothing else in the reference changes: its validation, containers, counters
and tests run unmodified on top.  ``ij`` and ``nb`` are not needed on the GPU:
every voxel accumulates all angles in ascending order, which the reference's
batch seeding makes bitwise identical for every nb (_kernels.py:3-10).

Used by tools/run_reference_tests.py to run the reference's own test suite on
the GPU path (the drop-in proof), and by anyone adopting the GPU kernels while
keeping ``conebp`` itself.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["install", "uninstall", "calls"]

_RUNGS = {"baseline": 0, "transpose": 1, "share": 2, "symmetry": 3, "subline": 4, "subline_prefetch": 5}
calls = {name: 0 for name in _RUNGS}
_saved: dict = {}


def _run(img: np.ndarray, mats: np.ndarray, vol: np.ndarray, variant: int, natural: bool) -> None:
    for a in (img, mats, vol):
        if a.dtype != np.float32 or not a.flags.c_contiguous:
            raise TypeError("the kernel seam takes C-contiguous float32 arrays")
    if natural:
        n_proj, nh, nw = img.shape
        nz, ny, nx = vol.shape
    else:
        n_proj, nw, nh = img.shape
        nx, ny, nz = vol.shape
    lay = _lib.NATURAL if natural else _lib.TRANSPOSED
    _lib.check(_lib.lib().cbp_backproject_host_f32(_lib.f32ptr(img), n_proj, nh, nw, lay, _lib.f32ptr(mats),
                                                   _lib.f32ptr(vol), nx, ny, nz, lay, variant, 0))


def _make(name: str, variant: int):
    if variant == 0:
        def baseline(img, mats, vol):  # _kernels.py:29-61
            calls[name] += 1
            _run(img, mats, vol, 0, True)
        return baseline

    def rung(img, mats, vol, ij, nb):  # _kernels.py:64-369
        calls[name] += 1
        _run(img, mats, vol, variant, False)
    rung.__name__ = name
    return rung


def install(conebp) -> None:
    """Point ``conebp._kernels.<variant>`` at the GPU library (idempotent)."""
    k = conebp._kernels
    for name, variant in _RUNGS.items():
        if name not in _saved:
            _saved[name] = getattr(k, name)
        setattr(k, name, _make(name, variant))


def uninstall(conebp) -> None:
    k = conebp._kernels
    for name, fn in _saved.items():
        setattr(k, name, fn)
    _saved.clear()
