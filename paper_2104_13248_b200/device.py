"""Device-resident entry points (torch CUDA tensors in, stream-ordered).

PyTorch is only the hand-off layer here: it owns device memory and streams;
every value is computed by libconebp_b200.so.  These calls are what the
multi-GPU slab driver and the benchmark's device-timed leg use; the numpy
drop-in API lives in :mod:`paper_2104_13248_b200.backprojector`.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .backprojector import KernelVariant
from .tensors import Layout

__all__ = ["StagedProjections", "backproject_device", "backproject_staged", "backproject_window", "backproject_multi",
           "copy_band", "ipc_export", "ipc_open", "ipc_close", "selftest_rcp", "sync_status", "last_plan",
           "stream_handle"]


def _torch():
    import torch

    return torch


def stream_handle(stream=None) -> int:
    torch = _torch()
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _check_tensor(t, shape, what):
    torch = _torch()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
        raise ValueError(f"{what} must be a contiguous float32 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what}: expected shape {tuple(shape)}, got {tuple(t.shape)}")


class StagedProjections:
    """Projections in the device staging layout staged[s][r][u] (u pitch % 4 == 0).

    Holds detector rows [v0, v0+rows) of an (np, nh, nw) stack (the whole
    detector by default).  Built by cbp_stage_projections, the replacement of
    tensors.transpose_projections (tensors.py:138-147) for TRANSPOSED inputs.
    """

    def __init__(self, img_dev, n_proj: int, nh: int, nw: int, layout: Layout = Layout.NATURAL, v0: int = 0,
                 rows: int | None = None, stream=None):
        torch = _torch()
        layout = Layout(layout)
        shape = (n_proj, nh, nw) if layout is Layout.NATURAL else (n_proj, nw, nh)
        _check_tensor(img_dev, shape, "projections")
        rows = nh - v0 if rows is None else rows
        self.np, self.nh, self.nw, self.v0, self.rows = n_proj, nh, nw, v0, rows
        self.pitch = int(_lib.lib().cbp_staged_pitch(nw))
        self.data = torch.empty((n_proj, rows, self.pitch), dtype=torch.float32, device=img_dev.device)
        _lib.check(_lib.lib().cbp_stage_projections(img_dev.data_ptr(), 0 if layout is Layout.NATURAL else 1, n_proj,
                                                    nh, nw, v0, rows, self.data.data_ptr(), self.pitch,
                                                    stream_handle(stream)))

    @classmethod
    def wrap(cls, staged_dev, n_proj: int, nh: int, nw: int, v0: int, rows: int) -> "StagedProjections":
        """Adopt an existing staging buffer (e.g. a band received over NCCL)."""
        obj = cls.__new__(cls)
        obj.np, obj.nh, obj.nw, obj.v0, obj.rows = n_proj, nh, nw, v0, rows
        obj.pitch = int(staged_dev.shape[2])
        _check_tensor(staged_dev, (n_proj, rows, obj.pitch), "staged projections")
        obj.data = staged_dev
        return obj


def _vol_shape(nx, ny, nz, layout: Layout):
    return (nz, ny, nx) if layout is Layout.NATURAL else (nx, ny, nz)


def backproject_staged(staged: StagedProjections, mats: np.ndarray, vol_dev, nx: int, ny: int, nz: int,
                       variant: KernelVariant = KernelVariant.BASELINE, vol_layout: Layout = Layout.NATURAL,
                       k0: int = 0, nz_total: int | None = None, s_begin: int = 0, s_end: int | None = None,
                       flags: int = 0, stream=None) -> None:
    """Accumulate slab [k0, k0+nz) of a volume with nz_total slices (stream-ordered)."""
    vol_layout = Layout(vol_layout)
    _check_tensor(vol_dev, _vol_shape(nx, ny, nz, vol_layout), "volume")
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    if mats.shape != (staged.np, 3, 4):
        raise ValueError(f"expected ({staged.np}, 3, 4) matrices, got {mats.shape}")
    nz_total = nz if nz_total is None else nz_total
    s_end = staged.np if s_end is None else s_end
    _lib.check(_lib.lib().cbp_backproject_staged(
        staged.data.data_ptr(), staged.pitch, staged.np, staged.nh, staged.nw, staged.v0, staged.rows,
        _lib.f32ptr(mats), vol_dev.data_ptr(), 0 if vol_layout is Layout.NATURAL else 1, nx, ny, nz, k0, nz_total,
        s_begin, s_end, int(KernelVariant(variant)), flags, stream_handle(stream)))


def backproject_window(band_dev, s_base: int, mats: np.ndarray, vol_dev, n_proj: int, nh: int, nw: int, v0: int,
                       rows: int, nx: int, ny: int, nz: int, variant: KernelVariant = KernelVariant.BASELINE,
                       k0: int = 0, nz_total: int | None = None, s_begin: int | None = None,
                       s_end: int | None = None, vol_layout: Layout = Layout.NATURAL, flags: int = 0,
                       stream=None) -> None:
    """Accumulate angles [s_begin, s_end) from a band buffer holding only angles
    [s_base, s_base + band_dev.shape[0]) (layout [n][rows][pitch]) into slab [k0, k0+nz)."""
    vol_layout = Layout(vol_layout)
    torch = _torch()
    if not (isinstance(band_dev, torch.Tensor) and band_dev.is_cuda and band_dev.dtype == torch.float32
            and band_dev.is_contiguous() and band_dev.dim() == 3 and band_dev.shape[1] == rows):
        raise ValueError("band must be a contiguous float32 CUDA tensor [n][rows][pitch]")
    _check_tensor(vol_dev, _vol_shape(nx, ny, nz, vol_layout), "volume")
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    if mats.shape != (n_proj, 3, 4):
        raise ValueError(f"expected ({n_proj}, 3, 4) matrices, got {mats.shape}")
    n = int(band_dev.shape[0])
    s_begin = s_base if s_begin is None else s_begin
    s_end = s_base + n if s_end is None else s_end
    nz_total = nz if nz_total is None else nz_total
    _lib.check(_lib.lib().cbp_backproject_window(
        band_dev.data_ptr(), int(band_dev.shape[2]), n_proj, nh, nw, v0, rows, s_base, n, _lib.f32ptr(mats),
        vol_dev.data_ptr(), 0 if vol_layout is Layout.NATURAL else 1, nx, ny, nz, k0, nz_total, s_begin, s_end,
        int(KernelVariant(variant)), flags, stream_handle(stream)))


def copy_band(src_ptr: int, n_proj: int, nh: int, nw: int, s0: int, s1: int, v0: int, rows: int, dst_dev,
              src_device: int = -1, stream=None) -> None:
    """Copy-engine transfer of angles [s0, s1) x rows [v0, v0+rows) of a NATURAL stack at
    device address ``src_ptr`` (local or IPC-mapped) into ``dst_dev`` [s1-s0][rows][pitch]."""
    _lib.check(_lib.lib().cbp_copy_band(src_ptr, src_device, n_proj, nh, nw, s0, s1, v0, rows, dst_dev.data_ptr(),
                                        int(dst_dev.shape[2]), stream_handle(stream)))


def ipc_export(t) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t in it)."""
    import ctypes

    h = ctypes.create_string_buffer(64)
    off = np.zeros(1, np.int64)
    _lib.check(_lib.lib().cbp_ipc_export(t.data_ptr(), h, _lib.i64ptr(off)))
    return bytes(h.raw), int(off[0])


def ipc_open(handle: bytes, offset: int) -> int:
    import ctypes

    p = ctypes.c_void_p()
    _lib.check(_lib.lib().cbp_ipc_open(ctypes.create_string_buffer(handle, 64), offset, ctypes.byref(p)))
    return int(p.value)


def ipc_close(ptr: int, offset: int) -> None:
    _lib.check(_lib.lib().cbp_ipc_close(ptr, offset))


def backproject_multi(img_dev, mats: np.ndarray, slabs: list, k_bounds, nx: int, ny: int, nz: int,
                      devices: list[int] | None = None, variant: KernelVariant = KernelVariant.BASELINE,
                      n_chunks: int = 8, flags: int = 0) -> dict:
    """Single-process multi-GPU z-slab back-projection (cbp_backproject_multi): ``img_dev``
    NATURAL on devices[0], ``slabs[r]`` the NATURAL slab tensor of rank r on devices[r]
    (``None`` for empty slabs).  Synchronous; returns the summed status counters."""
    import ctypes

    n = len(slabs)
    devices = [s.device.index if s is not None else 0 for s in slabs] if devices is None else list(devices)
    if len(devices) != n or len(k_bounds) != n + 1:
        raise ValueError("need one device and one slab per rank and n_ranks + 1 slice bounds")
    n_proj, nh, nw = (int(v) for v in img_dev.shape)
    _check_tensor(img_dev, (n_proj, nh, nw), "projections")
    for r, t in enumerate(slabs):
        depth = int(k_bounds[r + 1]) - int(k_bounds[r])
        if depth > 0:
            _check_tensor(t, (depth, ny, nx), f"slab {r}")
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() if t is not None else 0 for t in slabs])
    devs = (ctypes.c_int * n)(*devices)
    kb = np.ascontiguousarray(np.asarray(k_bounds, dtype=np.int64))
    st = np.zeros(5, np.int64)
    rc = _lib.lib().cbp_backproject_multi(img_dev.data_ptr(), n_proj, nh, nw, _lib.f32ptr(mats), ptrs, nx, ny, nz,
                                          _lib.i64ptr(kb), n, devs, int(KernelVariant(variant)), flags, n_chunks,
                                          _lib.i64ptr(st))
    stats = {"smem_pairs": int(st[0]), "global_pairs": int(st[1]), "skipped_pairs": int(st[2]),
             "band_violations": int(st[3]), "box_misses": int(st[4])}
    _lib.check(rc)
    return stats


def selftest_rcp(lo_bits: int, hi_bits: int) -> tuple[int, int]:
    """(mismatches, first mismatching bit pattern) of rcp_rn_normal vs __frcp_rn."""
    import ctypes

    n = ctypes.c_uint64()
    first = ctypes.c_uint32()
    _lib.check(_lib.lib().cbp_selftest_rcp(lo_bits, hi_bits, ctypes.byref(n), ctypes.byref(first)))
    return int(n.value), int(first.value)


def backproject_device(img_dev, mats: np.ndarray, vol_dev, n_proj: int, nh: int, nw: int, nx: int, ny: int, nz: int,
                       variant: KernelVariant = KernelVariant.BASELINE, img_layout: Layout = Layout.NATURAL,
                       vol_layout: Layout = Layout.NATURAL, flags: int = 0, stream=None) -> None:
    """One-call device path (stages internally when needed), stream-ordered."""
    img_layout, vol_layout = Layout(img_layout), Layout(vol_layout)
    _check_tensor(img_dev, (n_proj, nh, nw) if img_layout is Layout.NATURAL else (n_proj, nw, nh), "projections")
    _check_tensor(vol_dev, _vol_shape(nx, ny, nz, vol_layout), "volume")
    mats = np.ascontiguousarray(mats, dtype=np.float32)
    _lib.check(_lib.lib().cbp_backproject_f32(
        img_dev.data_ptr(), n_proj, nh, nw, 0 if img_layout is Layout.NATURAL else 1, _lib.f32ptr(mats),
        vol_dev.data_ptr(), nx, ny, nz, 0 if vol_layout is Layout.NATURAL else 1, int(KernelVariant(variant)), flags,
        stream_handle(stream)))


def sync_status(stream=None) -> dict:
    """Synchronise and return device-side counters; raises on band violations."""
    st = np.zeros(5, np.int64)
    rc = _lib.lib().cbp_sync_status(stream_handle(stream), _lib.i64ptr(st))
    stats = {"smem_pairs": int(st[0]), "global_pairs": int(st[1]), "skipped_pairs": int(st[2]),
             "band_violations": int(st[3]), "box_misses": int(st[4])}
    _lib.check(rc)
    return stats


def last_plan() -> dict:
    out = np.zeros(9, np.int64)
    _lib.check(_lib.lib().cbp_last_plan(_lib.i64ptr(out)))
    keys = ["tile_x", "tile_y", "tile_z", "box_w", "box_h", "stages", "blocks", "smem_bytes", "kernel_kind"]
    return dict(zip(keys, (int(v) for v in out)))
