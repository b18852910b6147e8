"""Complete FDK on the GPU: pre-processing (row f1) + the back-projection hot path.

The reference stops at back-projection of already-filtered projections (SPEC.md:8,
SURVEY F5).  This module adds the standard circular-orbit FDK pre-processing on the
device, written straight into the back-projector's staging layout:

* ``filter_projections`` -- cosine weight ``D / sqrt(D^2 + u^2 + v^2)`` and row-wise
  spatial Ram-Lak filter (tau = pixel pitch scaled to the isocentre), exactly the
  definition of :func:`paper_2104_13248_b200.phantom.cosine_weight` /
  :func:`~paper_2104_13248_b200.phantom.ramp_filter`, computed by
  ``cbp_fdk_filter_f32`` (one fused kernel: weight, zero-padded shared-memory FFT of
  two rows per complex transform, exact Ram-Lak spectrum, inverse, crop into the
  staging layout -- each row read once and written once);
* ``fdk_reconstruct`` -- filter, back-project (reference BASELINE arithmetic), scale
  by ``pi * d^2 / np`` (dbeta/2 with the reference's 1/z^2 weight, z = d at the
  isocentre) for a full 360-degree orbit.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .backprojector import KernelVariant
from .tensors import Layout, ProjectionStack, Volume

__all__ = ["ramp_tau", "filter_projections", "fdk_reconstruct", "fdk_scale", "check_full_orbit"]


def ramp_tau(geom) -> float:
    """Detector pitch scaled to the rotation axis (the Ram-Lak sampling interval)."""
    return geom.pixel_pitch_u * geom.d / geom.D


def fdk_scale(geom) -> float:
    """pi * d^2 / np: dbeta / 2 times the d^2 that turns the kernel's 1/z^2 into FDK's d^2/U^2."""
    return math.pi * geom.d * geom.d / geom.np


def filter_projections(img_dev, geom, stream=None):
    """Weighted + Ram-Lak filtered projections in the staging layout (device)."""
    import torch

    from .device import StagedProjections, _check_tensor, stream_handle

    _check_tensor(img_dev, (geom.np, geom.nh, geom.nw), "raw projections")
    pitch = int(_lib.lib().cbp_staged_pitch(geom.nw))
    out = torch.empty((geom.np, geom.nh, pitch), dtype=torch.float32, device=img_dev.device)
    cu, cv = geom.detector_center
    _lib.check(_lib.lib().cbp_fdk_filter_f32(img_dev.data_ptr(), geom.np, geom.nh, geom.nw, float(geom.D),
                                             float(geom.pixel_pitch_u), float(geom.pixel_pitch_v), float(cu),
                                             float(cv), float(ramp_tau(geom)), out.data_ptr(), pitch,
                                             stream_handle(stream)))
    return StagedProjections.wrap(out, geom.np, geom.nh, geom.nw, 0, geom.nh)


def check_full_orbit(geom, rtol: float = 1e-6) -> None:
    """FDK's pi * d^2 / np scale assumes angles evenly spaced over a whole turn (each ray
    measured twice, no redundancy weighting).  Short scans (e.g. config 2's 200 degrees)
    need Parker weights, which this module does not implement: they are rejected."""
    a = np.sort(np.mod(np.asarray(geom.angles, dtype=np.float64), 2.0 * math.pi))
    n = a.size
    if n < 2:
        raise ValueError("FDK needs projections over a full 360-degree orbit (got one angle)")
    gaps = np.diff(np.concatenate([a, [a[0] + 2.0 * math.pi]]))
    step = 2.0 * math.pi / n
    if np.abs(gaps - step).max() > max(rtol * 2.0 * math.pi, 1e-9) + 1e-6 * step:
        raise ValueError("fdk_reconstruct needs angles evenly spaced over a full 360-degree orbit "
                         "(short scans need Parker weighting, which is not implemented)")


def fdk_reconstruct(proj: ProjectionStack, geom, mats: np.ndarray | None = None) -> Volume:
    """Raw (unfiltered) NATURAL projections -> FDK volume (host in, host out).

    Full circular orbits only (``check_full_orbit``)."""
    import torch

    from .device import backproject_staged, sync_status
    from .geometry import projection_matrices

    if proj.layout is not Layout.NATURAL:
        raise ValueError("fdk_reconstruct expects NATURAL projections")
    if (proj.np, proj.nh, proj.nw) != (geom.np, geom.nh, geom.nw):
        raise ValueError("projection stack does not match the geometry")
    check_full_orbit(geom)
    mats = projection_matrices(geom) if mats is None else np.ascontiguousarray(mats, np.float32)
    img = torch.from_numpy(proj.data).cuda()
    staged = filter_projections(img, geom)
    vol = torch.zeros((geom.nz, geom.ny, geom.nx), dtype=torch.float32, device=img.device)
    backproject_staged(staged, mats, vol, geom.nx, geom.ny, geom.nz, KernelVariant.BASELINE)
    vol.mul_(fdk_scale(geom))
    sync_status()
    return Volume(vol.cpu().numpy(), geom.nx, geom.ny, geom.nz, Layout.NATURAL)
