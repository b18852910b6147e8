"""Synthetic inputs for the BASELINE.json configurations (test/bench scaffolding).

The reference ships only a rasterised phantom and a ray-marching forward
projector (/root/reference/pkg/src/conebp/phantom.py:36-268); BASELINE.json
asks for inputs it does not have, so they are generated here:

* ``uniform_projections``   i.i.d. uniform[-1, 1) float32 from
  ``np.random.default_rng(seed)``, drawn in (np, nh, nw) order (configs 0, 4
  and the parity fixtures); ``uniform_projections_device`` is the torch-RNG
  stand-in used where host generation of tens of GiB would dominate;
* ``random_ellipsoids``     seeded ellipsoid phantoms (centres uniform in the
  inner 80% of the field of view, semi-axes a fraction of it, densities
  uniform[0.1, 1));
* ``ellipsoid_projections`` analytic chord-length line integrals through every
  detector pixel centre (source and detector pose per view, so jittered views
  are simulated with their own geometry);
* ``cosine_weight`` / ``ramp_filter``  FDK pre-weighting D/sqrt(D^2+u^2+v^2) and a
  row-wise spatial Ram-Lak filter (FFT convolution, zero padded), in float32.

Input values never affect parity (oracle and GPU read the same arrays); they
only set the realistic value distribution.  ``rmse`` matches phantom.py:271-287.
"""

from __future__ import annotations

import math
import numpy as np

__all__ = [
    "uniform_projections",
    "uniform_projections_device",
    "random_ellipsoids",
    "ellipsoid_projections",
    "cosine_weight",
    "ramp_filter",
    "filtered_phantom_projections",
    "rmse",
]


def uniform_projections(n_proj: int, nh: int, nw: int, seed: int) -> np.ndarray:
    """default_rng(seed).uniform(-1, 1, (np, nh, nw)) as float32, drawn per projection."""
    rng = np.random.default_rng(seed)
    out = np.empty((n_proj, nh, nw), np.float32)
    for s in range(n_proj):  # same stream as one big draw, without the float64 copy
        out[s] = rng.uniform(-1.0, 1.0, size=(nh, nw))
    return out


def uniform_projections_device(n_proj: int, nh: int, nw: int, seed: int, device="cuda"):
    """torch-RNG uniform[-1, 1) float32 on ``device`` (large configs)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((n_proj, nh, nw), dtype=torch.float32, device=device)
    for s in range(n_proj):
        out[s].uniform_(-1.0, 1.0, generator=g)
    return out


def random_ellipsoids(n: int, geom, semi_frac=(0.05, 0.40), seed: int = 0) -> np.ndarray:
    """(n, 8) rows: centre xyz, semi-axes xyz, rotation about z, density."""
    rng = np.random.default_rng(seed)
    hx = 0.5 * geom.nx * geom.voxel_size
    hy = 0.5 * geom.ny * geom.voxel_size
    hz = 0.5 * geom.nz * geom.voxel_size
    fov = min(hx, hy)
    out = np.empty((n, 8), np.float64)
    out[:, 0] = rng.uniform(-0.8 * hx, 0.8 * hx, n)
    out[:, 1] = rng.uniform(-0.8 * hy, 0.8 * hy, n)
    out[:, 2] = rng.uniform(-0.8 * hz, 0.8 * hz, n)
    out[:, 3:6] = rng.uniform(semi_frac[0], semi_frac[1], (n, 3)) * fov
    out[:, 6] = rng.uniform(0.0, math.pi, n)
    out[:, 7] = rng.uniform(0.1, 1.0, n)
    return out


def ellipsoid_projections(geom, views: list, ellipsoids: np.ndarray, device="cpu", batch: int = 8):
    """Analytic line integrals, float32 tensor (np, nh, nw) on ``device``."""
    import torch

    dt = torch.float64
    cu, cv = geom.detector_center
    iu = (torch.arange(geom.nw, dtype=dt, device=device) - cu) * geom.pixel_pitch_u
    iv = (torch.arange(geom.nh, dtype=dt, device=device) - cv) * geom.pixel_pitch_v
    out = torch.empty((len(views), geom.nh, geom.nw), dtype=torch.float32, device=device)
    ell = torch.as_tensor(ellipsoids, dtype=dt, device=device)
    for b0 in range(0, len(views), batch):
        vb = views[b0:b0 + batch]
        S = torch.tensor([v.source for v in vb], dtype=dt, device=device)[:, None, None, :]
        C = torch.tensor([v.det_center for v in vb], dtype=dt, device=device)[:, None, None, :]
        eu = torch.tensor([v.e_u for v in vb], dtype=dt, device=device)[:, None, None, :]
        ev = torch.tensor([v.e_v for v in vb], dtype=dt, device=device)[:, None, None, :]
        P = C + iu[None, None, :, None] * eu + iv[None, :, None, None] * ev  # (b, nh, nw, 3)
        ray = P - S
        length = torch.linalg.vector_norm(ray, dim=-1)
        acc = torch.zeros(P.shape[:3], dtype=dt, device=device)
        for e in ell:
            c, sn = torch.cos(e[6]), torch.sin(e[6])
            # rotate into the ellipsoid frame (inverse rotation about z), then scale to a unit sphere
            def to_frame(vec):
                x = c * vec[..., 0] + sn * vec[..., 1]
                y = -sn * vec[..., 0] + c * vec[..., 1]
                return x / e[3], y / e[4], vec[..., 2] / e[5]

            q = to_frame(S - e[0:3])
            r = to_frame(ray)
            A = r[0] * r[0] + r[1] * r[1] + r[2] * r[2]
            B = q[0] * r[0] + q[1] * r[1] + q[2] * r[2]
            Cq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] - 1.0
            disc = torch.clamp(B * B - A * Cq, min=0.0)
            acc += e[7] * (2.0 * torch.sqrt(disc) / A) * length
        out[b0:b0 + len(vb)] = acc.to(torch.float32)
    return out


def cosine_weight(proj, geom):
    """FDK pre-weight D / sqrt(D^2 + u^2 + v^2) (u, v in world units on the detector), in place."""
    import torch

    cu, cv = geom.detector_center
    u = (torch.arange(geom.nw, dtype=torch.float64, device=proj.device) - cu) * geom.pixel_pitch_u
    v = (torch.arange(geom.nh, dtype=torch.float64, device=proj.device) - cv) * geom.pixel_pitch_v
    w = geom.D / torch.sqrt(geom.D ** 2 + u[None, :] ** 2 + v[:, None] ** 2)
    proj.mul_(w.to(torch.float32)[None])
    return proj


def ramp_filter(proj, geom):
    """Row-wise spatial Ram-Lak filter (h[0]=1/4t^2, h[odd n]=-1/(n pi t)^2), float32, in place.

    t is the detector pitch scaled to the isocentre; rows are zero padded to a
    power of two >= 2*nw before the FFT convolution.
    """
    import torch

    nw = geom.nw
    tau = geom.pixel_pitch_u * geom.d / geom.D
    n_fft = 1 << int(math.ceil(math.log2(2 * nw)))
    n = torch.arange(n_fft, device=proj.device)
    n = torch.where(n < n_fft // 2, n, n - n_fft).to(torch.float32)  # circular indices
    h = torch.zeros(n_fft, dtype=torch.float32, device=proj.device)
    h[n == 0] = 1.0 / (4.0 * tau * tau)
    odd = (n.abs() % 2) == 1
    h[odd] = -1.0 / (math.pi * math.pi * tau * tau * n[odd] * n[odd])
    H = torch.fft.rfft(h)
    for s in range(proj.shape[0]):
        row = torch.fft.rfft(proj[s], n=n_fft, dim=-1)
        proj[s] = (torch.fft.irfft(row * H, n=n_fft, dim=-1)[..., :nw] * tau).to(torch.float32)
    return proj


def filtered_phantom_projections(geom, views, ellipsoids, device="cpu"):
    """Analytic projections -> cosine weight -> ramp filter (float32, natural layout)."""
    proj = ellipsoid_projections(geom, views, ellipsoids, device=device)
    cosine_weight(proj, geom)
    ramp_filter(proj, geom)
    return proj


def rmse(a, b) -> float:
    """Root mean square difference in float64 (phantom.py:271-287)."""
    from .tensors import ProjectionStack, Volume

    if isinstance(a, (Volume, ProjectionStack)) or isinstance(b, (Volume, ProjectionStack)):
        if type(a) is not type(b):
            raise ValueError("rmse operands must be the same container type")
        if a.data.shape != b.data.shape or a.layout is not b.layout:
            raise ValueError(f"rmse operands must share dims and layout, got {a.data.shape}/{a.layout.value} "
                             f"vs {b.data.shape}/{b.layout.value}")
        a, b = a.data, b.data
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"rmse operands must share shape, got {a.shape} vs {b.shape}")
    return float(math.sqrt(np.mean((a - b) ** 2)))


# ---------------------------------------------------------------------------
# the reference's phantom pipeline (conebp.phantom, phantom.py:36-322): ellipsoid
# phantom, rasteriser (host, numpy float64: bitwise equal), forward projector on the
# GPU (libconebp_b200 cbp_forward_project_f32: bitwise equal), dataset helper

from dataclasses import dataclass as _dataclass
import json as _json


@_dataclass(frozen=True)
class Ellipsoid:
    """Axis-aligned ellipsoid rotated about Z; world units and radians (phantom.py:36-53)."""

    center: tuple
    semi_axes: tuple
    intensity: float
    rotation: float = 0.0

    def __post_init__(self):
        if len(self.center) != 3 or len(self.semi_axes) != 3:
            raise ValueError("center and semi_axes must have three components")
        if min(self.semi_axes) <= 0:
            raise ValueError(f"semi-axes must be positive, got {self.semi_axes}")

    @property
    def bounding_radius(self) -> float:
        return math.hypot(*self.center) + max(self.semi_axes)


@_dataclass(frozen=True)
class EllipsoidPhantom:
    """A set of ellipsoids; voxel values sum the intensities containing them."""

    ellipsoids: tuple

    def check_fits(self, dims, voxel_size: float) -> None:
        radius = 0.5 * min(dims) * voxel_size
        for e in self.ellipsoids:
            if e.bounding_radius > radius:
                raise ValueError(f"ellipsoid at {e.center} (bounding radius {e.bounding_radius:.3f}) "
                                 f"exceeds the inscribed sphere radius {radius:.3f}")


def default_phantom(nx: int, ny: int, nz: int, voxel_size: float = 1.0) -> EllipsoidPhantom:
    """Nested off-centre ellipsoids scaled to the volume (phantom.py:73-87)."""
    r = 0.5 * min(nx, ny, nz) * voxel_size
    return EllipsoidPhantom((
        Ellipsoid((0.0, 0.0, 0.0), (0.60 * r, 0.80 * r, 0.70 * r), 0.5, 0.35),
        Ellipsoid((-0.22 * r, -0.18 * r, -0.28 * r), (0.22 * r, 0.16 * r, 0.20 * r), 0.2, 0.6),
        Ellipsoid((0.26 * r, 0.22 * r, 0.17 * r), (0.12 * r, 0.17 * r, 0.11 * r), 0.3, -0.8),
        Ellipsoid((0.02 * r, -0.32 * r, 0.33 * r), (0.24 * r, 0.12 * r, 0.18 * r), 0.2, 2.1),
    ))


def rasterize_phantom(ph: EllipsoidPhantom, dims, voxel_size: float = 1.0):
    """Voxel value = sum of the intensities of the ellipsoids containing the voxel centre.

    float64 evaluation in the reference's order (phantom.py:90-131), vectorised over
    the grid and accumulated ellipsoid by ellipsoid, stored as float32.
    """
    from .tensors import Layout, Volume

    nx, ny, nz = (int(d) for d in dims)
    if min(nx, ny, nz) < 8:
        raise ValueError(f"phantom grids start at 8^3, got {nx}x{ny}x{nz}")
    ph.check_fits((nx, ny, nz), voxel_size)
    s = float(voxel_size)
    wz = ((np.arange(nz) - (nz - 1) / 2.0) * s)[:, None, None]
    wy = ((np.arange(ny) - (ny - 1) / 2.0) * s)[None, :, None]
    wx = ((np.arange(nx) - (nx - 1) / 2.0) * s)[None, None, :]
    value = np.zeros((nz, ny, nx), np.float64)
    for e in ph.ellipsoids:
        c, sn = math.cos(e.rotation), math.sin(e.rotation)
        dx = wx - e.center[0]
        dy = wy - e.center[1]
        dz = wz - e.center[2]
        px = c * dx + sn * dy
        py = -sn * dx + c * dy
        q = (px / e.semi_axes[0]) ** 2 + (py / e.semi_axes[1]) ** 2 + (dz / e.semi_axes[2]) ** 2
        value = value + np.where(q <= 1.0, e.intensity, 0.0)
    return Volume(value.astype(np.float32), nx, ny, nz, Layout.NATURAL)


def _views_array(views) -> np.ndarray:
    return np.ascontiguousarray(
        np.array([tuple(v.source) + tuple(v.det_center) + tuple(v.e_u) + tuple(v.e_v) for v in views], np.float64))


def forward_project(vol, geom, views=None):
    """Line integrals through every detector pixel centre, on the GPU (phantom.py:225-252).

    ``views`` defaults to the circular orbit of ``geom`` (jittered poses may be passed).
    Returns a NATURAL ProjectionStack (host numpy), bitwise equal to the reference.
    """
    import torch

    from . import _lib
    from .geometry import circular_views
    from .tensors import Layout, ProjectionStack

    if vol.layout is not Layout.NATURAL:
        raise ValueError("forward_project expects a NATURAL volume")
    if (vol.nx, vol.ny, vol.nz) != (geom.nx, geom.ny, geom.nz):
        raise ValueError(f"volume {vol.nx}x{vol.ny}x{vol.nz} does not match geometry grid "
                         f"{geom.nx}x{geom.ny}x{geom.nz}")
    va = _views_array(circular_views(geom) if views is None else views)
    cu, cv = geom.detector_center
    v_dev = torch.from_numpy(vol.data).cuda()
    out = torch.empty((geom.np, geom.nh, geom.nw), dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().cbp_forward_project_f32(
        v_dev.data_ptr(), vol.nx, vol.ny, vol.nz, float(geom.voxel_size),
        va.ctypes.data_as(_lib.POINTER(_lib.ctypes.c_double)), geom.np, geom.nh, geom.nw, float(geom.pixel_pitch_u),
        float(geom.pixel_pitch_v), float(cu), float(cv), out.data_ptr(), stream))
    torch.cuda.current_stream().synchronize()
    return ProjectionStack(out.cpu().numpy(), geom.np, geom.nh, geom.nw, Layout.NATURAL)


def make_dataset(geom, phantom=None):
    """Rasterise, forward project (GPU), normalise to peak 1 (phantom.py:255-268)."""
    from .geometry import projection_matrices

    if phantom is None:
        phantom = default_phantom(geom.nx, geom.ny, geom.nz, geom.voxel_size)
    truth = rasterize_phantom(phantom, (geom.nx, geom.ny, geom.nz), geom.voxel_size)
    proj = forward_project(truth, geom)
    peak = float(proj.data.max())
    if peak > 0:
        proj.data /= np.float32(peak)
    return truth, proj, projection_matrices(geom)


def save_phantom(path, ph: EllipsoidPhantom) -> None:
    doc = {"ellipsoids": [{"center": list(e.center), "semi_axes": list(e.semi_axes), "intensity": e.intensity,
                           "rotation": e.rotation} for e in ph.ellipsoids]}
    with open(path, "w") as fh:
        _json.dump(doc, fh, indent=2)
        fh.write("\n")


def load_phantom(path) -> EllipsoidPhantom:
    with open(path) as fh:
        doc = _json.load(fh)
    try:
        ells = tuple(Ellipsoid(center=tuple(float(c) for c in e["center"]),
                               semi_axes=tuple(float(c) for c in e["semi_axes"]), intensity=float(e["intensity"]),
                               rotation=float(e.get("rotation", 0.0))) for e in doc["ellipsoids"])
    except (KeyError, TypeError) as exc:
        raise ValueError(f"invalid phantom document {path}: {exc}") from exc
    return EllipsoidPhantom(ellipsoids=ells)
