"""Scan geometry and 3x4 projection matrices (host side of the hot path).

Keeps the public surface of ``conebp.geometry`` (/root/reference/pkg/src/
conebp/geometry.py:46-292): ``ScanGeometry``, ``build_geometry``,
``projection_matrix``/``projection_matrices`` (circular orbit, composed in
float64, stored float32), ``apply_matrix`` (kernel float32 order) and the JSON /
raw I/O.  Added for the B200 build:

* ``pinhole_matrix``        general pinhole composition from source, detector
                            centre and detector axes (world units);
* ``jittered_matrices``     per-angle seeded Gaussian jitter of source and
                            detector-centre positions (BASELINE config 2);
* ``u_offset``              principal-point shift in u (config 4: +16 px);
* ``slab_band`` / ``slab_plan``  detector-row footprint of a z-slab and the
                            cost-balanced slab partition used by the multi-GPU
                            driver -- computed by libconebp_b200's host planner
                            with the kernels' own float32 corner arithmetic.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np

__all__ = [
    "ScanGeometry",
    "ProjectionMatrix",
    "build_geometry",
    "projection_matrix",
    "projection_matrices",
    "apply_matrix",
    "pinhole_matrix",
    "View",
    "circular_views",
    "jittered_views",
    "view_matrices",
    "jittered_matrices",
    "u_offset",
    "has_vertical_columns",
    "slab_band",
    "slab_plan",
    "save_geometry",
    "load_geometry",
    "save_matrices",
    "load_matrices",
]

# auto-fit constants of the reference (geometry.py:40-43)
DETECTOR_MARGIN = 2.0
PITCH_SLACK = 1.02


@dataclass(frozen=True)
class ScanGeometry:
    """Circular cone-beam scan and the voxel grid it reconstructs into.

    ``d`` source-to-axis, ``D`` source-to-detector (world units); detector V is
    parallel to the rotation axis Z; the isotropic grid is centred on the axis.
    """

    d: float
    D: float
    nw: int
    nh: int
    pixel_pitch_u: float
    pixel_pitch_v: float
    voxel_size: float
    np: int
    angles: tuple[float, ...]
    nx: int
    ny: int
    nz: int

    def __post_init__(self):
        checks = [
            (self.d > 0, f"source distance d must be > 0, got {self.d}"),
            (self.D >= self.d, f"detector distance D must be >= d, got D={self.D}, d={self.d}"),
            (self.nw >= 2 and self.nh >= 2, f"detector must be at least 2x2 pixels, got {self.nw}x{self.nh}"),
            (self.np >= 1, "need at least one projection"),
            (min(self.nx, self.ny, self.nz) >= 1, f"degenerate volume {self.nx}x{self.ny}x{self.nz}"),
            (self.pixel_pitch_u > 0 and self.pixel_pitch_v > 0 and self.voxel_size > 0,
             "pixel pitches and voxel size must be positive"),
            (len(self.angles) == self.np, f"expected {self.np} angles, got {len(self.angles)}"),
            (all(math.isfinite(a) for a in self.angles), "angles must be finite"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        if self.axis_radius >= self.d:
            raise ValueError(f"volume XY radius {self.axis_radius:.3f} reaches the source orbit d={self.d}")

    @property
    def axis_radius(self) -> float:
        return 0.5 * self.voxel_size * math.hypot(self.nx - 1, self.ny - 1)

    @property
    def detector_center(self) -> tuple[float, float]:
        return ((self.nw - 1) / 2.0, (self.nh - 1) / 2.0)

    @property
    def grid_origin(self) -> tuple[float, float, float]:
        """Index-space centre of the grid (world origin)."""
        return ((self.nx - 1) / 2.0, (self.ny - 1) / 2.0, (self.nz - 1) / 2.0)


@dataclass(frozen=True)
class ProjectionMatrix:
    """3x4 float32 map of homogeneous voxel indices to (u*z, v*z, z)."""

    m: np.ndarray

    def __post_init__(self):
        m = np.ascontiguousarray(self.m, dtype=np.float32)
        if m.shape != (3, 4):
            raise ValueError(f"projection matrix must be 3x4, got {m.shape}")
        if not np.isfinite(m).all():
            raise ValueError("projection matrix has non-finite entries")
        object.__setattr__(self, "m", m)


def build_geometry(*, nx: int, ny: int, nz: int, nw: int, nh: int, np: int, d: float | None = None,
                   D: float | None = None, pixel_pitch_u: float | None = None, pixel_pitch_v: float | None = None,
                   voxel_size: float = 1.0, angles=None) -> ScanGeometry:
    """Circular scan; omitted distances / pitches are fitted as in geometry.py:120-187."""
    n_proj = np
    if min(nx, ny, nz) < 1:
        raise ValueError(f"degenerate volume {nx}x{ny}x{nz}")
    if voxel_size <= 0:
        raise ValueError("voxel size must be positive")
    r_xy = 0.5 * voxel_size * math.hypot(nx - 1, ny - 1)
    r_z = 0.5 * voxel_size * (nz - 1)
    d = 2.5 * max(r_xy, voxel_size) if d is None else d
    D = 1.536 * d if D is None else D
    if d <= r_xy:
        raise ValueError(f"d={d} too small: volume XY radius is {r_xy:.3f}")
    closest = d - r_xy  # worst-case magnification
    half_u = (nw - 1) / 2.0 - DETECTOR_MARGIN
    half_v = (nh - 1) / 2.0 - DETECTOR_MARGIN
    if half_u <= 0 or half_v <= 0:
        raise ValueError(f"detector {nw}x{nh} too small for the border margin")
    if pixel_pitch_u is None:
        pixel_pitch_u = PITCH_SLACK * D * max(r_xy, voxel_size) / (closest * half_u)
    if pixel_pitch_v is None:
        pixel_pitch_v = PITCH_SLACK * D * max(r_z, voxel_size) / (closest * half_v)
    if angles is None:
        angles = tuple(2.0 * math.pi * s / n_proj for s in range(n_proj))
    else:
        angles = tuple(float(a) for a in angles)
    return ScanGeometry(d=float(d), D=float(D), nw=int(nw), nh=int(nh), pixel_pitch_u=float(pixel_pitch_u),
                        pixel_pitch_v=float(pixel_pitch_v), voxel_size=float(voxel_size), np=int(n_proj),
                        angles=angles, nx=int(nx), ny=int(ny), nz=int(nz))


def _circular_rows(geom: ScanGeometry, angle: float) -> np.ndarray:
    """float64 rows of the circular-orbit matrix (same composition as geometry.py:190-211)."""
    s = geom.voxel_size
    ox, oy, oz = geom.grid_origin
    cu, cv = geom.detector_center
    mu, mv = geom.D / geom.pixel_pitch_u, geom.D / geom.pixel_pitch_v
    c, sn = math.cos(angle), math.sin(angle)
    depth = np.array([c * s, sn * s, 0.0, geom.d - s * (c * ox + sn * oy)])
    urow = np.array([-sn * s * mu, c * s * mu, 0.0, mu * s * (sn * ox - c * oy)]) + cu * depth
    vrow = np.array([0.0, 0.0, mv * s, -mv * s * oz]) + cv * depth
    return np.stack([urow, vrow, depth])


def _corner_depths(geom: ScanGeometry, m64: np.ndarray) -> np.ndarray:
    ii, jj, kk = np.meshgrid([0, geom.nx - 1], [0, geom.ny - 1], [0, geom.nz - 1], indexing="ij")
    pts = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.float64)
    return pts @ m64[2, :3] + m64[2, 3]


def _finish(geom: ScanGeometry, m64: np.ndarray) -> ProjectionMatrix:
    if not (_corner_depths(geom, m64) > 0).all():
        raise ValueError("geometry yields non-positive depth inside the volume")
    return ProjectionMatrix(m=m64.astype(np.float32))


def projection_matrix(geom: ScanGeometry, angle_index: int) -> ProjectionMatrix:
    """Matrix of one angle; IndexError out of range, ValueError for non-positive depth."""
    if not 0 <= angle_index < geom.np:
        raise IndexError(f"angle index {angle_index} out of range [0, {geom.np})")
    return _finish(geom, _circular_rows(geom, geom.angles[angle_index]))


def projection_matrices(geom: ScanGeometry) -> np.ndarray:
    """All matrices of the scan as float32 (np, 3, 4) (geometry.py:234-242)."""
    return np.stack([projection_matrix(geom, s).m for s in range(geom.np)]).astype(np.float32)


def apply_matrix(m: np.ndarray, i, j, k):
    """(u, v, z) of voxel indices in the kernels' float32 order (geometry.py:245-258)."""
    m = np.asarray(m, dtype=np.float32)
    fi, fj, fk = (np.asarray(a, dtype=np.float32) for a in (i, j, k))
    z = ((m[2, 0] * fi + m[2, 1] * fj) + m[2, 2] * fk) + m[2, 3]
    f = np.float32(1.0) / z
    u = (((m[0, 0] * fi + m[0, 1] * fj) + m[0, 2] * fk) + m[0, 3]) * f
    v = (((m[1, 0] * fi + m[1, 1] * fj) + m[1, 2] * fk) + m[1, 3]) * f
    return u, v, z


def pinhole_matrix(geom: ScanGeometry, source, det_center, e_u, e_v, u0: float | None = None,
                   v0: float | None = None) -> np.ndarray:
    """float64 3x4 matrix of a general pinhole view.

    ``source`` and ``det_center`` are world positions, ``e_u``/``e_v`` unit
    detector axes; the normal is the unit vector from the source to the detector
    centre.  Depth is the distance along that normal (so z = d at the isocentre
    of an unperturbed circular view, as geometry.py normalises it) and (u, v) are
    pixel coordinates with principal point (u0, v0) (default: detector centre).
    """
    S = np.asarray(source, dtype=np.float64)
    C = np.asarray(det_center, dtype=np.float64)
    eu = np.asarray(e_u, dtype=np.float64)
    ev = np.asarray(e_v, dtype=np.float64)
    n = C - S
    dist = float(np.linalg.norm(n))
    n = n / dist
    cu, cv = geom.detector_center
    u0 = cu if u0 is None else u0
    v0 = cv if v0 is None else v0
    s = geom.voxel_size
    org = np.asarray(geom.grid_origin, dtype=np.float64) * s

    def affine(vec):  # vec . (P - S) with P = s*(i,j,k) - org
        return np.concatenate([s * vec, [-float(vec @ (org + S))]])

    depth = affine(n)
    # hit - C = (S - C) + (P - S) * dist/depth, so u*depth = a_u*depth + (dist/pu) e_u.(P-S)
    a_u = u0 + float((S - C) @ eu) / geom.pixel_pitch_u
    a_v = v0 + float((S - C) @ ev) / geom.pixel_pitch_v
    urow = a_u * depth + (dist / geom.pixel_pitch_u) * affine(eu)
    vrow = a_v * depth + (dist / geom.pixel_pitch_v) * affine(ev)
    return np.stack([urow, vrow, depth])


@dataclass(frozen=True)
class View:
    """World pose of one projection: source, detector centre, unit detector axes."""

    source: tuple
    det_center: tuple
    e_u: tuple
    e_v: tuple


def circular_views(geom: ScanGeometry) -> list[View]:
    """Poses of the circular orbit behind projection_matrices."""
    views = []
    for ang in geom.angles:
        c, sn = math.cos(ang), math.sin(ang)
        views.append(View((-geom.d * c, -geom.d * sn, 0.0), ((geom.D - geom.d) * c, (geom.D - geom.d) * sn, 0.0),
                          (-sn, c, 0.0), (0.0, 0.0, 1.0)))
    return views


def jittered_views(geom: ScanGeometry, sigma: float, seed: int) -> list[View]:
    """Circular poses with seeded Gaussian jitter of source and detector centre.

    For each angle in order, ``np.random.default_rng(seed)`` draws 3 source
    offsets then 3 detector-centre offsets (world units, std ``sigma``).  The
    detector normal follows the perturbed source -> centre ray; e_v is world Z
    orthogonalised against it and e_u = e_v x n.
    """
    rng = np.random.default_rng(seed)
    views = []
    for ang in geom.angles:
        c, sn = math.cos(ang), math.sin(ang)
        src = np.array([-geom.d * c, -geom.d * sn, 0.0]) + rng.normal(0.0, sigma, 3)
        det = np.array([(geom.D - geom.d) * c, (geom.D - geom.d) * sn, 0.0]) + rng.normal(0.0, sigma, 3)
        n = (det - src) / np.linalg.norm(det - src)
        ev = np.array([0.0, 0.0, 1.0]) - n[2] * n
        ev /= np.linalg.norm(ev)
        eu = np.cross(ev, n)
        views.append(View(tuple(src), tuple(det), tuple(eu), tuple(ev)))
    return views


def view_matrices(geom: ScanGeometry, views: list[View]) -> np.ndarray:
    """float32 (np, 3, 4) matrices of arbitrary poses (depth checked at the grid corners)."""
    out = np.empty((len(views), 3, 4), dtype=np.float32)
    for s, v in enumerate(views):
        out[s] = _finish(geom, pinhole_matrix(geom, v.source, v.det_center, v.e_u, v.e_v)).m
    return out


def jittered_matrices(geom: ScanGeometry, sigma: float, seed: int) -> np.ndarray:
    """Matrices of ``jittered_views``: the u and depth rows get non-zero k coefficients."""
    return view_matrices(geom, jittered_views(geom, sigma, seed))


def u_offset(mats: np.ndarray, pixels: float) -> np.ndarray:
    """Shift the principal point by ``pixels`` in u: m[s,0,:] += pixels * m[s,2,:]."""
    m = np.array(mats, dtype=np.float64)
    m[:, 0, :] += pixels * m[:, 2, :]
    return m.astype(np.float32)


def has_vertical_columns(mats: np.ndarray) -> bool:
    """True when every u and depth row has a zero k coefficient (geometry.py:204,206)."""
    m = np.asarray(mats, dtype=np.float32)
    return bool((m[:, 0, 2] == 0).all() and (m[:, 2, 2] == 0).all())


def slab_band(mats: np.ndarray, nh: int, nw: int, nx: int, ny: int, nz: int, k0: int, k1: int,
              variant: int = 0) -> tuple[int, int]:
    """Detector rows [v0, v0+rows) sampled by slices [k0, k1) (rows == 0: none)."""
    from . import _lib

    m = np.ascontiguousarray(mats, dtype=np.float32)
    v0 = np.zeros(1, np.int64)
    rows = np.zeros(1, np.int64)
    _lib.check(_lib.lib().cbp_slab_band(_lib.f32ptr(m), m.shape[0], nh, nw, nx, ny, nz, int(variant), k0, k1,
                                        _lib.i64ptr(v0), _lib.i64ptr(rows)))
    return int(v0[0]), int(rows[0])


def slab_plan(mats: np.ndarray, nh: int, nw: int, nx: int, ny: int, nz: int, n_ranks: int, align: int = 32,
              variant: int = 0) -> tuple[list[int], list[tuple[int, int]]]:
    """Cost-balanced contiguous z-slabs (boundaries on multiples of ``align``) and their row bands."""
    from . import _lib

    m = np.ascontiguousarray(mats, dtype=np.float32)
    kb = np.zeros(n_ranks + 1, np.int64)
    bands = np.zeros(2 * n_ranks, np.int64)
    _lib.check(_lib.lib().cbp_slab_plan(_lib.f32ptr(m), m.shape[0], nh, nw, nx, ny, nz, int(variant), n_ranks, align,
                                        _lib.i64ptr(kb), _lib.i64ptr(bands)))
    return [int(k) for k in kb], [(int(bands[2 * r]), int(bands[2 * r + 1])) for r in range(n_ranks)]


def save_geometry(path, geom: ScanGeometry) -> None:
    doc = asdict(geom)
    doc["angles"] = list(geom.angles)
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2)
        fh.write("\n")


def load_geometry(path) -> ScanGeometry:
    with open(path) as fh:
        doc = json.load(fh)
    try:
        doc["angles"] = tuple(float(a) for a in doc["angles"])
        return ScanGeometry(**doc)
    except (KeyError, TypeError) as exc:
        raise ValueError(f"invalid geometry document {path}: {exc}") from exc


def save_matrices(path, mats: np.ndarray) -> None:
    mats = np.asarray(mats, dtype=np.float32)
    if mats.ndim != 3 or mats.shape[1:] != (3, 4):
        raise ValueError(f"expected (np, 3, 4) matrices, got {mats.shape}")
    mats.astype("<f4").tofile(path)


def load_matrices(path, n_proj: int) -> np.ndarray:
    flat = np.fromfile(path, dtype="<f4")
    if flat.size != n_proj * 12:
        raise ValueError(f"{path}: expected {n_proj * 12} floats, found {flat.size}")
    return flat.reshape(n_proj, 3, 4).astype(np.float32)
