"""Host geometry: matrices bitwise equal to the reference's, invariants of
pkg/tests/test_geometry.py, the general pinhole / jitter builders and the
slab planner (host-only functions of libconebp_b200.so)."""

import json
import math

import numpy as np
import pytest

from conftest import load_golden
from paper_2104_13248_b200 import geometry as G


def test_circular_matrices_bitwise_equal_reference():
    # the golden tiny / const_kat matrices came from conebp.projection_matrices
    geom = G.build_geometry(nx=12, ny=12, nz=12, nw=24, nh=24, np=8)
    assert G.projection_matrices(geom).tobytes() == load_golden("tiny")["mats"].tobytes()
    g9 = G.build_geometry(nx=9, ny=9, nz=9, nw=32, nh=32, np=1)
    assert G.projection_matrices(g9).tobytes() == load_golden("const_kat")["mats"].tobytes()
    g0 = G.build_geometry(nx=64, ny=64, nz=64, nw=128, nh=128, np=90, d=1000.0, D=1500.0, pixel_pitch_u=1.0,
                          pixel_pitch_v=1.0, voxel_size=0.5)
    assert G.projection_matrices(g0).tobytes() == load_golden("cfg0")["mats"].tobytes()


def test_default_angles_and_errors():
    geom = G.build_geometry(nx=8, ny=8, nz=8, nw=16, nh=16, np=4)
    assert geom.angles == pytest.approx((0.0, math.pi / 2, math.pi, 3 * math.pi / 2))
    base = dict(nx=8, ny=8, nz=8, nw=16, nh=16, np=4, d=100.0, D=150.0)
    for bad in (dict(d=0.0), dict(D=10.0), dict(nw=1), dict(np=0), dict(nx=0), dict(voxel_size=0.0),
                dict(pixel_pitch_u=-1.0)):
        with pytest.raises(ValueError):
            G.build_geometry(**{**base, **bad})
    with pytest.raises(ValueError):
        G.build_geometry(nx=300, ny=300, nz=300, nw=64, nh=64, np=4, d=100.0, D=150.0)
    with pytest.raises(IndexError):
        G.projection_matrix(geom, 4)
    with pytest.raises(ValueError):
        G.ProjectionMatrix(m=np.full((3, 4), np.nan, np.float32))


def test_center_voxel_principal_point_and_zero_k():
    geom = G.build_geometry(nx=17, ny=17, nz=17, nw=33, nh=33, np=12)
    mats = G.projection_matrices(geom)
    assert G.has_vertical_columns(mats)
    cu, cv = geom.detector_center
    for s in range(geom.np):
        u, v, z = G.apply_matrix(mats[s], 8, 8, 8)
        assert abs(float(u) - cu) < 1e-4 and abs(float(v) - cv) < 1e-4
        assert abs(float(z) - geom.d) < 1e-3 * geom.d


def test_pinhole_builder_matches_circular_orbit():
    geom = G.build_geometry(nx=32, ny=32, nz=32, nw=64, nh=64, np=16, d=100.0, D=150.0)
    circ = G.projection_matrices(geom)
    gen = G.view_matrices(geom, G.circular_views(geom))
    ii, jj, kk = np.meshgrid(np.arange(0, 32, 5), np.arange(0, 32, 5), np.arange(0, 32, 5), indexing="ij")
    for s in range(geom.np):
        a = G.apply_matrix(circ[s], ii, jj, kk)
        b = G.apply_matrix(gen[s], ii, jj, kk)
        for x, y in zip(a, b):
            assert np.abs(x - y).max() < 1e-3


def ray_oracle(view, geom, wx, wy, wz, u0=None):
    S = np.array(view.source)
    C = np.array(view.det_center)
    n = (C - S) / np.linalg.norm(C - S)
    P = np.array([wx, wy, wz])
    t = np.dot(C - S, n) / np.dot(P - S, n)
    hit = S + t * (P - S)
    cu, cv = geom.detector_center
    return (cu + np.dot(hit - C, view.e_u) / geom.pixel_pitch_u, cv + np.dot(hit - C, view.e_v) / geom.pixel_pitch_v)


def test_jittered_matrices_agree_with_ray_oracle():
    geom = G.build_geometry(nx=64, ny=64, nz=64, nw=160, nh=128, np=24, d=200.0, D=320.0, pixel_pitch_u=0.5,
                            pixel_pitch_v=0.5, voxel_size=1.0)
    views = G.jittered_views(geom, 0.5, 2)
    mats = G.view_matrices(geom, views)
    assert not G.has_vertical_columns(mats)
    rng = np.random.default_rng(1)
    ox, oy, oz = geom.grid_origin
    for s in range(geom.np):
        for _ in range(20):
            i, j, k = rng.integers(0, 64, 3)
            u, v, z = G.apply_matrix(mats[s], i, j, k)
            uo, vo = ray_oracle(views[s], geom, (i - ox), (j - oy), (k - oz))
            assert abs(float(u) - uo) < 2e-3 and abs(float(v) - vo) < 2e-3 and float(z) > 0


def test_u_offset_shifts_principal_point():
    geom = G.build_geometry(nx=17, ny=17, nz=17, nw=64, nh=33, np=6)
    m = G.u_offset(G.projection_matrices(geom), 16.0)
    cu, _ = geom.detector_center
    for s in range(geom.np):
        u, _, _ = G.apply_matrix(m[s], 8, 8, 8)
        assert abs(float(u) - (cu + 16.0)) < 1e-3


def test_geometry_io_roundtrip(tmp_path):
    geom = G.build_geometry(nx=8, ny=10, nz=12, nw=20, nh=24, np=5)
    G.save_geometry(tmp_path / "g.json", geom)
    assert G.load_geometry(tmp_path / "g.json") == geom
    assert "angles" in json.loads((tmp_path / "g.json").read_text())
    mats = G.projection_matrices(geom)
    G.save_matrices(tmp_path / "m.raw", mats)
    assert G.load_matrices(tmp_path / "m.raw", 5).tobytes() == mats.tobytes()
    with pytest.raises(ValueError):
        G.load_matrices(tmp_path / "m.raw", 6)
