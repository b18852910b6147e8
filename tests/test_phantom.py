"""Phantom pipeline: rasteriser (host) and forward projector (GPU)
bit for bit against the reference's conebp.phantom outputs (tests/golden/forward.npz)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2104_13248_b200 import geometry as G
from paper_2104_13248_b200 import phantom as P

ODD = P.EllipsoidPhantom((P.Ellipsoid((1.0, -1.0, 0.5), (2.5, 1.6, 2.0), 0.8, 0.4),
                          P.Ellipsoid((-1.2, 0.8, -0.5), (1.2, 1.8, 1.4), 0.5, -0.7)))


def tiny_geom():
    return G.build_geometry(nx=12, ny=12, nz=12, nw=24, nh=24, np=8)


def odd_geom():
    return G.build_geometry(nx=16, ny=14, nz=10, nw=40, nh=28, np=7, d=30.0, D=45.0, voxel_size=1.0,
                            angles=[0.0, 0.3, 1.0, 1.5707963267948966, 2.2, 3.141592653589793, 4.0])


def test_rasterizer_bitwise():
    g = load_golden("forward")
    geom = tiny_geom()
    t = P.rasterize_phantom(P.default_phantom(12, 12, 12, geom.voxel_size), (12, 12, 12), geom.voxel_size)
    assert t.data.tobytes() == g["tiny_truth"].tobytes()
    assert P.rasterize_phantom(ODD, (16, 14, 10), 1.0).data.tobytes() == g["odd_truth"].tobytes()


def test_phantom_validation_and_io(tmp_path):
    with pytest.raises(ValueError):
        P.Ellipsoid((0, 0, 0), (1, 0, 1), 1.0)
    with pytest.raises(ValueError):
        P.rasterize_phantom(ODD, (4, 4, 4), 1.0)
    with pytest.raises(ValueError):
        P.rasterize_phantom(P.EllipsoidPhantom((P.Ellipsoid((5, 0, 0), (3, 3, 3), 1.0),)), (8, 8, 8), 1.0)
    P.save_phantom(tmp_path / "p.json", ODD)
    assert P.load_phantom(tmp_path / "p.json") == ODD


@pytest.mark.gpu
def test_forward_projector_bitwise():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = load_golden("forward")
    from paper_2104_13248_b200.tensors import Volume

    p1 = P.forward_project(Volume.from_array(g["tiny_truth"]), tiny_geom())
    assert p1.data.tobytes() == g["tiny_proj"].tobytes()
    p2 = P.forward_project(Volume.from_array(g["odd_truth"]), odd_geom())
    assert p2.data.tobytes() == g["odd_proj"].tobytes()
    # voxel sizes other than 1: 0.5 (multiplication by the exact reciprocal) and 0.7 (division)
    for tag, vs in (("half", 0.5), ("p7", 0.7)):
        g3 = G.build_geometry(nx=10, ny=12, nz=9, nw=30, nh=22, np=5, d=20.0, D=33.0, voxel_size=vs,
                              pixel_pitch_u=0.6, pixel_pitch_v=0.55)
        p3 = P.forward_project(Volume.from_array(g[f"{tag}_truth"]), g3)
        assert p3.data.tobytes() == g[f"{tag}_proj"].tobytes(), tag


@pytest.mark.gpu
def test_make_dataset_matches_reference_fixture():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    # tests/golden/tiny.npz holds conebp.make_dataset(build_geometry(12^3, 24^2, 8)) outputs
    t = load_golden("tiny")
    truth, proj, mats = P.make_dataset(tiny_geom())
    assert mats.tobytes() == t["mats"].tobytes()
    assert proj.data.tobytes() == t["img"].tobytes()
