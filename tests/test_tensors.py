"""Containers and layouts (mirrors pkg/tests/test_tensors.py behaviour)."""

import numpy as np
import pytest

from paper_2104_13248_b200 import tensors as T


def test_layout_shapes_and_zeros():
    p = T.ProjectionStack.zeros(3, 5, 7)
    assert p.data.shape == (3, 5, 7) and p.layout is T.Layout.NATURAL
    pt = T.ProjectionStack.zeros(3, 5, 7, T.Layout.TRANSPOSED)
    assert pt.data.shape == (3, 7, 5)
    v = T.Volume.zeros(2, 3, 4)
    assert v.data.shape == (4, 3, 2)
    assert T.Volume.zeros(2, 3, 4, "transposed").data.shape == (2, 3, 4)


def test_from_array_infers_dims_and_coerces():
    p = T.ProjectionStack.from_array(np.ones((2, 3, 4), np.float64))
    assert (p.np, p.nh, p.nw) == (2, 3, 4) and p.data.dtype == np.float32
    pt = T.ProjectionStack.from_array(np.ones((2, 4, 3)), T.Layout.TRANSPOSED)
    assert (pt.nh, pt.nw) == (3, 4)
    v = T.Volume.from_array(np.ones((4, 3, 2)))
    assert (v.nx, v.ny, v.nz) == (2, 3, 4)
    with pytest.raises(ValueError):
        T.ProjectionStack.from_array(np.ones((2, 3)))
    with pytest.raises(ValueError):
        T.Volume(np.ones((2, 2, 2)), 3, 2, 2)
    with pytest.raises(ValueError):
        T.Volume.zeros(0, 1, 1)


def test_transposes_are_involutions():
    rng = np.random.default_rng(0)
    p = T.ProjectionStack.from_array(rng.random((3, 5, 7), dtype=np.float32))
    pt = T.transpose_projections(p)
    assert pt.layout is T.Layout.TRANSPOSED and pt.data[1, 6, 4] == p.data[1, 4, 6]
    assert T.transpose_projections(pt).data.tobytes() == p.data.tobytes()
    v = T.Volume.from_array(rng.random((4, 3, 2), dtype=np.float32))
    vt = T.transpose_volume(v)
    assert vt.data[1, 2, 3] == v.data[3, 2, 1]
    assert T.transpose_volume(vt).data.tobytes() == v.data.tobytes()
    with pytest.raises(TypeError):
        T.transpose_volume(p)


def test_ij_list_order():
    ij = T.make_ij_list(3, 2).pairs
    assert ij.tolist() == [[0, 0], [1, 0], [2, 0], [0, 1], [1, 1], [2, 1]]
    assert not ij.flags.writeable
    with pytest.raises(ValueError):
        T.make_ij_list(0, 2)


def test_raw_io_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    p = T.ProjectionStack.from_array(rng.random((2, 3, 4), dtype=np.float32), T.Layout.TRANSPOSED)
    T.save_projections(tmp_path / "p.raw", p)
    q = T.load_projections(tmp_path / "p.raw")
    assert q.layout is p.layout and q.data.tobytes() == p.data.tobytes()
    v = T.Volume.from_array(rng.random((4, 3, 2), dtype=np.float32))
    T.save_volume(tmp_path / "v.raw", v)
    assert T.load_volume(tmp_path / "v.raw").data.tobytes() == v.data.tobytes()
    (tmp_path / "v.raw").write_bytes(b"\0" * 8)
    with pytest.raises(ValueError):
        T.load_volume(tmp_path / "v.raw")
