"""FDK pre-processing on the GPU (row f1): cosine weight + Ram-Lak filter vs a float64
direct-convolution restatement (tolerance: FFT vs direct summation order), and an
end-to-end FDK reconstruction sanity check against the rasterised truth."""

import math

import numpy as np
import pytest

from paper_2104_13248_b200 import geometry as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def filter_reference(raw, geom):
    """float64 direct evaluation of the definition (zero-padded linear convolution)."""
    n_proj, nh, nw = raw.shape
    cu, cv = geom.detector_center
    u = (np.arange(nw) - cu) * geom.pixel_pitch_u
    v = (np.arange(nh) - cv) * geom.pixel_pitch_v
    w = geom.D / np.sqrt(geom.D ** 2 + u[None, :] ** 2 + v[:, None] ** 2)
    x = raw.astype(np.float64) * w.astype(np.float32)[None].astype(np.float64)
    tau = geom.pixel_pitch_u * geom.d / geom.D
    n = np.arange(-(nw - 1), nw).astype(float)
    h = np.zeros_like(n)
    h[n == 0] = 1.0 / (4 * tau * tau)
    odd = np.abs(n) % 2 == 1
    h[odd] = -1.0 / (math.pi ** 2 * n[odd] ** 2 * tau * tau)
    out = np.empty_like(x)
    for s in range(n_proj):
        for r in range(nh):
            out[s, r] = tau * np.convolve(x[s, r], h)[nw - 1: 2 * nw - 1]
    return out


def test_filter_matches_float64_definition(torch_cuda):
    torch = torch_cuda
    from paper_2104_13248_b200 import fdk

    geom = G.build_geometry(nx=16, ny=16, nz=16, nw=37, nh=21, np=3, d=100.0, D=160.0, pixel_pitch_u=0.9,
                            pixel_pitch_v=1.1, voxel_size=1.0)
    raw = np.random.default_rng(4).uniform(0.0, 2.0, (3, 21, 37)).astype(np.float32)
    staged = fdk.filter_projections(torch.from_numpy(raw).cuda(), geom)
    got = staged.data.cpu().numpy()[:, :, :37].astype(np.float64)
    ref = filter_reference(raw, geom)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 1e-5, rel
    assert np.all(staged.data.cpu().numpy()[:, :, 37:] == 0)


@pytest.mark.parametrize("nw,nh,n_proj", [(2, 3, 2), (3, 2, 3), (5, 3, 1), (9, 5, 1), (17, 2, 2), (40, 3, 3),
                                          (100, 7, 1), (300, 5, 3), (513, 3, 1), (1100, 2, 3), (2100, 3, 1)])
def test_filter_every_transform_length(torch_cuda, nw, nh, n_proj):
    """One case per transform length 2^2 .. 2^13 of the fused filter kernel (radix-8 passes
    with an innermost radix of 8, 4 or 2), odd row counts included (rows are filtered in
    pairs), against the float64 definition."""
    torch = torch_cuda
    import types

    from paper_2104_13248_b200 import _lib
    from paper_2104_13248_b200.device import stream_handle

    # detectors this small are below build_geometry's border margin: call the C ABI directly
    geom = types.SimpleNamespace(D=170.0, d=100.0, pixel_pitch_u=0.8, pixel_pitch_v=1.2,
                                 detector_center=((nw - 1) / 2.0, (nh - 1) / 2.0))
    raw = np.random.default_rng(nw).uniform(-1.0, 2.0, (n_proj, nh, nw)).astype(np.float32)
    pitch = int(_lib.lib().cbp_staged_pitch(nw))
    raw_dev = torch.from_numpy(raw).cuda()
    staged = torch.full((n_proj, nh, pitch), float("nan"), dtype=torch.float32, device="cuda")
    cu, cv = geom.detector_center
    _lib.check(_lib.lib().cbp_fdk_filter_f32(raw_dev.data_ptr(), n_proj, nh, nw, geom.D, geom.pixel_pitch_u,
                                             geom.pixel_pitch_v, cu, cv, geom.pixel_pitch_u * geom.d / geom.D,
                                             staged.data_ptr(), pitch, stream_handle()))
    full = staged.cpu().numpy()
    got = full[:, :, :nw].astype(np.float64)
    ref = filter_reference(raw, geom)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 1e-5, rel
    assert np.abs(got - ref).max() <= 1e-4 * np.abs(ref).max()
    assert np.all(full[:, :, nw:] == 0)


def test_filter_matches_phantom_pipeline(torch_cuda):
    torch = torch_cuda
    from paper_2104_13248_b200 import fdk, phantom

    geom = G.build_geometry(nx=32, ny=32, nz=32, nw=64, nh=48, np=6, d=200.0, D=320.0, pixel_pitch_u=1.0,
                            pixel_pitch_v=1.0, voxel_size=1.0)
    raw = torch.rand((6, 48, 64), device="cuda")
    staged = fdk.filter_projections(raw, geom)
    ref = phantom.ramp_filter(phantom.cosine_weight(raw.clone(), geom), geom)
    got = staged.data[:, :, :64]
    rel = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    assert rel < 1e-5, rel


def test_fdk_reconstruction_recovers_the_phantom(torch_cuda):
    from paper_2104_13248_b200 import fdk, phantom

    geom = G.build_geometry(nx=48, ny=48, nz=48, nw=128, nh=128, np=180, d=300.0, D=450.0, pixel_pitch_u=0.75,
                            pixel_pitch_v=0.75, voxel_size=1.0)
    ph = phantom.EllipsoidPhantom((phantom.Ellipsoid((0.0, 0.0, 0.0), (16.0, 14.0, 12.0), 1.0),))
    truth = phantom.rasterize_phantom(ph, (48, 48, 48), 1.0)
    raw = phantom.forward_project(truth, geom)
    vol = fdk.fdk_reconstruct(raw, geom)
    inner = truth.data[20:28, 20:28, 20:28]
    rec = vol.data[20:28, 20:28, 20:28]
    assert abs(float(rec.mean()) - float(inner.mean())) < 0.08 * float(inner.mean())
    outside = vol.data[:, :4, :4]
    assert abs(float(outside.mean())) < 0.1

