"""Tolerance mode CBP_FLAG_FMA_LERP (opt-in; the default stays bit-exact).

The three bilinear lerps become one FMA each (x + a*(y - x)) and the accumulation
one FMA: 11 instead of 16 FP32 lane-ops per update on the fast path.  The
coordinates, guards and truncation keep the reference's exact float32 order, so
only the interpolation rounding differs from /root/reference/pkg/src/conebp/
_kernels.py:57-61.  North-star tolerance, asserted on all five BASELINE configs
against the C oracle: max|d| <= 1e-4 * max|ref| and relL2 <= 1e-5 (float64
metrics; full volumes for configs 0-2, z-slab subsets with global indices for
configs 3-4).  The measured metrics are written to gpurun_out/fma_lerp_metrics.json
when that directory exists.
"""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2104_13248_b200 import _lib

pytestmark = pytest.mark.gpu

MAX_REL = 1e-4
REL_L2 = 1e-5
OUT = Path(__file__).resolve().parents[1] / "gpurun_out"


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def metrics(out, ref):
    d = np.abs(out.astype(np.float64) - ref.astype(np.float64))
    mx = float(np.abs(ref).max()) or 1.0
    rel = float(np.sqrt((d ** 2).sum()) / max(np.sqrt((ref.astype(np.float64) ** 2).sum()), 1e-300))
    return float(d.max()) / mx, rel


def record(name, mx, rel):
    if OUT.is_dir():
        p = OUT / "fma_lerp_metrics.json"
        data = json.loads(p.read_text()) if p.exists() else {}
        data[name] = {"max_abs_over_max_ref": mx, "rel_l2": rel}
        p.write_text(json.dumps(data, indent=1))


@pytest.mark.parametrize("index", [0, 1, 2, 3, 4])
def test_fma_lerp_within_north_star_tolerance(torch_cuda, index):
    from paper_2104_13248_b200 import configs, geometry as G
    from paper_2104_13248_b200 import device as D

    torch = torch_cuda
    spec = configs.get_config(index)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    n_proj, nh, nw, nx, ny, nz = geom.np, geom.nh, geom.nw, geom.nx, geom.ny, geom.nz
    img = spec.projections_device(geom, device="cuda")
    vol = torch.zeros((nz, ny, nx), device="cuda")
    D.backproject_device(img, mats, vol, n_proj, nh, nw, nx, ny, nz, flags=_lib.FLAG_FMA_LERP)
    st = D.sync_status()
    assert st["band_violations"] == 0 and st["smem_pairs"] > 0
    if index <= 2:
        slabs = [(0, nz)]
    else:
        slabs = [(0, 2), (nz // 2 - 1, nz // 2 + 1), (nz // 3, nz // 3 + 1), (nz - 2, nz)]
    outs, refs = [], []
    for k0, k1 in slabs:
        ref = np.zeros((k1 - k0, ny, nx), np.float32)
        if index <= 2:
            oracle.baseline(img.cpu().numpy(), mats, ref)
        else:
            v0, rows = G.slab_band(mats, nh, nw, nx, ny, nz, k0, k1)
            if rows:
                band = img[:, v0:v0 + rows, :].contiguous().cpu().numpy()
                oracle.baseline(band, mats, ref, nh=nh, v0=v0, k_lo=k0)
        outs.append(vol[k0:k1].cpu().numpy())
        refs.append(ref)
    out, ref = np.concatenate(outs), np.concatenate(refs)
    mx, rel = metrics(out, ref)
    record(spec.name, mx, rel)
    assert mx <= MAX_REL and rel <= REL_L2, (spec.name, mx, rel)
    assert out.tobytes() != ref.tobytes() or index == 0  # it is a different rounding, not the exact path


def test_fma_lerp_is_rejected_outside_the_baseline_tiled_kernel(torch_cuda):
    from conftest import load_golden
    from paper_2104_13248_b200 import KernelVariant
    from paper_2104_13248_b200 import device as D

    torch = torch_cuda
    g = load_golden("uoffset")
    n_proj, nh, nw = g["img"].shape
    nz, ny, nx = g["vol0"].shape
    img = torch.from_numpy(g["img"]).cuda()
    vol = torch.zeros((nz, ny, nx), device="cuda")
    with pytest.raises(ValueError, match="FMA_LERP"):
        D.backproject_device(img, g["mats"], vol, n_proj, nh, nw, nx, ny, nz, KernelVariant.BASELINE,
                             flags=_lib.FLAG_FMA_LERP | _lib.FLAG_NAIVE)
    img_t = torch.from_numpy(np.ascontiguousarray(g["img"].transpose(0, 2, 1))).cuda()
    vol_t = torch.zeros((nx, ny, nz), device="cuda")
    from paper_2104_13248_b200 import Layout

    with pytest.raises(ValueError, match="FMA_LERP"):
        D.backproject_device(img_t, g["mats"], vol_t, n_proj, nh, nw, nx, ny, nz, KernelVariant.SHARE,
                             Layout.TRANSPOSED, Layout.TRANSPOSED, flags=_lib.FLAG_FMA_LERP)
