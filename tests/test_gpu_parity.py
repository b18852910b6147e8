"""GPU parity: libconebp_b200 (sm_100a) vs the reference, bit for bit.

Golden vectors come from the live reference (tests/golden/make_golden.py);
larger cases are checked against the C oracle (itself pinned to the reference
in test_oracle_golden.py) and, at BASELINE.json's full sizes, through
sha256 digests of reference outputs (big_sha.json) and voxel-subset oracles.
Tolerance (north star): max|d| <= 1e-4 max|ref| and relL2 <= 1e-5 -- the
kernels are bitwise identical, so every check here is exact equality and the
tolerance metrics are reported for information.
"""

import hashlib
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, RUNG_NAMES, SMALL_CASES, load_golden, uniform
from paper_2104_13248_b200 import (
    KernelVariant,
    Layout,
    ProjectionStack,
    Volume,
    backproject,
    backproject_baseline,
    backproject_optimized,
    transpose_projections,
)
from paper_2104_13248_b200 import _lib

pytestmark = pytest.mark.gpu

RUNG = {n: KernelVariant[n.upper()] for n in RUNG_NAMES}
FLAG_SETS = {"tiled": 0, "naive": _lib.FLAG_NAIVE, "tiled_global": _lib.FLAG_NO_SMEM, "tiled_check": _lib.FLAG_CHECK}


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert _lib.lib().cbp_device_count() > 0
    return torch


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tol_metrics(out, ref):
    d = np.abs(out.astype(np.float64) - ref.astype(np.float64))
    mx = float(np.abs(ref).max()) or 1.0
    rel = float(np.sqrt((d ** 2).sum()) / max(np.sqrt((ref.astype(np.float64) ** 2).sum()), 1e-300))
    return float(d.max()) / mx, rel


def run_device(torch, img, mats, vol0, variant, img_layout, vol_layout, flags):
    from paper_2104_13248_b200 import device as D

    n_proj = img.shape[0]
    if img_layout is Layout.NATURAL:
        nh, nw = img.shape[1:]
    else:
        nw, nh = img.shape[1:]
    if vol_layout is Layout.NATURAL:
        nz, ny, nx = vol0.shape
    else:
        nx, ny, nz = vol0.shape
    ti = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    tv = torch.from_numpy(np.ascontiguousarray(vol0)).cuda()
    D.backproject_device(ti, mats, tv, n_proj, nh, nw, nx, ny, nz, variant, img_layout, vol_layout, flags=flags)
    stats = D.sync_status()
    assert stats["band_violations"] == 0
    if flags & _lib.FLAG_CHECK:
        assert stats["box_misses"] == 0, "a sample fell outside its tile's TMA footprint box"
    return tv.cpu().numpy(), stats


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("path", list(FLAG_SETS))
def test_baseline_bitwise_small(torch_cuda, case, path):
    g = load_golden(case)
    out, _ = run_device(torch_cuda, g["img"], g["mats"], g["vol0"], KernelVariant.BASELINE, Layout.NATURAL,
                        Layout.NATURAL, FLAG_SETS[path])
    assert out.tobytes() == g["baseline"].tobytes()


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("rung", RUNG_NAMES)
@pytest.mark.parametrize("path", ["tiled", "naive"])
def test_rungs_bitwise_small(torch_cuda, case, rung, path):
    g = load_golden(case)
    if rung not in g:
        pytest.skip("odd nz")
    img_t = np.ascontiguousarray(g["img"].transpose(0, 2, 1))
    vol_t = np.ascontiguousarray(g["vol0"].transpose(2, 1, 0))
    out, _ = run_device(torch_cuda, img_t, g["mats"], vol_t, RUNG[rung], Layout.TRANSPOSED, Layout.TRANSPOSED,
                        FLAG_SETS[path])
    assert out.tobytes() == g[rung].tobytes()


@pytest.mark.parametrize("case", ["tiny", "ragged", "tilted", "uoffset"])
def test_numpy_dropin_api_bitwise(torch_cuda, case):
    g = load_golden(case)
    nz, ny, nx = g["vol0"].shape
    proj = ProjectionStack.from_array(g["img"])
    vol = Volume(g["vol0"].copy(), nx, ny, nz)
    ret = backproject_baseline(proj, g["mats"], vol)
    assert ret is vol and vol.data.tobytes() == g["baseline"].tobytes()
    img_t = transpose_projections(proj)
    nb = int(g["nb"])
    for rung in RUNG_NAMES:
        if rung not in g:
            continue
        vt = Volume(np.ascontiguousarray(g["vol0"].transpose(2, 1, 0)), nx, ny, nz, Layout.TRANSPOSED)
        backproject(img_t, g["mats"], vt, RUNG[rung], batch=nb)
        assert vt.data.tobytes() == g[rung].tobytes(), rung


@pytest.mark.parametrize("case", SMALL_CASES)
def test_count_mode_matches_twin(torch_cuda, case):
    g = load_golden(case)
    nz, ny, nx = g["vol0"].shape
    proj = ProjectionStack.from_array(g["img"])
    vol, c = backproject_baseline(proj, g["mats"], Volume(g["vol0"].copy(), nx, ny, nz), count=True)
    assert vol.data.tobytes() == g["baseline"].tobytes()
    got = [c.dot_ops, c.vol_word_accesses, c.proj_word_accesses, c.interp_ops, c.subline_builds]
    assert got == g["count_baseline"].tolist()
    img_t = transpose_projections(proj)
    for rung in RUNG_NAMES:
        if "count_" + rung not in g:
            continue
        vt = Volume(np.ascontiguousarray(g["vol0"].transpose(2, 1, 0)), nx, ny, nz, Layout.TRANSPOSED)
        _, c = backproject_optimized(img_t, g["mats"], vt, RUNG[rung], batch=int(g["nb"]), count=True)
        got = [c.dot_ops, c.vol_word_accesses, c.proj_word_accesses, c.interp_ops, c.subline_builds]
        assert got == g["count_" + rung].tolist(), rung


def test_known_answers(torch_cuda):
    # constant image, single projection: centre voxel = c / d^2 (test_backprojector.py:101-109)
    g = load_golden("const_kat")
    proj = ProjectionStack.from_array(g["img"])
    vol = backproject_baseline(proj, g["mats"], Volume.zeros(9, 9, 9))
    d = 2.5 * 0.5 * np.hypot(8, 8)  # auto-fitted source distance of build_geometry(9^3)
    assert float(vol.data[4, 4, 4]) == pytest.approx(0.75 / d ** 2, rel=1e-5)
    # zero projections leave a random start volume bitwise unchanged (accumulate semantics)
    t = load_golden("tiny")
    start = np.abs(np.random.default_rng(5).normal(size=(12, 12, 12))).astype(np.float32)
    v = Volume.from_array(start.copy())
    backproject_baseline(ProjectionStack.zeros(8, 24, 24), t["mats"], v)
    assert v.data.tobytes() == start.tobytes()


def test_cfg0_bitwise_all_paths(torch_cuda):
    g = load_golden("cfg0")
    img = uniform(90, 128, 128, 0)
    assert sha(img) == g["input_sha"].item().decode()
    for flags in FLAG_SETS.values():
        out, _ = run_device(torch_cuda, img, g["mats"], np.zeros((64, 64, 64), np.float32), KernelVariant.BASELINE,
                            Layout.NATURAL, Layout.NATURAL, flags)
        assert out.tobytes() == g["baseline"].tobytes()
    digests = json.loads(g["rung_sha"].item().decode())
    img_t = np.ascontiguousarray(img.transpose(0, 2, 1))
    for rung, digest in digests.items():
        out, _ = run_device(torch_cuda, img_t, g["mats"], np.zeros((64, 64, 64), np.float32), RUNG[rung],
                            Layout.TRANSPOSED, Layout.TRANSPOSED, 0)
        assert sha(out) == digest, rung


def big_sha():
    p = GOLDEN / "big_sha.json"
    return json.loads(p.read_text()) if p.exists() else None


def test_cfg1_size_bitwise_vs_reference_digests(torch_cuda):
    ref = big_sha()
    if ref is None:
        pytest.skip("big_sha.json not generated")
    from paper_2104_13248_b200 import configs

    spec = configs.get_config(1)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    r = ref["cfg1_uniform11"]
    assert sha(mats) == r["mats_sha"]
    img = uniform(360, 512, 512, 11)
    assert sha(img) == r["input_sha"]
    out, stats = run_device(torch_cuda, img, mats, np.zeros((256, 256, 256), np.float32), KernelVariant.BASELINE,
                            Layout.NATURAL, Layout.NATURAL, 0)
    assert sha(out) == r["baseline"]
    assert stats["smem_pairs"] > 0
    img_t = np.ascontiguousarray(img.transpose(0, 2, 1))
    for rung in RUNG_NAMES:
        out, _ = run_device(torch_cuda, img_t, mats, np.zeros((256, 256, 256), np.float32), RUNG[rung],
                            Layout.TRANSPOSED, Layout.TRANSPOSED, 0)
        assert sha(out) == r[rung], rung


def test_cfg2_jitter_bitwise_vs_reference_digest(torch_cuda):
    ref = big_sha()
    if ref is None or not (GOLDEN / "cfg2_mats.npy").exists():
        pytest.skip("big_sha.json not generated")
    r = ref["cfg2_uniform12"]
    mats = np.load(GOLDEN / "cfg2_mats.npy")
    assert sha(mats) == r["mats_sha"]
    img = uniform(496, 960, 1248, 12)
    assert sha(img) == r["input_sha"]
    out, _ = run_device(torch_cuda, img, mats, np.zeros((512, 512, 512), np.float32), KernelVariant.BASELINE,
                        Layout.NATURAL, Layout.NATURAL, 0)
    assert sha(out) == r["baseline"]


def test_cfg1_phantom_inputs_vs_oracle(torch_cuda):
    """Config 1 as specified (filtered ellipsoid phantom): GPU == C oracle, full volume."""
    from paper_2104_13248_b200 import configs

    spec = configs.get_config(1)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    img_dev = spec.projections_device(geom, device="cuda")
    img = img_dev.cpu().numpy()
    out, _ = run_device(torch_cuda, img, mats, np.zeros((256, 256, 256), np.float32), KernelVariant.BASELINE,
                        Layout.NATURAL, Layout.NATURAL, 0)
    ref = np.zeros((256, 256, 256), np.float32)
    oracle.baseline(img, mats, ref)
    mx, rel = tol_metrics(out, ref)
    assert mx <= 1e-4 and rel <= 1e-5
    assert out.tobytes() == ref.tobytes()


def _big_config_slab_check(torch_cuda, index, slabs):
    """Full-size config: GPU volume vs the C oracle on thin z-slabs (global indices),
    each slab evaluated from only its detector-row band copied back to the host."""
    from paper_2104_13248_b200 import configs, geometry as G
    from paper_2104_13248_b200 import device as D

    torch = torch_cuda
    spec = configs.get_config(index)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    img = torch.rand((geom.np, geom.nh, geom.nw), device="cuda", generator=torch.Generator("cuda").manual_seed(index))
    img = img * 2 - 1
    vol = torch.zeros((geom.nz, geom.ny, geom.nx), dtype=torch.float32, device="cuda")
    D.backproject_device(img, mats, vol, geom.np, geom.nh, geom.nw, geom.nx, geom.ny, geom.nz)
    stats = D.sync_status()
    assert stats["band_violations"] == 0 and stats["smem_pairs"] > 0
    checked = 0
    for k0, k1 in slabs:
        v0, rows = G.slab_band(mats, geom.nh, geom.nw, geom.nx, geom.ny, geom.nz, k0, k1)
        got = vol[k0:k1].cpu().numpy()
        ref = np.zeros((k1 - k0, geom.ny, geom.nx), np.float32)
        if rows:
            band = img[:, v0:v0 + rows, :].contiguous().cpu().numpy()
            assert oracle.baseline(band, mats, ref, nh=geom.nh, v0=v0, k_lo=k0) == 0
        assert got.tobytes() == ref.tobytes(), (index, k0, k1)
        checked += int(np.count_nonzero(ref))
    assert checked > 0


def test_cfg3_full_size_slabs_bitwise(torch_cuda):
    _big_config_slab_check(torch_cuda, 3, [(0, 1), (511, 513), (1023, 1024)])


def test_cfg4_full_size_slabs_bitwise(torch_cuda):
    _big_config_slab_check(torch_cuda, 4, [(0, 1), (700, 701), (1023, 1025), (2047, 2048)])


def test_band_violation_is_reported(torch_cuda):
    """A slab given a too-narrow band must fail loudly (CBP_EBAND), never silently."""
    from paper_2104_13248_b200 import device as D
    from paper_2104_13248_b200._lib import CbpError

    torch = torch_cuda
    g = load_golden("uoffset")
    n_proj, nh, nw = g["img"].shape
    img = torch.from_numpy(g["img"]).cuda()
    staged = D.StagedProjections(img, n_proj, nh, nw, v0=10, rows=6)  # far too few rows
    vol = torch.zeros((8, 32, 32), dtype=torch.float32, device="cuda")
    D.backproject_staged(staged, g["mats"], vol, 32, 32, 8, k0=12, nz_total=32)
    with pytest.raises(CbpError):
        D.sync_status()


@pytest.mark.parametrize("tile_cfg", range(7))
def test_every_tile_shape_bitwise(torch_cuda, tile_cfg):
    """Every tile shape the planner can pick (one or two CTAs per SM, 8..20 consumer
    warps) reproduces the reference's config-1 bits, and the general (tilted-matrix)
    path its config-2 bits: the tile shape never changes a voxel's addition chain."""
    import os
    import subprocess
    import sys

    ref = big_sha()
    if ref is None:
        pytest.skip("big_sha.json not generated")
    here = GOLDEN.parent
    cases = ["cfg1"] + (["cfg2"] if tile_cfg in (0, 1) and (GOLDEN / "cfg2_mats.npy").exists() else [])
    for case in cases:
        env = dict(os.environ, CBP_TILE_CFG=str(tile_cfg))
        out = subprocess.run([sys.executable, str(here / "tile_case.py"), case], env=env, capture_output=True,
                             text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        digest = out.stdout.split()[0]
        want = ref["cfg1_uniform11" if case == "cfg1" else "cfg2_uniform12"]["baseline"]
        assert digest == want, (case, tile_cfg, out.stdout)


@pytest.mark.parametrize("jitter", [False, True])
@pytest.mark.parametrize("path", ["tiled", "tiled_check"])
def test_awkward_medium_sizes_bitwise(torch_cuda, jitter, path):
    """Partial tiles in x, y and z (100 x 70 x 45 volume), a non-square detector whose
    u pitch is not a multiple of 4, a volume that overhangs the detector (guarded loops,
    skipped and never-queued (tile, angle) pairs), 97 angles; fast path (circular) and
    general path (jittered matrices): GPU == C oracle, full volume, random start volume."""
    from paper_2104_13248_b200 import geometry as G

    geom = G.build_geometry(nx=100, ny=70, nz=45, nw=151, nh=130, np=97, d=400.0, D=700.0, pixel_pitch_u=1.1,
                            pixel_pitch_v=0.9, voxel_size=1.3)
    mats = G.jittered_matrices(geom, 2.0, 5) if jitter else G.u_offset(G.projection_matrices(geom), 7.0)
    img = uniform(97, 130, 151, 21)
    vol0 = np.random.default_rng(22).uniform(-1, 1, size=(45, 70, 100)).astype(np.float32)
    out, stats = run_device(torch_cuda, img, mats, vol0, KernelVariant.BASELINE, Layout.NATURAL, Layout.NATURAL,
                            FLAG_SETS[path])
    ref = vol0.copy()
    oracle.baseline(img, mats, ref)
    assert out.tobytes() == ref.tobytes()
    assert stats["smem_pairs"] > 0


@pytest.mark.parametrize("nh,nw", [(1, 16), (16, 1), (1, 1)])
def test_degenerate_detector_samples_nothing(torch_cuda, nh, nw):
    """A 1-pixel-high or -wide detector is legal in the reference (sizes >= 1,
    tensors.py:44-58) and samples nothing (guard x < nw-1, y < nh-1, _kernels.py:52):
    every entry point leaves the volume bitwise unchanged."""
    t = load_golden("tiny")
    n_proj = t["mats"].shape[0]
    start = np.random.default_rng(3).normal(size=(12, 12, 12)).astype(np.float32)
    img = np.ones((n_proj, nh, nw), np.float32)
    v = Volume.from_array(start.copy())
    backproject_baseline(ProjectionStack.from_array(img), t["mats"], v)
    assert v.data.tobytes() == start.tobytes()
    out, _ = run_device(torch_cuda, img, t["mats"], start, KernelVariant.BASELINE, Layout.NATURAL, Layout.NATURAL, 0)
    assert out.tobytes() == start.tobytes()
