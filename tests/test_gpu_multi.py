"""GPU parity of the paths the product runs beyond one whole-volume launch.

* the chunked host pipeline (``cbp_backproject_host_f32``: angle-range launches with
  s_begin > 0, the path bench.py's e2e leg times) at config-1 size;
* the multi-rank z-slab driver with the REAL CudaBackend on one GPU (loopback harness,
  tests/loopback.py): banded copies (v0 > 0), angle-window launches on double buffers,
  slabs with k0 > 0 and nz_total > nz, both band transports, N = 2, 4, 8;
* the single-process multi-device entry point ``cbp_backproject_multi`` (every rank on
  device 0), including the config-4 volume at N = 8 against a single launch and the oracle;
* CUDA IPC between two processes sharing one GPU (the one-process-per-GPU transport);
* the exhaustive check of the branch-free reciprocal ``rcp_rn_normal``.

Reference anchors: results are bitwise for any chunking and any worker count
(/root/reference/pkg/src/conebp/_kernels.py:3-10), one writer per voxel (:12-14),
ascending-s accumulation (:38,61).
"""

import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, load_golden, uniform
from paper_2104_13248_b200 import KernelVariant, ProjectionStack, Volume, backproject_baseline
from paper_2104_13248_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert _lib.lib().cbp_device_count() > 0
    return torch


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def cfg1(torch_cuda):
    from paper_2104_13248_b200 import configs

    ref = json.loads((GOLDEN / "big_sha.json").read_text())["cfg1_uniform11"]
    spec = configs.get_config(1)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    assert sha(mats) == ref["mats_sha"]
    img = uniform(360, 512, 512, 11)
    assert sha(img) == ref["input_sha"]
    return geom, mats, img, ref


# ------------------------------------------------------------------ host pipeline
@pytest.mark.parametrize("chunks,slabs", [(1, 1), (7, 1), (22, 1), (7, 3), (5, 8)])
def test_host_path_angle_chunks_bitwise(cfg1, chunks, slabs, monkeypatch):
    """Angle-chunked uploads with s_begin > 0 launches, and z-slab pipelining (slab k+1
    uploads / slab k-1 downloads while slab k computes; slabs with k0 > 0, nz_total > nz)."""
    geom, mats, img, ref = cfg1
    monkeypatch.setenv("CBP_HOST_CHUNKS", str(chunks))
    monkeypatch.setenv("CBP_HOST_SLABS", str(slabs))
    vol = Volume.zeros(256, 256, 256)
    backproject_baseline(ProjectionStack.from_array(img), mats, vol)
    assert sha(vol.data) == ref["baseline"]


def test_host_path_pageable_and_transposed(torch_cuda):
    """TRANSPOSED projections through the host pipeline (staged per chunk), odd pitch."""
    from paper_2104_13248_b200 import backproject, transpose_projections

    g = load_golden("uoffset")
    nz, ny, nx = g["vol0"].shape
    os.environ["CBP_HOST_CHUNKS"] = "5"
    try:
        img_t = transpose_projections(ProjectionStack.from_array(g["img"]))
        vt = Volume(np.ascontiguousarray(g["vol0"].transpose(2, 1, 0)), nx, ny, nz, img_t.layout)
        backproject(img_t, g["mats"], vt, KernelVariant.TRANSPOSE, batch=int(g["nb"]))
        assert vt.data.tobytes() == g["transpose"].tobytes()
    finally:
        del os.environ["CBP_HOST_CHUNKS"]


# ------------------------------------------------------------------ z-slab driver, loopback
@pytest.mark.parametrize("transport", ["p2p", "ipc"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_loopback_slabs_cfg1_bitwise(torch_cuda, cfg1, world, transport):
    from loopback import run_loopback
    from paper_2104_13248_b200 import slabs

    torch = torch_cuda
    geom, mats, img, ref = cfg1
    # 16-slice boundaries where the planner allows, and odd chunk counts: every launch an angle window
    plan = slabs.plan_slabs(mats, geom.nh, geom.nw, 256, 256, 256, world, align=16)
    assert any(v0 > 0 for v0, rows in plan.bands if rows), "expected at least one banded rank"
    img_dev = torch.from_numpy(img).cuda()
    vols, dist = run_loopback(torch, img_dev, mats, plan, n_chunks=5, transport=transport)
    full = torch.cat([v for v in vols if v.shape[0] > 0]).cpu().numpy()
    assert sha(full) == ref["baseline"], (world, transport, plan.k_bounds, plan.bands)
    if transport == "p2p":  # only bands travel: far less than the whole stack per rank
        assert dist.sent_bytes < (world - 1) * img.nbytes


def test_loopback_slabs_symmetry_rung_bitwise(torch_cuda, cfg1):
    """The mirror rung (global-k mirroring at nz_total/2) across slab boundaries."""
    from loopback import run_loopback
    from paper_2104_13248_b200 import slabs

    torch = torch_cuda
    geom, mats, img, ref = cfg1
    plan = slabs.plan_slabs(mats, geom.nh, geom.nw, 256, 256, 256, 4, align=16, variant=int(KernelVariant.SYMMETRY))
    vols, _ = run_loopback(torch, torch.from_numpy(img).cuda(), mats, plan, n_chunks=3, transport="ipc")
    full = torch.cat([v for v in vols if v.shape[0] > 0]).cpu().numpy()  # [z][y][x]
    assert sha(full.transpose(2, 1, 0)) == ref["symmetry"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_backproject_multi_cfg1_bitwise(torch_cuda, cfg1, world):
    from paper_2104_13248_b200 import device as D, slabs

    torch = torch_cuda
    geom, mats, img, ref = cfg1
    plan = slabs.plan_slabs(mats, geom.nh, geom.nw, 256, 256, 256, world, align=16)
    img_dev = torch.from_numpy(img).cuda()
    slab_t = [torch.zeros((plan.k_bounds[r + 1] - plan.k_bounds[r], 256, 256), device="cuda") for r in range(world)]
    stats = D.backproject_multi(img_dev, mats, slab_t, plan.k_bounds, 256, 256, 256, devices=[0] * world,
                                n_chunks=7)
    assert stats["band_violations"] == 0 and stats["smem_pairs"] > 0
    full = torch.cat([t for t in slab_t if t.shape[0] > 0]).cpu().numpy()
    assert sha(full) == ref["baseline"]


def test_backproject_multi_cfg4_n8(torch_cuda):
    """Config 4 (2048^3 <- 2048 x 2048^2, +16 px u offset) as 8 z-slab ranks on one GPU:
    every slab equals the single-launch volume bit for bit, and the slices on both sides
    of every slab boundary equal the C oracle (global indices, from the band only)."""
    from paper_2104_13248_b200 import configs, geometry as G
    from paper_2104_13248_b200 import device as D, slabs

    torch = torch_cuda
    spec = configs.get_config(4)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    n = geom.nx
    img = torch.rand((geom.np, geom.nh, geom.nw), device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    img.mul_(2).sub_(1)
    plan = slabs.plan_slabs(mats, geom.nh, geom.nw, n, n, n, 8, align=16)
    ref_vol = torch.zeros((n, n, n), device="cuda")
    D.backproject_device(img, mats, ref_vol, geom.np, geom.nh, geom.nw, n, n, n)
    D.sync_status()
    # the whole 8-rank call (slabs are the volume's z-ranges)
    slab_t = [torch.zeros((plan.k_bounds[r + 1] - plan.k_bounds[r], n, n), device="cuda") for r in range(8)]
    stats = D.backproject_multi(img, mats, slab_t, plan.k_bounds, n, n, n, devices=[0] * 8, n_chunks=8)
    assert stats["band_violations"] == 0
    for r in range(8):
        k0, k1 = plan.slab(r)
        assert torch.equal(slab_t[r].view(torch.int32), ref_vol[k0:k1].view(torch.int32)), (r, k0, k1)
    del slab_t
    checked = 0
    bounds = sorted({k for k in plan.k_bounds[1:-1]})
    for kb in bounds:
        for k0, k1 in ((kb - 1, kb), (kb, kb + 1)):
            v0, rows = G.slab_band(mats, geom.nh, geom.nw, n, n, n, k0, k1)
            got = ref_vol[k0:k1].cpu().numpy()
            want = np.zeros((1, n, n), np.float32)
            if rows:
                band = img[:, v0:v0 + rows, :].contiguous().cpu().numpy()
                assert oracle.baseline(band, mats, want, nh=geom.nh, v0=v0, k_lo=k0) == 0
            assert got.tobytes() == want.tobytes(), (k0, k1)
            checked += int(np.count_nonzero(want))
    assert checked > 0


def test_multi_rejects_bad_bounds(torch_cuda):
    from paper_2104_13248_b200 import device as D

    torch = torch_cuda
    g = load_golden("uoffset")
    img = torch.from_numpy(g["img"]).cuda()
    nz, ny, nx = g["vol0"].shape
    slab = torch.zeros((nz, ny, nx), device="cuda")
    with pytest.raises(ValueError):
        D.backproject_multi(img, g["mats"], [slab, None], [0, nz - 1, nz], nx, ny, nz, devices=[0, 0])


# ------------------------------------------------------------------ IPC between processes
def _ipc_worker(rank, port, q):
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    for p in (str(repo), str(repo / "tests"), str(repo / "oracle")):
        sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from conftest import load_golden
    from paper_2104_13248_b200 import slabs

    dist.init_process_group("gloo", rank=rank, world_size=2)  # plumbing only: the bands move by CUDA IPC
    try:
        torch.cuda.set_device(0)
        g = load_golden("uoffset")
        n_proj, nh, nw = g["img"].shape
        nz, ny, nx = g["vol0"].shape
        plan = slabs.plan_slabs(g["mats"], nh, nw, nx, ny, nz, 2, align=4)
        backend = slabs.CudaBackend(torch)
        img = torch.from_numpy(g["img"]).cuda() if rank == 0 else None
        shared = backend.ipc_share(img, dist)
        k0, k1 = plan.slab(rank)
        vol = torch.from_numpy(g["vol0"][k0:k1].copy()).cuda()
        slabs.run_slabs(img, g["mats"], plan, backend, dist, n_chunks=3, vol=vol, transport="ipc", shared=shared)
        dist.barrier()  # rank 0 keeps its buffer alive until every pull is done
        ok = vol.cpu().numpy().tobytes() == g["baseline"][k0:k1].tobytes()
        q.put(("ok", rank, ok, list(plan.k_bounds), list(plan.bands)))
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        q.put(("error", rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_ipc_transport_two_processes_bitwise(torch_cuda):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert not [r for r in res if r[0] == "error"], res
    assert all(r[2] for r in res), res
    assert any(r[4][1][0] > 0 for r in res if r[1] == 0), "rank 1 should hold a band starting below row 0"


# ------------------------------------------------------------------ reciprocal
def test_rcp_rn_normal_is_exact_on_its_whole_range(torch_cuda):
    """rcp_rn_normal == __frcp_rn for every float with 2^-100 <= |z| < 2^100 (3.4e9 values)."""
    from paper_2104_13248_b200 import device as D

    lo, hi = 0x0D800000, 0x71800000  # 2^-100, 2^100
    assert np.uint32(lo).view(np.float32) == np.float32(2.0 ** -100)
    assert np.uint32(hi).view(np.float32) == np.float32(2.0 ** 100)
    for sign in (0, 0x80000000):
        bad, first = D.selftest_rcp(sign | lo, sign | hi)
        assert bad == 0, hex(first)
    # the footprint's admission bounds sit inside the proven range
    assert np.float32(7.9e-31) >= np.float32(2.0 ** -100) and np.float32(1.2e30) < np.float32(2.0 ** 100)


@pytest.mark.parametrize("jitter", [False, True])
def test_half_zrun_tiles_bitwise(torch_cuda, jitter):
    """Slabs of 32m + 16 slices run their last 16 slices as a layer of half z-run tiles
    (bp_tiled_half_kernel); a 16-slice slab runs on it alone.  Fast (circular + u offset)
    and general (jittered) paths, global slice indices, bitwise vs the C oracle."""
    from paper_2104_13248_b200 import device as D, geometry as G

    torch = torch_cuda
    geom = G.build_geometry(nx=100, ny=70, nz=80, nw=151, nh=130, np=61, d=400.0, D=700.0, pixel_pitch_u=1.1,
                            pixel_pitch_v=0.9, voxel_size=1.3)
    mats = G.jittered_matrices(geom, 2.0, 5) if jitter else G.u_offset(G.projection_matrices(geom), 7.0)
    img = uniform(61, 130, 151, 31)
    vol0 = np.random.default_rng(32).uniform(-1, 1, size=(80, 70, 100)).astype(np.float32)
    ref = vol0.copy()
    oracle.baseline(img, mats, ref)
    staged = D.StagedProjections(torch.from_numpy(img).cuda(), 61, 130, 151)
    for k0, k1 in [(0, 48), (48, 64), (64, 80), (16, 64)]:
        v = torch.from_numpy(vol0[k0:k1].copy()).cuda()
        D.backproject_staged(staged, mats, v, 100, 70, k1 - k0, k0=k0, nz_total=80)
        st = D.sync_status()
        assert st["band_violations"] == 0
        assert v.cpu().numpy().tobytes() == ref[k0:k1].tobytes(), (k0, k1, jitter)
    assert D.last_plan()["tile_z"] in (16, 32)
