"""Generate golden vectors from the LIVE reference package (run in the build container).

    python tests/golden/make_golden.py [--big]

Imports ``conebp`` from /root/reference/pkg/src (read-only; numba's cache is
redirected to a temp dir), runs its back-projection entry points on seeded
inputs and writes the results under tests/golden/:

* small cases (``*.npz``): inputs, matrices, start volume, the reference output
  of ``backproject_baseline`` and of every optimized rung (TRANSPOSED, given
  nb), and the instrumented twin's OpCounters (count=True);
* ``cfg0.npz``: BASELINE config 0 (64^3, 90 x 128^2, uniform seed 0) -- the
  full reference output volume plus the sha256 of the regenerated input;
* ``--big`` adds ``big_sha.json``: sha256 digests of the reference outputs at
  full BASELINE config 1 and config-2 sizes (inputs regenerated from seeds; the
  jittered config-2 matrices are stored in ``cfg2_mats.npy``).

The product code never reads /root/reference; tests only read these fixtures.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_ref_"))
os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import conebp  # noqa: E402  (the live reference)
from conebp import (  # noqa: E402
    KernelVariant,
    Layout,
    ProjectionStack,
    Volume,
    backproject_baseline,
    backproject_optimized,
    build_geometry,
    make_dataset,
    projection_matrices,
    transpose_projections,
    transpose_volume,
)

RUNGS = [KernelVariant.TRANSPOSE, KernelVariant.SHARE, KernelVariant.SYMMETRY, KernelVariant.SUBLINE,
         KernelVariant.SUBLINE_PREFETCH]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def uniform(n_proj, nh, nw, seed):
    rng = np.random.default_rng(seed)
    out = np.empty((n_proj, nh, nw), np.float32)
    for s in range(n_proj):
        out[s] = rng.uniform(-1.0, 1.0, size=(nh, nw))
    return out


def run_case(name, img, mats, vol0, nb, counters=True, rungs=True):
    """Reference outputs for one case; img NATURAL (np, nh, nw), vol0 NATURAL (nz, ny, nx)."""
    n_proj, nh, nw = img.shape
    nz, ny, nx = vol0.shape
    proj = ProjectionStack(img.copy(), n_proj, nh, nw)
    out = {"img": img, "mats": mats, "vol0": vol0, "nb": np.int64(nb)}
    vol = Volume(vol0.copy(), nx, ny, nz)
    backproject_baseline(proj, mats, vol)
    out["baseline"] = vol.data.copy()
    if counters:
        _, c = backproject_baseline(proj, mats, Volume(vol0.copy(), nx, ny, nz), count=True)
        out["count_baseline"] = np.array([c.dot_ops, c.vol_word_accesses, c.proj_word_accesses, c.interp_ops,
                                          c.subline_builds], np.int64)
    if rungs:
        img_t = transpose_projections(proj)
        vol0_t = np.ascontiguousarray(vol0.transpose(2, 1, 0))
        for v in RUNGS:
            if v.uses_symmetry and nz % 2:
                continue
            vt = Volume(vol0_t.copy(), nx, ny, nz, Layout.TRANSPOSED)
            backproject_optimized(img_t, mats, vt, v, batch=nb)
            out[v.name.lower()] = vt.data.copy()
            if counters:
                _, c = backproject_optimized(img_t, mats, Volume(vol0_t.copy(), nx, ny, nz, Layout.TRANSPOSED), v,
                                             batch=nb, count=True)
                out["count_" + v.name.lower()] = np.array(
                    [c.dot_ops, c.vol_word_accesses, c.proj_word_accesses, c.interp_ops, c.subline_builds], np.int64)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: {sorted(out)}", flush=True)


def small_cases():
    # conftest `tiny` fixture (pkg/tests/conftest.py:32-43): phantom data, all in bounds
    geom = build_geometry(nx=12, ny=12, nz=12, nw=24, nh=24, np=8)
    _, proj, mats = make_dataset(geom)
    run_case("tiny", proj.data, mats, np.zeros((12, 12, 12), np.float32), nb=2)

    # guard-firing perturbation of test_backprojector.py:61-77
    m2 = mats.copy()
    m2[:, 0, 3] += np.float32(0.4 * geom.nw * geom.d)
    m2[:, 1, 3] += np.float32(0.3 * geom.nh * geom.d)
    run_case("tiny_guard", proj.data, m2, np.zeros((12, 12, 12), np.float32), nb=2)

    # constant-image KAT (test_backprojector.py:101-109)
    g9 = build_geometry(nx=9, ny=9, nz=9, nw=32, nh=32, np=1)
    run_case("const_kat", np.full((1, 32, 32), 0.75, np.float32), projection_matrices(g9),
             np.zeros((9, 9, 9), np.float32), nb=1)

    # ragged dims, non-zero start volume, partially off-detector (scanner distances)
    rng = np.random.default_rng(5)
    gr = build_geometry(nx=13, ny=7, nz=6, nw=17, nh=11, np=6, d=40.0, D=60.0, pixel_pitch_u=1.6,
                        pixel_pitch_v=1.9, voxel_size=1.0)
    run_case("ragged", uniform(6, 11, 17, 11), projection_matrices(gr),
             rng.normal(size=(6, 7, 13)).astype(np.float32), nb=3)

    # tilted / jittered matrices: non-zero k coefficients in the u and depth rows
    from paper_2104_13248_b200 import geometry as G

    gt = G.build_geometry(nx=20, ny=18, nz=16, nw=40, nh=36, np=12, d=60.0, D=96.0, pixel_pitch_u=1.0,
                        pixel_pitch_v=1.0, voxel_size=1.0)
    mt = G.jittered_matrices(gt, sigma=2.0, seed=9)
    assert (mt[:, 2, 2] != 0).any() and (mt[:, 0, 2] != 0).any()
    run_case("tilted", uniform(12, 36, 40, 13), mt, np.zeros((16, 18, 20), np.float32), nb=4)

    # u principal-point offset (config 4 style) on a small grid; rows partly off detector
    from paper_2104_13248_b200.geometry import u_offset

    go = build_geometry(nx=32, ny=32, nz=32, nw=48, nh=40, np=16, d=100.0, D=150.0, pixel_pitch_u=1.0,
                        pixel_pitch_v=1.0, voxel_size=1.0)
    run_case("uoffset", uniform(16, 40, 48, 14), u_offset(projection_matrices(go), 16.0),
             np.zeros((32, 32, 32), np.float32), nb=8)

    # config 0 (BASELINE.json configs[0]) -- outputs only; inputs regenerated from the seed
    g0 = build_geometry(nx=64, ny=64, nz=64, nw=128, nh=128, np=90, d=1000.0, D=1500.0, pixel_pitch_u=1.0,
                        pixel_pitch_v=1.0, voxel_size=0.5)
    img0 = uniform(90, 128, 128, 0)
    mats0 = projection_matrices(g0)
    proj0 = ProjectionStack(img0, 90, 128, 128)
    vol = Volume.zeros(64, 64, 64)
    backproject_baseline(proj0, mats0, vol)
    digests = {}
    img_t = transpose_projections(proj0)
    for v in RUNGS:
        vt = Volume.zeros(64, 64, 64, Layout.TRANSPOSED)
        backproject_optimized(img_t, mats0, vt, v, batch=30)
        digests[v.name.lower()] = sha(vt.data)
    np.savez_compressed(HERE / "cfg0.npz", mats=mats0, baseline=vol.data, input_sha=np.bytes_(sha(img0)),
                        rung_sha=np.bytes_(json.dumps(digests)))
    print("cfg0 done", flush=True)


def forward_cases():
    """Reference rasterize_phantom + forward_project (phantom.py:90-252) outputs."""
    from conebp import EllipsoidPhantom, Ellipsoid, default_phantom, forward_project, rasterize_phantom

    out = {}
    g1 = build_geometry(nx=12, ny=12, nz=12, nw=24, nh=24, np=8)
    truth = rasterize_phantom(default_phantom(12, 12, 12, g1.voxel_size), (12, 12, 12), g1.voxel_size)
    out["tiny_truth"] = truth.data
    out["tiny_proj"] = forward_project(truth, g1).data
    g2 = build_geometry(nx=16, ny=14, nz=10, nw=40, nh=28, np=7, d=30.0, D=45.0, voxel_size=1.0,
                        angles=[0.0, 0.3, 1.0, 1.5707963267948966, 2.2, 3.141592653589793, 4.0])
    ph = EllipsoidPhantom((Ellipsoid((1.0, -1.0, 0.5), (2.5, 1.6, 2.0), 0.8, 0.4),
                           Ellipsoid((-1.2, 0.8, -0.5), (1.2, 1.8, 1.4), 0.5, -0.7)))
    t2 = rasterize_phantom(ph, (16, 14, 10), 1.0)
    out["odd_truth"] = t2.data
    out["odd_proj"] = forward_project(t2, g2).data
    # voxel sizes other than 1: a power of two (the projector multiplies by the exact reciprocal)
    # and 0.7 (it divides, like the reference)
    for tag, vs in (("half", 0.5), ("p7", 0.7)):
        g3 = build_geometry(nx=10, ny=12, nz=9, nw=30, nh=22, np=5, d=20.0, D=33.0, voxel_size=vs,
                            pixel_pitch_u=0.6, pixel_pitch_v=0.55)
        rng = np.random.default_rng(17)
        from conebp import Volume
        t3 = Volume.from_array(rng.uniform(0.0, 1.0, (9, 12, 10)).astype(np.float32))
        out[f"{tag}_truth"] = t3.data
        out[f"{tag}_proj"] = forward_project(t3, g3).data
    np.savez_compressed(HERE / "forward.npz", **out)
    print("forward:", sorted(out), flush=True)


def big_cases():
    res = {}
    t0 = time.time()
    # config 1 size, uniform inputs (seed 11) -- baseline and every rung at nb=30
    g1 = build_geometry(nx=256, ny=256, nz=256, nw=512, nh=512, np=360, d=750.0, D=1200.0, pixel_pitch_u=0.8,
                        pixel_pitch_v=0.8, voxel_size=1.0)
    img1 = uniform(360, 512, 512, 11)
    m1 = projection_matrices(g1)
    p1 = ProjectionStack(img1, 360, 512, 512)
    v = Volume.zeros(256, 256, 256)
    backproject_baseline(p1, m1, v)
    res["cfg1_uniform11"] = {"input_sha": sha(img1), "mats_sha": sha(m1), "baseline": sha(v.data)}
    del v
    img_t = transpose_projections(p1)
    for rv in RUNGS:
        vt = Volume.zeros(256, 256, 256, Layout.TRANSPOSED)
        backproject_optimized(img_t, m1, vt, rv, batch=30)
        res["cfg1_uniform11"][rv.name.lower()] = sha(vt.data)
        print(f"cfg1 {rv.name} {time.time() - t0:.0f}s", flush=True)
    del img_t, p1, img1
    # config 2 geometry with the jittered matrices, uniform inputs (seed 12), baseline only
    import math

    from paper_2104_13248_b200 import geometry as G

    g2 = G.build_geometry(nx=512, ny=512, nz=512, nw=1248, nh=960, np=496, d=750.0, D=1200.0, pixel_pitch_u=0.32,
                        pixel_pitch_v=0.32, voxel_size=0.5,
                        angles=[math.radians(200.0) * s / 496 for s in range(496)])
    m2 = G.jittered_matrices(g2, 0.5, 2)
    np.save(HERE / "cfg2_mats.npy", m2)
    img2 = uniform(496, 960, 1248, 12)
    v = Volume.zeros(512, 512, 512)
    backproject_baseline(ProjectionStack(img2, 496, 960, 1248), m2, v)
    res["cfg2_uniform12"] = {"input_sha": sha(img2), "mats_sha": sha(m2), "baseline": sha(v.data),
                             "abs_sum": float(np.abs(v.data, dtype=np.float64).sum())}
    print(f"cfg2 done {time.time() - t0:.0f}s", flush=True)
    (HERE / "big_sha.json").write_text(json.dumps(res, indent=2) + "\n")


if __name__ == "__main__":
    print("reference conebp", conebp.__version__, "from", conebp.__file__)
    small_cases()
    forward_cases()
    if "--big" in sys.argv:
        big_cases()
