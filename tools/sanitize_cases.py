"""Small back-projection cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Every case runs through the library's device API and is checked bit for bit against the
C oracle (test infrastructure), so a sanitizer run also proves the kernels still compute
the right thing under instrumentation.  Cases cover the tiled kernel's fast path (guard-free
and guarded loops, TMA ring, skip-free queue), the general path (jittered matrices,
per-voxel 1/z), the CHECK build, the naive kernel, the FMA-lerp tolerance kernel, the
staging kernels (odd detector pitch), angle windows on band buffers and the multi-rank
entry point.  Sizes are small: racecheck slows kernels down by orders of magnitude.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
for p in (str(REPO), str(REPO / "oracle"), str(REPO / "tests")):
    sys.path.insert(0, p)

import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2104_13248_b200 import KernelVariant, Layout, _lib, configs, geometry as G  # noqa: E402
from paper_2104_13248_b200 import device as D  # noqa: E402


def run(img, mats, vol0, flags=0, variant=KernelVariant.BASELINE):
    n_proj, nh, nw = img.shape
    nz, ny, nx = vol0.shape
    ti = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    tv = torch.from_numpy(vol0.copy()).cuda()
    D.backproject_device(ti, mats, tv, n_proj, nh, nw, nx, ny, nz, variant, flags=flags)
    st = D.sync_status()
    assert st["band_violations"] == 0, st
    if flags & _lib.FLAG_CHECK:
        assert st["box_misses"] == 0, st
    return tv.cpu().numpy()


def ref(img, mats, vol0):
    out = vol0.copy()
    oracle.baseline(img, mats, out)
    return out


def medium(jitter: bool):
    geom = G.build_geometry(nx=40, ny=36, nz=34, nw=71, nh=62, np=23, d=300.0, D=520.0, pixel_pitch_u=1.1,
                            pixel_pitch_v=0.9, voxel_size=1.3)
    mats = G.jittered_matrices(geom, 2.0, 5) if jitter else G.u_offset(G.projection_matrices(geom), 5.0)
    rng = np.random.default_rng(3)
    img = rng.uniform(-1, 1, size=(23, 62, 71)).astype(np.float32)
    vol0 = rng.uniform(-1, 1, size=(34, 36, 40)).astype(np.float32)
    return img, mats, vol0


def case_cfg0():
    spec = configs.get_config(0)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    img = spec.projections_host(geom)[:24]
    mats = mats[:24]
    vol0 = np.zeros((64, 64, 64), np.float32)
    assert run(img, mats, vol0).tobytes() == ref(img, mats, vol0).tobytes()


def case_medium_fast():
    img, mats, vol0 = medium(False)
    want = ref(img, mats, vol0)
    for flags in (0, _lib.FLAG_CHECK, _lib.FLAG_NAIVE, _lib.FLAG_NO_SMEM):
        assert run(img, mats, vol0, flags).tobytes() == want.tobytes(), flags


def case_medium_general():
    img, mats, vol0 = medium(True)
    want = ref(img, mats, vol0)
    for flags in (0, _lib.FLAG_CHECK):
        assert run(img, mats, vol0, flags).tobytes() == want.tobytes(), flags


def case_fma_lerp():
    img, mats, vol0 = medium(False)
    out = run(img, mats, vol0, _lib.FLAG_FMA_LERP)
    want = ref(img, mats, vol0)
    d = np.abs(out.astype(np.float64) - want)
    assert d.max() <= 1e-4 * np.abs(want).max()


def case_multi():
    from paper_2104_13248_b200 import slabs

    img, mats, vol0 = medium(False)
    n_proj, nh, nw = img.shape
    nz, ny, nx = vol0.shape
    plan = slabs.plan_slabs(mats, nh, nw, nx, ny, nz, 3, align=4)
    ti = torch.from_numpy(img).cuda()
    parts = [torch.from_numpy(vol0[plan.k_bounds[r]:plan.k_bounds[r + 1]].copy()).cuda() for r in range(3)]
    D.backproject_multi(ti, mats, parts, plan.k_bounds, nx, ny, nz, devices=[0, 0, 0], n_chunks=3)
    out = np.concatenate([p.cpu().numpy() for p in parts])
    assert out.tobytes() == ref(img, mats, vol0).tobytes()


CASES = {"cfg0": case_cfg0, "medium_fast": case_medium_fast, "medium_general": case_medium_general,
         "fma_lerp": case_fma_lerp, "multi": case_multi}


def main(names):
    for name in names or list(CASES):
        CASES[name]()
        print(f"{name}: ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
