"""z-slab planning (host functions of libconebp_b200.so, no GPU needed).

Each slab's detector-row band must contain every row its voxels sample: a
slab back-projected by the CPU oracle from its band alone reproduces the
full-volume reference result bit for bit, with no band violation.
"""

import numpy as np
import pytest

import oracle
from conftest import load_golden
from paper_2104_13248_b200 import geometry as G


@pytest.mark.parametrize("case", ["uoffset", "tiny", "tilted", "ragged"])
@pytest.mark.parametrize("n_ranks", [1, 2, 3, 4])
def test_slab_bands_cover_sampled_rows(case, n_ranks):
    g = load_golden(case)
    img, mats, full = g["img"], g["mats"], g["baseline"]
    n_proj, nh, nw = img.shape
    nz, ny, nx = full.shape
    kb, bands = G.slab_plan(mats, nh, nw, nx, ny, nz, n_ranks, align=2)
    assert kb[0] == 0 and kb[-1] == nz and all(a <= b for a, b in zip(kb, kb[1:]))
    for r in range(n_ranks):
        k0, k1 = kb[r], kb[r + 1]
        if k1 == k0:
            continue
        v0, rows = bands[r]
        assert (v0, rows) == G.slab_band(mats, nh, nw, nx, ny, nz, k0, k1)
        vol = g["vol0"][k0:k1].copy()
        if rows == 0:  # nothing sampled: the slab must be unchanged in the reference too
            assert full[k0:k1].tobytes() == vol.tobytes()
            continue
        assert 0 <= v0 and v0 + rows <= nh
        viol = oracle.baseline(img[:, v0:v0 + rows], mats, vol, nh=nh, v0=v0, k_lo=k0)
        assert viol == 0
        assert vol.tobytes() == full[k0:k1].tobytes()


def test_cost_balanced_slabs_on_truncated_fov():
    # config-4 geometry scaled down 8x: most of the volume top and bottom is never sampled
    geom = G.build_geometry(nx=256, ny=256, nz=256, nw=256, nh=256, np=64, d=1000.0, D=1500.0, pixel_pitch_u=0.8,
                            pixel_pitch_v=0.8, voxel_size=1.0)
    mats = G.u_offset(G.projection_matrices(geom), 2.0)
    kb, bands = G.slab_plan(mats, 256, 256, 256, 256, 256, 8, align=8)
    widths = np.diff(kb)
    assert widths.sum() == 256
    # equal slabs would give the outer ranks almost nothing; balanced ones are narrower in the middle
    assert widths[0] > widths[3] and widths[-1] > widths[4]
    rows = [b[1] for b in bands]
    assert sum(rows) < 2 * 256


def test_slab_band_rejects_bad_ranges():
    g = load_golden("tiny")
    with pytest.raises(ValueError):
        G.slab_band(g["mats"], 24, 24, 12, 12, 12, 5, 5)
    with pytest.raises(ValueError):
        G.slab_band(g["mats"], 24, 24, 12, 12, 12, 0, 13)
