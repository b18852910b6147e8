"""Drop-in API contract on the CPU: validation order and messages of
pkg/src/conebp/backprojector.py (checked before any device work), the
closed-form counters and the variant enum (mirrors pkg/tests/
test_backprojector.py:210-238 and test_counters.py)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2104_13248_b200 import (
    BatchConfig,
    KernelVariant,
    Layout,
    ProjectionStack,
    Volume,
    backproject_baseline,
    backproject_optimized,
    build_geometry,
    count_ops,
    dot_reduction_ratio,
    asymptotic_dot_reduction_ratio,
    projection_matrices,
    transpose_projections,
)


@pytest.fixture(scope="module")
def tiny():
    g = load_golden("tiny")
    proj = ProjectionStack.from_array(g["img"])
    return proj, transpose_projections(proj), g["mats"]


def test_error_paths(tiny):
    proj, img_t, mats = tiny
    vol_t = Volume.zeros(12, 12, 12, Layout.TRANSPOSED)
    vol_n = Volume.zeros(12, 12, 12)
    with pytest.raises(ValueError, match="nb must divide np"):
        backproject_optimized(img_t, mats, vol_t, KernelVariant.SUBLINE, batch=3)
    for nb in (0, 33):
        with pytest.raises(ValueError, match="batch size"):
            BatchConfig(nb)
    with pytest.raises(ValueError, match="TRANSPOSED"):
        backproject_optimized(proj, mats, vol_t, KernelVariant.SUBLINE, batch=1)
    with pytest.raises(ValueError, match="NATURAL"):
        backproject_baseline(img_t, mats, vol_n)
    with pytest.raises(ValueError, match="BASELINE"):
        backproject_optimized(img_t, mats, vol_t, KernelVariant.BASELINE)
    with pytest.raises(ValueError, match=r"expected \(8, 3, 4\) matrices"):
        backproject_baseline(proj, mats[:3], vol_n)
    bad = mats.copy()
    bad[0, 0, 0] = np.nan
    with pytest.raises(ValueError, match="finite"):
        backproject_baseline(proj, bad, vol_n)
    with pytest.raises(ValueError, match="worker count"):
        backproject_baseline(proj, mats, vol_n, threads=0)
    geom_odd = build_geometry(nx=8, ny=8, nz=9, nw=24, nh=24, np=4)
    img_odd = transpose_projections(ProjectionStack.zeros(4, 24, 24))
    with pytest.raises(ValueError, match="even nz"):
        backproject_optimized(img_odd, projection_matrices(geom_odd), Volume.zeros(8, 8, 9, Layout.TRANSPOSED),
                              KernelVariant.SYMMETRY, batch=1)


def test_validation_order_layout_before_mats(tiny):
    proj, img_t, mats = tiny
    # layout is checked first (backprojector.py:150-151 before :152)
    with pytest.raises(ValueError, match="NATURAL"):
        backproject_baseline(img_t, mats[:2], Volume.zeros(12, 12, 12))
    # nb before nz parity before matrices (backprojector.py:187-190)
    with pytest.raises(ValueError, match="nb must divide"):
        backproject_optimized(img_t, mats[:2], Volume.zeros(12, 12, 11, Layout.TRANSPOSED), KernelVariant.SYMMETRY,
                              batch=3)


def test_variant_parse_and_flags():
    assert KernelVariant.parse("subline_prefetch") is KernelVariant.SUBLINE_PREFETCH
    assert KernelVariant.parse(" Baseline ") is KernelVariant.BASELINE
    with pytest.raises(ValueError, match="unknown kernel variant"):
        KernelVariant.parse("turbo")
    assert not KernelVariant.BASELINE.uses_transposed_layout
    assert KernelVariant.SYMMETRY.uses_symmetry and not KernelVariant.SHARE.uses_symmetry
    assert KernelVariant.SUBLINE.uses_subline and not KernelVariant.SYMMETRY.uses_subline


def test_closed_form_counters_match_twin_on_in_bounds_problem():
    # `tiny` lands entirely on the detector: the twin's tallies equal the closed forms
    g = load_golden("tiny")
    names = ["baseline", "transpose", "share", "symmetry", "subline", "subline_prefetch"]
    for v, name in zip(KernelVariant, names):
        c = count_ops(v, 12, 12, 12, 8, nb=2, nh=24)
        twin = g["count_" + name]
        assert [c.dot_ops, c.vol_word_accesses, c.proj_word_accesses, c.interp_ops, c.subline_builds] == \
            twin.tolist(), name


def test_counter_errors_and_ratios():
    with pytest.raises(ValueError):
        count_ops(KernelVariant.SUBLINE, 8, 8, 8, 8, nb=2)
    with pytest.raises(ValueError):
        count_ops(KernelVariant.SYMMETRY, 8, 8, 7, 8, nb=2)
    with pytest.raises(ValueError):
        count_ops(KernelVariant.SHARE, 8, 8, 8, 8, nb=3)
    assert count_ops(KernelVariant.BASELINE, 64, 64, 64, 64).dot_ops == 3 * 64 ** 4
    assert dot_reduction_ratio(256) == pytest.approx(1 - 130 / 768)
    assert asymptotic_dot_reduction_ratio(1 << 20) == pytest.approx(5 / 6, rel=1e-5)


def test_fdk_rejects_short_scans():
    """fdk_reconstruct's pi*d^2/np scale is only right for a full, evenly sampled orbit."""
    import math

    from paper_2104_13248_b200 import geometry as G
    from paper_2104_13248_b200.fdk import check_full_orbit

    full = G.build_geometry(nx=8, ny=8, nz=8, nw=16, nh=16, np=12)
    check_full_orbit(full)
    short = G.build_geometry(nx=8, ny=8, nz=8, nw=16, nh=16, np=12,
                             angles=[s * math.radians(200.0) / 12 for s in range(12)])
    with pytest.raises(ValueError, match="360"):
        check_full_orbit(short)
