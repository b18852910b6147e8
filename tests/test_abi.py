"""The C-ABI library: builds for sm_100a, loads, exports every declared symbol.

No compute calls (this container has no GPU); the host-only planners are
exercised in test_slabs.py.
"""

import re
import subprocess
from pathlib import Path

import pytest

from paper_2104_13248_b200 import _lib

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "conebp_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(cbp_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for name in ("cbp_backproject_f32", "cbp_backproject_staged", "cbp_stage_projections", "cbp_slab_plan",
                 "cbp_count_ops", "cbp_last_error", "cbp_version"):
        assert name in syms
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with include/conebp_b200.h"


def test_library_loads_and_exports_every_symbol():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.cbp_version() >= 100
    assert isinstance(L.cbp_last_error(), bytes)


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_device_entry_points_fail_loudly_without_gpu():
    L = _lib.lib()
    if L.cbp_device_count() > 0:
        pytest.skip("a GPU is visible")
    import numpy as np

    mats = np.zeros((1, 3, 4), np.float32)
    mats[0, 2, 3] = 1.0
    img = np.zeros((1, 4, 4), np.float32)
    vol = np.zeros((2, 2, 2), np.float32)
    rc = L.cbp_backproject_host_f32(_lib.f32ptr(img), 1, 4, 4, 0, _lib.f32ptr(mats), _lib.f32ptr(vol), 2, 2, 2, 0,
                                    0, 0)
    assert rc == _lib.CBP_ENODEV
    assert b"no CUDA device" in L.cbp_last_error()


def test_no_fma_contraction_in_backprojection_sass():
    """Bit-exactness needs separately rounded products and sums: the SASS of the
    back-projection kernels must contain no fused multiply-add on sample values.  The only
    FFMA2 allowed are the texel ADDRESSES of the guard-free loops (floor * pitch + base on
    subnormal floats, exact by construction: bp_kernels.cuh hot_loop / gen_loop): one per slice
    pair on the fast path (multiplier and addend broadcast scalars), two on the general path
    (fx * 4 + base, then fy * pitch + that), every multiplier a broadcast scalar.  A contraction
    of the sample arithmetic would add several FFMA2 per slice pair (ten mul+add pairs in the
    blend), so the COUNT per kernel is checked as well.  (Scalar FFMA are the explicit Newton
    steps of the correctly rounded reciprocal.)"""
    out = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    funcs = re.split(r"\n\s+Function : ", out.stdout)
    reg = r"R\d+(\.reuse)?"
    mult = rf"(U?{reg}\.F32|5\.605\d+e-45)"  # broadcast row pitch, or the immediate 4 * 2^-149 (x step in bytes)
    addr_fma = re.compile(rf"FFMA2 R\d+, {reg}\.F32x2\.LO_HI, {mult}, {reg}\.F32(x2\.(LO_HI|HI_LO))? ;")
    fast_form = re.compile(rf"FFMA2 R\d+, {reg}\.F32x2\.LO_HI, {mult}, {reg}\.F32 ;")
    checked = with_addr = 0
    for f in funcs:
        name = f.split("\n", 1)[0]
        if "bp_tiled_kernel" in name or "bp_naive_kernel" in name or "bp_tiled_half_kernel" in name:
            checked += 1
            fused = [ln for ln in f.split("\n") if "FFMA2" in ln]
            assert all(addr_fma.search(ln) for ln in fused), (name, [ln for ln in fused if not addr_fma.search(ln)][:3])
            # 16 slice pairs per guard-free loop (8 in the half z-run kernels), one address FMA per
            # pair on the fast path, two on the general path
            assert len(fused) in (0, 8, 16, 32), (name, len(fused))
            # at least half of them have the fast path's all-broadcast form (the general path's
            # second FMA adds the packed result of its first)
            assert 2 * sum(bool(fast_form.search(ln)) for ln in fused) >= len(fused), name
            with_addr += bool(fused)
        if "bp_tiled_fmalerp_kernel" in name:  # the opt-in tolerance mode does fuse its lerps
            assert "FFMA2" in f, name
    assert with_addr > 0
    assert checked > 0
