"""Pin the CPU oracle (oracle/) to golden vectors from the live reference.

Bit-for-bit: the C restatement and the numpy restatement must reproduce the
reference's ``backproject_baseline`` and every optimized rung exactly.
"""

import hashlib
import json

import numpy as np
import pytest

import oracle
from conftest import RUNG_NAMES, SMALL_CASES, load_golden, uniform

RUNG_ID = {"transpose": 1, "share": 2, "symmetry": 3, "subline": 4, "subline_prefetch": 5}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", SMALL_CASES)
def test_c_oracle_baseline_bitwise(case):
    g = load_golden(case)
    vol = g["vol0"].copy()
    viol = oracle.baseline(g["img"], g["mats"], vol, threads=3)
    assert viol == 0
    assert vol.tobytes() == g["baseline"].tobytes()


@pytest.mark.parametrize("case", SMALL_CASES)
def test_numpy_oracle_baseline_bitwise(case):
    g = load_golden(case)
    vol = oracle.numpy_baseline(g["img"], g["mats"], g["vol0"].copy())
    assert vol.tobytes() == g["baseline"].tobytes()


@pytest.mark.parametrize("case", SMALL_CASES)
@pytest.mark.parametrize("rung", RUNG_NAMES)
def test_c_oracle_rungs_bitwise(case, rung):
    g = load_golden(case)
    if rung not in g:
        pytest.skip("rung not applicable (odd nz)")
    img_t = np.ascontiguousarray(g["img"].transpose(0, 2, 1))
    vol_t = np.ascontiguousarray(g["vol0"].transpose(2, 1, 0))
    oracle.rung(RUNG_ID[rung], img_t, g["mats"], vol_t, int(g["nb"]), threads=2)
    assert vol_t.tobytes() == g[rung].tobytes()


def test_cfg0_oracle_bitwise():
    g = load_golden("cfg0")
    img = uniform(90, 128, 128, 0)
    assert sha(img) == g["input_sha"].item().decode(), "seeded input generator drifted"
    vol = np.zeros((64, 64, 64), np.float32)
    oracle.baseline(img, g["mats"], vol)
    assert vol.tobytes() == g["baseline"].tobytes()
    digests = json.loads(g["rung_sha"].item().decode())
    img_t = np.ascontiguousarray(img.transpose(0, 2, 1))
    for rung, digest in digests.items():
        vt = np.zeros((64, 64, 64), np.float32)
        oracle.rung(RUNG_ID[rung], img_t, g["mats"], vt, 30)
        assert sha(vt) == digest, rung


def test_voxel_list_oracle_matches_full_volume():
    g = load_golden("uoffset")
    rng = np.random.default_rng(3)
    nz, ny, nx = g["vol0"].shape
    idx = np.stack([rng.integers(0, nx, 500), rng.integers(0, ny, 500), rng.integers(0, nz, 500)], axis=1)
    vals = oracle.voxels(g["img"], g["mats"], idx)
    ref = g["baseline"][idx[:, 2], idx[:, 1], idx[:, 0]]
    assert vals.tobytes() == ref.tobytes()


def test_oracle_thread_count_determinism():
    g = load_golden("tiny")
    outs = set()
    for t in (1, 2, 5, 8):
        vol = np.zeros_like(g["vol0"])
        oracle.baseline(g["img"], g["mats"], vol, threads=t)
        outs.add(vol.tobytes())
        img_t = np.ascontiguousarray(g["img"].transpose(0, 2, 1))
        vt = np.zeros_like(g["vol0"])
        oracle.rung(5, img_t, g["mats"], vt, 2, threads=t)
        outs.add(("p", vt.tobytes()))
    assert len(outs) == 2
