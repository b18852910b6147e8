"""Shared test setup.

Markers: ``gpu`` tests need a CUDA device and the built libconebp_b200.so (run
with ``-m gpu`` on a B200); everything else runs on the CPU.  Golden vectors
under tests/golden/ were produced by the live reference (make_golden.py);
nothing here reads /root/reference.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
for p in (str(REPO), str(REPO / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

SMALL_CASES = ["tiny", "tiny_guard", "const_kat", "ragged", "tilted", "uoffset"]
RUNG_NAMES = ["transpose", "share", "symmetry", "subline", "subline_prefetch"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built sm_100a library")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


def uniform(n_proj, nh, nw, seed):
    rng = np.random.default_rng(seed)
    out = np.empty((n_proj, nh, nw), np.float32)
    for s in range(n_proj):
        out[s] = rng.uniform(-1.0, 1.0, size=(nh, nw))
    return out
