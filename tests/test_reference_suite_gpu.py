"""Drop-in proof: the reference package's OWN tests pass with its kernel seam served by the
GPU library (paper_2104_13248_b200.seam; tools/run_reference_tests.py).

Needs the reference installed into baseline/_ref and its tests copied to baseline/_ref_tests
(tools/install_reference.sh, git-ignored; skipped when absent).  The numba kernels are never
called: the runner asserts the seam took every back-projection call.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


def test_reference_suite_through_the_gpu_seam():
    if not (REPO / "baseline" / "_ref_tests").is_dir() or not (REPO / "baseline" / "_ref" / "conebp").is_dir():
        pytest.skip("reference install not present (tools/install_reference.sh)")
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, str(REPO / "tools" / "run_reference_tests.py")], capture_output=True,
                       text=True, timeout=1800, cwd=REPO)
    summary = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert summary["passed"] >= 40 and not summary["failed"]
    assert summary["seam_calls"]["baseline"] > 0 and summary["seam_calls"]["subline_prefetch"] > 0
