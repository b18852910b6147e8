# fused FDK filter + forward projector fast path: tests and timings
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fdk.py tests/test_phantom.py tests/test_cli.py -q -m gpu > gpurun_out/pytest_f1f2.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_f1f2.log
timeout 900 python tools/time_f1_f2.py --configs 1 3 > gpurun_out/f1f2.log 2>&1; echo "f1f2 rc=$?"; tail -1 gpurun_out/f1f2.log
