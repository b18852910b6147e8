set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_fma_lerp.py tests/test_abi.py -x -q -m gpu > gpurun_out/pytest_fma.log 2>&1; echo "fma rc=$?"; tail -3 gpurun_out/pytest_fma.log
timeout 900 python tools/run_reference_tests.py > gpurun_out/reftests.log 2>&1; echo "reftests rc=$?"; tail -5 gpurun_out/reftests.log
TAG=r02a CONFIGS="4 1" bash tools/gpu/ncu_pass.sh
