# re-validation of the final library (shared-window address hoist, FDK constant-stride addressing, reference-suite retry)
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
CBP_REFTEST_FORCE_RETRY=1 timeout 900 python tools/run_reference_tests.py > gpurun_out/reftest_forced_retry.log 2>&1; echo "forced retry rc=$?"; tail -1 gpurun_out/reftest_forced_retry.log | cut -c1-600
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?"; tail -c 500 gpurun_out/bench_cfg4.json
timeout 600 python bench.py --config 1 --steps 20 --e2e-pageable > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "bench1 rc=$?"
timeout 900 python bench.py --no-cpu --steps 2 --e2e-pageable > gpurun_out/bench_cfg4_pageable.json 2> gpurun_out/bench_cfg4_pageable.err; echo "bench pageable rc=$?"
timeout 600 python tools/time_f1_f2.py --skip-f2 > gpurun_out/f1.log 2>&1; echo "f1 rc=$?"; tail -1 gpurun_out/f1.log | cut -c1-700
