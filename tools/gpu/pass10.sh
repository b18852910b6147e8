# full GPU pass of HEAD: smoke, all GPU tests, bench cfg4 (default) and cfg1
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?"; tail -c 1200 gpurun_out/bench_cfg4.json
timeout 600 python bench.py --config 1 --steps 20 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "bench1 rc=$?"; tail -c 600 gpurun_out/bench_cfg1.json
