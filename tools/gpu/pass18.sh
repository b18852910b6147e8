# validation of the final library (general-path address FMAs): every GPU test, benches, the cfg2 capture
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench_cfg4.json
timeout 600 python bench.py --config 2 --steps 10 --no-cpu > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench2 rc=$?"; tail -c 300 gpurun_out/bench_cfg2.json
for c in 0 1 2 3 4; do echo "== cfg$c $(timeout 600 python tools/prof_run.py --config $c --uniform --iters 3 2>&1 | tail -2 | tr '\n' ' ')"; done > gpurun_out/kernel_all_configs.txt 2>&1; cut -c1-60,330-420 gpurun_out/kernel_all_configs.txt
bash tools/gpu/ncu_one.sh r02g_cfg2 --config 2 --uniform --iters 1
CBP_LIB_PATH=$PWD/ab/assert/paper_2104_13248_b200/libconebp_b200.so timeout 600 python tools/sanitize_cases.py medium_general > gpurun_out/assert_general.log 2>&1; echo "assert rc=$?"; tail -2 gpurun_out/assert_general.log
