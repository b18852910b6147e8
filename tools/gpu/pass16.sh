# final round-2 pass: smoke, every GPU test, benches (both arms), NCCL launch path, kernel times on every config,
# launch list, f1/f2 timings, assert-checked build, slab balance
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_cfg4.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "bench ref rc=$?"; tail -c 900 gpurun_out/bench_reference.json
timeout 600 python bench.py --config 1 --steps 20 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "bench1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo "torchrun rc=$?"; tail -c 400 gpurun_out/bench_torchrun1.json
for c in 0 1 2 3 4; do echo "== cfg$c $(timeout 600 python tools/prof_run.py --config $c --uniform --iters 3 2>&1 | tail -2 | tr '\n' ' ')"; done > gpurun_out/kernel_all_configs.txt 2>&1; cat gpurun_out/kernel_all_configs.txt | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:bp_|stage_|fdk_" -c 400 --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r02f_launches_bench.log 2>&1; echo "launch list rc=$?"
timeout 900 python tools/time_f1_f2.py > gpurun_out/f1f2.log 2>&1; echo "f1f2 rc=$?"; tail -1 gpurun_out/f1f2.log
CBP_LIB_PATH=$PWD/ab/assert/paper_2104_13248_b200/libconebp_b200.so timeout 1200 python tools/sanitize_cases.py > gpurun_out/assert_build_cases.log 2>&1; echo "assert cases rc=$?"; tail -3 gpurun_out/assert_build_cases.log
CBP_LIB_PATH=$PWD/ab/assert/paper_2104_13248_b200/libconebp_b200.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "cfg0 or rungs_bitwise_small or awkward or every_tile_shape or cfg1_size" > gpurun_out/assert_build_pytest.log 2>&1; echo "assert pytest rc=$?"; tail -3 gpurun_out/assert_build_pytest.log
for c in 2 3 4; do timeout 900 python tools/slab_balance.py --config $c --ranks 2 4 8 --align 16 > gpurun_out/slab_cfg${c}.log 2>&1; echo "slab cfg$c rc=$?"; grep "N=" gpurun_out/slab_cfg${c}.log; done
