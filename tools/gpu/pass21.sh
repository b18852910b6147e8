# planner with general-path cost weights: slab balance on cfg2 (changed) and cfg3 (must not change), planner-dependent tests
cd $GRAFT_REPO_ROOT
for c in 2 3; do timeout 900 python tools/slab_balance.py --config $c --ranks 2 4 8 --align 16 > gpurun_out/slab_cfg${c}.log 2>&1; echo "slab cfg$c rc=$?"; grep "N=" gpurun_out/slab_cfg${c}.log; done
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_slabs.py -q -m gpu > gpurun_out/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_multi.log
