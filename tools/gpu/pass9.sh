set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench.json
SAN_TIMEOUT=900 bash tools/gpu/sanitize.sh
timeout 900 python tools/time_f1_f2.py > gpurun_out/f1f2.log 2>&1; echo "f1f2 rc=$?"; tail -2 gpurun_out/f1f2.log
for c in 3 2; do for a in 32 16; do
  timeout 900 python tools/slab_balance.py --config $c --ranks 2 4 8 --align $a > gpurun_out/slab_cfg${c}_a${a}.log 2>&1; echo "slab cfg$c a$a rc=$?"; grep "N=" gpurun_out/slab_cfg${c}_a${a}.log
done; done
