cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fdk.py -q -m gpu > gpurun_out/pytest_f1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_f1.log
timeout 600 python tools/time_f1_f2.py --configs 1 3 --skip-f2 2>&1 | tail -1
# box row pitch modulo 32 words: bank conflicts on the magnification-2 configs
for c in 1 2; do for pad in 16 0 4 8 12 20 24 28; do
  echo "== cfg$c pad$pad $(CBP_BOX_PAD=$pad timeout 300 python tools/prof_run.py --config $c --uniform --iters 3 2>&1 | tail -2 | tr '\n' ' ' | cut -c1-60,200-420)"
done; done
