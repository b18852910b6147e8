cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_fdk.py -q -m gpu > gpurun_out/pytest_f1.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_f1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fdk_ --csv --log-file gpurun_out/f1_launches.csv python tools/time_f1_f2.py --configs 1 3 --skip-f2 > gpurun_out/f1_ncu.log 2>&1
echo "ncu rc=$?"; grep -E "fdk_" gpurun_out/f1_launches.csv | awk -F'","' '{print $5, $NF}' | head -20
timeout 600 python tools/time_f1_f2.py --configs 1 3 --skip-f2 2>&1 | tail -1
