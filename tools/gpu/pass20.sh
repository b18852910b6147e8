# FDK filter with the XOR index swizzle: tests, timing, one ncu capture (bank conflicts), then a last smoke + quick parity subset
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_fdk.py tests/test_cli.py tests/test_phantom.py -q -m gpu > gpurun_out/pytest_f1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_f1.log
for r in 1 2; do timeout 600 python tools/time_f1_f2.py --skip-f2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('== f1', {k:round(v['f1_fdk_filter']['ms'],3) for k,v in d.items()})"; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fdk_filter -c 1 -o /tmp/r02h_f1 -f python tools/time_f1_f2.py --configs 3 --skip-f2 > gpurun_out/r02h_f1_ncu.log 2>&1; echo "ncu f1 rc=$?"
ncu -i /tmp/r02h_f1.ncu-rep --page raw --csv > gpurun_out/r02h_f1_raw.csv 2>/dev/null
ncu -i /tmp/r02h_f1.ncu-rep --page source --csv --print-source sass > gpurun_out/r02h_f1_src.csv 2>/dev/null; gzip -f gpurun_out/r02h_f1_src.csv
timeout 900 python tools/time_f1_f2.py > gpurun_out/f1f2.log 2>&1; echo "f1f2 rc=$?"; tail -1 gpurun_out/f1f2.log | cut -c1-300
