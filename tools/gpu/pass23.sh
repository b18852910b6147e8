# forward projector with the y-contiguous volume copy: bitwise tests and timing
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_phantom.py tests/test_cli.py tests/test_fdk.py -q -m gpu > gpurun_out/pytest_f2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_f2.log
timeout 900 python tools/time_f1_f2.py > gpurun_out/f1f2.log 2>&1; echo "f1f2 rc=$?"; tail -1 gpurun_out/f1f2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v['f1_fdk_filter']['ms'],2), round(v['f2_forward_projector']['ms'],1), round(v['f2_forward_projector']['rays_per_s']/1e6,1)) for k,v in d.items()})"
