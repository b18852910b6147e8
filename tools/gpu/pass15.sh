# host pipeline with the central slab first: parity of the chunked / slabbed host path, then the bench (e2e leg)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -m gpu -k "host or numpy or chunk or slab" > gpurun_out/pytest_host.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_host.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench_cfg4_b.json 2> gpurun_out/bench_cfg4_b.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_cfg4_b.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "exec", d["roofline"]["executed"]["frac"], "traffic", d["roofline"]["traffic"], d["clocks"])
PY
for sl in 8 12 16; do echo "== slabs $sl: $(CBP_HOST_SLABS=$sl timeout 600 python bench.py --no-cpu --steps 1 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e']['value'], d['e2e']['ms_per_step'])")"; done
