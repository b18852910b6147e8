# env sweeps (no rebuild): angle chunks of the host pipeline's first slab; tile launch group size
cd $GRAFT_REPO_ROOT
for ch in 24 12 16 32 48 64; do echo "== e2e chunks $ch: $(CBP_HOST_CHUNKS=$ch timeout 600 python bench.py --no-cpu --steps 1 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1))")"; done
for g in 8 4 16 32; do echo "== tile group $g cfg3: $(CBP_TILE_GROUP=$g timeout 300 python tools/prof_run.py --config 3 --uniform --iters 3 2>&1 | tail -1)"; done
