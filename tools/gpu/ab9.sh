cd $GRAFT_REPO_ROOT
for v in genaf genxm; do echo "== sha $v cfg2 $(timeout 300 python ab/$v/tools/prof_run.py --config 2 --uniform --iters 1 --sha 2>&1 | tail -1)"; done
for r in 1 2; do for v in genaf genxm; do
  echo "== $v cfg2 $(timeout 300 python ab/$v/tools/prof_run.py --config 2 --uniform --iters 4 2>&1 | tail -1)"
done; done
for r in 1 2 3; do timeout 600 python tools/time_f1_f2.py --skip-f2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('== f1', {k:round(v['f1_fdk_filter']['ms'],3) for k,v in d.items()})"; done
