# general path (cfg2, jittered matrices): FRND floors + subnormal-FMA addresses vs magic-number floors + IMAD; slim builds
cd $GRAFT_REPO_ROOT
for v in genold genaf; do echo "== sha $v cfg2 $(timeout 300 python ab/$v/tools/prof_run.py --config 2 --uniform --iters 1 --sha 2>&1 | tail -1)"; done
echo "== sha lib cfg2 $(timeout 300 python tools/prof_run.py --config 2 --uniform --iters 1 --sha 2>&1 | tail -1)"
for r in 1 2; do for v in genold genaf; do
  echo "== $v cfg2 $(timeout 300 python ab/$v/tools/prof_run.py --config 2 --uniform --iters 4 2>&1 | tail -1)"
done; done
