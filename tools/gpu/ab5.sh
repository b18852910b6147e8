# software-pipelined column terms: nopipe / pipe (ptxas placement) / pipel (pinned placement); slim builds, baseline rung
cd $GRAFT_REPO_ROOT
for v in nopipe pipe pipel; do
  echo "== sha $v cfg1 $(timeout 300 python ab/$v/tools/prof_run.py --config 1 --uniform --iters 1 --sha 2>&1 | tail -1)"
  echo "== sha $v cfg4slab $(timeout 300 python ab/$v/tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:960 --sha 2>&1 | tail -1)"
done
echo "== sha HEAD cfg1 $(timeout 300 python tools/prof_run.py --config 1 --uniform --iters 1 --sha 2>&1 | tail -1)"
for r in 1 2; do
for c in 4 1; do
  if [ $c = 4 ]; then S="--slab 896:1152"; else S=""; fi
  for v in nopipe pipe pipel; do
    echo "== $v cfg$c $(timeout 300 python ab/$v/tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -2 | tr '\n' ' ')"
  done
  [ $r = 1 ] && for v in nopipe pipel; do
    echo "== $v+tile3 cfg$c $(CBP_TILE_CFG=3 timeout 300 python ab/$v/tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -2 | tr '\n' ' ')"
  done
done; done
