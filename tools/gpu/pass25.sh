# tile-shape sweep on the final library (env override, no rebuild): cfg1 (fast path) and cfg2 (general path)
cd $GRAFT_REPO_ROOT
for c in 1 2; do for t in 0 1 2 3 4 5 6; do
  echo "== cfg$c tile$t $(CBP_TILE_CFG=$t timeout 300 python tools/prof_run.py --config $c --uniform --iters 4 2>&1 | tail -1)"
done; done
