cd $GRAFT_REPO_ROOT
for c in ${CFGS:-1 3}; do for t in ${TILES:-0 1}; do
  echo "== cfg$c tile $t"; CBP_TILE_CFG=$t timeout 300 python tools/prof_run.py --config $c --uniform --iters ${ITERS:-3} 2>&1 | tail -2
done; done
