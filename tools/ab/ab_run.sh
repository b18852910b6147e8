# A/B driver on the GPU box: defaults vs env-switched variants
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-1 3}; do
  echo "== cfg$c default"; timeout 300 python tools/prof_run.py --config $c --uniform --iters 4 2>&1 | tail -2
  for e in ${ENVS:-CBP_NO_TY_TABLE=1}; do
    echo "== cfg$c $e"; env $e timeout 300 python tools/prof_run.py --config $c --uniform --iters 4 2>&1 | tail -1
  done
done
