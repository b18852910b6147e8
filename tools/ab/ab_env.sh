# same build, different env settings:  ENVS="A=1 B=2" CFGS="1"
cd $GRAFT_REPO_ROOT
for c in ${CFGS:-1}; do for e in X=0 ${ENVS}; do
  echo "== cfg$c $e $(env $e timeout 300 python tools/prof_run.py --config $c --uniform --iters ${ITERS:-3} 2>&1 | tail -1)"
done; done
