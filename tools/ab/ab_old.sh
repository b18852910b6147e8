# old (ab/old, previous commit build) vs new, interleaved, same box
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for c in ${CFGS:-1}; do
  echo "== old cfg$c"; timeout 300 python ab/old/tools/prof_run.py --config $c --uniform --iters 4 2>&1 | tail -1
  echo "== new cfg$c"; env ${NEWENV:-X=1} timeout 300 python tools/prof_run.py --config $c --uniform --iters 4 2>&1 | tail -1
done; done
