# interleaved A/B over builds: VARS="old s128" CFGS="1 3"; "new" = the working tree
cd $GRAFT_REPO_ROOT
for r in 1 2; do
for c in ${CFGS:-1}; do for v in ${VARS:-old new}; do
  if [ "$v" = new ]; then P=tools/prof_run.py; else P=ab/$v/tools/prof_run.py; fi
  echo "== $v cfg$c $(timeout 300 python $P --config $c --uniform --iters ${ITERS:-4} 2>&1 | tail -1)"
done; done; done
