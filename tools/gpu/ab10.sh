# header term for the column address constant (cden) and address FMAs in the guarded fast-path loop (gaf); slim builds
cd $GRAFT_REPO_ROOT
for v in base cden gaf both; do
  echo "== sha $v cfg1 $(timeout 300 python ab/$v/tools/prof_run.py --config 1 --uniform --iters 1 --sha 2>&1 | tail -1)"
  echo "== sha $v cfg4slab $(timeout 300 python ab/$v/tools/prof_run.py --config 4 --uniform --iters 1 --slab 0:64 --sha 2>&1 | tail -1)"
done
for r in 1 2; do for c in 4 1; do
  if [ $c = 4 ]; then S="--slab 896:1152"; else S=""; fi
  for v in base cden gaf both; do
    echo "== $v cfg$c $(timeout 300 python ab/$v/tools/prof_run.py --config $c --uniform --iters 4 $S 2>&1 | tail -1)"
  done
done; done
