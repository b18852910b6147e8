# 15-consumer-warp tiles (16 warps per CTA: 128 registers per thread) vs the 16+1-warp tile (96 registers); slim build
cd $GRAFT_REPO_ROOT
echo "== sha HEAD cfg1 $(timeout 300 python tools/prof_run.py --config 1 --uniform --iters 1 --sha 2>&1 | tail -1)"
echo "== sha HEAD cfg4slab $(timeout 300 python tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:960 --sha 2>&1 | tail -1)"
for t in 0 7 8; do
  echo "== sha t15+tile$t cfg1 $(CBP_TILE_CFG=$t timeout 300 python ab/t15/tools/prof_run.py --config 1 --uniform --iters 1 --sha 2>&1 | tail -1)"
  echo "== sha t15+tile$t cfg4slab $(CBP_TILE_CFG=$t timeout 300 python ab/t15/tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:960 --sha 2>&1 | tail -1)"
done
for r in 1 2; do
for c in 4 1; do
  if [ $c = 4 ]; then S="--slab 896:1152"; else S=""; fi
  echo "== t15 default cfg$c $(timeout 300 python ab/t15/tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -1)"
  for t in 0 7 8 3; do
    echo "== t15+tile$t cfg$c $(CBP_TILE_CFG=$t timeout 300 python ab/t15/tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -2 | tr '\n' ' ')"
  done
done; done
