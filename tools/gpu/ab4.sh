# TY table from the constant bank (new) vs stage header (ab/afma); tile shapes; per-warp poll diagnostic
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "cfg1_size_bitwise or cfg4_full or cfg0_bitwise or every_tile_shape or rungs_bitwise_small or awkward" > gpurun_out/ab4_parity.log 2>&1
echo "parity(new) rc=$?"; tail -3 gpurun_out/ab4_parity.log
for r in 1 2; do
for c in 4 1; do
  if [ $c = 4 ]; then S="--slab 896:1152"; else S=""; fi
  for v in new afma; do
    if [ "$v" = new ]; then P=tools/prof_run.py; else P=ab/$v/tools/prof_run.py; fi
    echo "== $v cfg$c $(timeout 300 python $P --config $c --uniform --iters 3 $S 2>&1 | tail -1)"
  done
  if [ $r = 1 ]; then for t in 1 2 6; do
    echo "== new+tile$t cfg$c $(CBP_TILE_CFG=$t timeout 300 python tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -2 | tr '\n' ' ')"
  done; fi
done; done
timeout 300 python ab/poll/tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:1152 > gpurun_out/ab4_poll.log 2>&1
grep POLL gpurun_out/ab4_poll.log | sort -k3,3n -k5,5n | head -40
