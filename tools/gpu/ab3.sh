# round-2 session-4 A/B: poll sleep, FRND + subnormal-FMA addresses, 24x24 tile (cfg 5)
cd $GRAFT_REPO_ROOT
# correctness of the new address arithmetic first (bitwise digests at cfg1 size, cfg4 slabs vs oracle)
CBP_LIB_PATH=$PWD/ab/both/paper_2104_13248_b200/libconebp_b200.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x \
  -k "cfg1_size_bitwise or cfg4_full or cfg0_bitwise or every_tile_shape" > gpurun_out/ab3_parity_both.log 2>&1
echo "parity(both) rc=$?"; tail -3 gpurun_out/ab3_parity_both.log
for r in 1 2; do
for c in 4 1; do
  if [ $c = 4 ]; then S="--slab 896:1152"; else S=""; fi
  for v in new sleep afma both; do
    if [ "$v" = new ]; then P=tools/prof_run.py; else P=ab/$v/tools/prof_run.py; fi
    echo "== $v cfg$c $(timeout 300 python $P --config $c --uniform --iters 3 $S 2>&1 | tail -1)"
  done
  echo "== new+tile5 cfg$c $(CBP_TILE_CFG=5 timeout 300 python tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -1)"
  echo "== both+tile5 cfg$c $(CBP_TILE_CFG=5 timeout 300 python ab/both/tools/prof_run.py --config $c --uniform --iters 3 $S 2>&1 | tail -1)"
done; done
