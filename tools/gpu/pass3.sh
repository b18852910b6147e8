set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
VARS="nopair new" ENVS="- CBP_TILE_CFG=3" CFGS="4 1" ITERS=2 bash tools/ab/ab_grid.sh > gpurun_out/ab_pair.log 2>&1
cat gpurun_out/ab_pair.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bp_tiled -c 1 -o gpurun_out/r02b_cfg4slab -f \
  python tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:1152 > gpurun_out/r02b_cfg4slab_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bp_tiled -c 1 -o gpurun_out/r02b_cfg4slab_nopair -f \
  python ab/nopair/tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:1152 > gpurun_out/r02b_cfg4slab_nopair_ncu.log 2>&1; echo "ncu rc=$?"
