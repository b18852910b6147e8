set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
VARS="new" ENVS="- CBP_TILE_GROUP=4 CBP_TILE_GROUP=8 CBP_TILE_GROUP=16" CFGS="4 1" ITERS=2 bash tools/ab/ab_grid.sh > gpurun_out/ab_group.log 2>&1
cat gpurun_out/ab_group.log
for g in 1 8; do
  CBP_TILE_GROUP=$g timeout 600 ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:bp_tiled -c 1 \
    python tools/prof_run.py --config 4 --uniform --iters 1 --slab 896:1152 > gpurun_out/dram_group$g.log 2>&1
  grep -E "dram__bytes_read|hit_rate|duration" gpurun_out/dram_group$g.log
done
