# ncu evidence for the final round-2 kernel: DRAM bytes per launch on every config, full captures of cfg4 (central slab) and cfg1
cd $GRAFT_REPO_ROOT
for c in 1 2 3 4; do
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none \
    -k regex:bp_tiled -c 1 --csv --log-file gpurun_out/r02f_traffic_cfg$c.csv python tools/prof_run.py --config $c --iters 1 --uniform \
    > gpurun_out/r02f_traffic_cfg$c.log 2>&1
  echo "traffic cfg$c rc=$?"; tail -2 gpurun_out/r02f_traffic_cfg$c.csv
done
bash tools/gpu/ncu_one.sh r02f_cfg4slab --config 4 --uniform --iters 1 --slab 896:1152
bash tools/gpu/ncu_one.sh r02f_cfg1 --config 1 --uniform --iters 1
bash tools/gpu/ncu_one.sh r02f_cfg2 --config 2 --uniform --iters 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    > gpurun_out/r02f_launches_bench.log 2>&1
echo "launch list rc=$?"
