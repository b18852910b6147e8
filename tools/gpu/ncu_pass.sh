# ncu captures of the back-projection kernel (run under gpurun from the repo root, one GPU)
# usage: TAG=r02a CONFIGS="1 4" bash tools/gpu/ncu_pass.sh
set -x
TAG=${TAG:-r02}
for c in ${CONFIGS:-1 4}; do
  U=""; [ "$c" = "4" ] && U="--uniform"
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:bp_tiled -c 1 \
    -o gpurun_out/${TAG}_cfg${c} -f python tools/prof_run.py --config $c --iters 1 $U ${EXTRA:-} \
    > gpurun_out/${TAG}_cfg${c}_ncu.log 2>&1
  echo "cfg$c ncu rc=$?"
  tail -3 gpurun_out/${TAG}_cfg${c}_ncu.log
done
if [ -n "$LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/${TAG}_launches_bench.log 2>&1
  echo "launch list rc=$?"
fi
