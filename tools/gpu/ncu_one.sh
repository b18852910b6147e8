# ncu --set full of ONE back-projection launch; reports stay on the box (/tmp), only CSV exports
# come back (gpurun_out/ is capped at 64 MiB).  usage: bash tools/gpu/ncu_one.sh TAG <prof_run args...>
TAG=$1; shift
PR=${PROF_RUN:-tools/prof_run.py}
timeout ${NCU_TIMEOUT:-900} ncu --set full --import-source on --clock-control none -k regex:bp_tiled -c 1 \
  -o /tmp/$TAG -f python $PR "$@" > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu $TAG rc=$?"
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_src.csv
ls -la gpurun_out/${TAG}_*
