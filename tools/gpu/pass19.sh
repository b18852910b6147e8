# ncu captures of the rows next to the hot path (f1 fused FDK filter on cfg3, f2 forward projector on cfg1) and the reference arm line
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fdk_filter -c 1 -o /tmp/r02g_f1 -f python tools/time_f1_f2.py --configs 3 --skip-f2 > gpurun_out/r02g_f1_ncu.log 2>&1; echo "ncu f1 rc=$?"
ncu -i /tmp/r02g_f1.ncu-rep --page raw --csv > gpurun_out/r02g_f1_raw.csv 2>/dev/null
ncu -i /tmp/r02g_f1.ncu-rep --page source --csv --print-source sass > gpurun_out/r02g_f1_src.csv 2>/dev/null; gzip -f gpurun_out/r02g_f1_src.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bp_forward -c 1 -o /tmp/r02g_f2 -f python tools/time_f1_f2.py --configs 1 > gpurun_out/r02g_f2_ncu.log 2>&1; echo "ncu f2 rc=$?"
ncu -i /tmp/r02g_f2.ncu-rep --page raw --csv > gpurun_out/r02g_f2_raw.csv 2>/dev/null
ncu -i /tmp/r02g_f2.ncu-rep --page source --csv --print-source sass > gpurun_out/r02g_f2_src.csv 2>/dev/null; gzip -f gpurun_out/r02g_f2_src.csv
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "bench ref rc=$?"; tail -c 700 gpurun_out/bench_reference.json
