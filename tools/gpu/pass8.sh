set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
VARS="new realloc" CFGS="4 1 3" ITERS=2 bash tools/ab/ab_grid.sh > gpurun_out/ab_realloc.log 2>&1
cat gpurun_out/ab_realloc.log
