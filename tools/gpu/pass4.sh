set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
VARS="new rowshift" CFGS="4 1" ITERS=2 bash tools/ab/ab_grid.sh > gpurun_out/ab_rowshift.log 2>&1
cat gpurun_out/ab_rowshift.log
bash tools/gpu/ncu_one.sh r02c_cfg4slab --config 4 --uniform --iters 1 --slab 896:1152
