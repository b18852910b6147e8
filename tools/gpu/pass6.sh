set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
VARS="new fwd" ENVS="- CBP_MAX_STAGES=3 CBP_MAX_STAGES=2" CFGS="4 1" ITERS=2 bash tools/ab/ab_grid.sh > gpurun_out/ab_fwd.log 2>&1
cat gpurun_out/ab_fwd.log
