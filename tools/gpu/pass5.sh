set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
VARS="new" ENVS="- CBP_STAGGER_GROUPS=2,CBP_STAGGER_NS=600 CBP_STAGGER_GROUPS=2,CBP_STAGGER_NS=300 CBP_STAGGER_GROUPS=4,CBP_STAGGER_NS=300 CBP_STAGGER_GROUPS=4,CBP_STAGGER_NS=150" CFGS="4 1" ITERS=2 bash tools/ab/ab_grid.sh > gpurun_out/ab_stagger.log 2>&1
cat gpurun_out/ab_stagger.log
