set -e
cd $GRAFT_REPO_ROOT
for c in 1 2 3; do python tools/prof_run.py --config $c --uniform --iters 5 2>&1 | tail -1; done
for v in subline transpose share symmetry; do python tools/prof_run.py --config 1 --uniform --iters 5 --variant $v 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -3
