set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import numba; print(numba.__version__)"
NUMBA_CACHE_DIR=/tmp/nbc PYTHONPATH=baseline/_ref timeout 300 python - <<'PY'
import os, time, numpy as np
import conebp
from conebp import geometry as G
import numba
print("numba threads", numba.get_num_threads(), os.cpu_count())
g = G.build_geometry(nx=256, ny=256, nz=256, nw=512, nh=512, np=360, d=750.0, D=1200.0, pixel_pitch_u=0.8, pixel_pitch_v=0.8, voxel_size=1.0)
m = G.projection_matrices(g)
img = np.random.default_rng(0).uniform(-1,1,(360,512,512)).astype(np.float32)
P = conebp.ProjectionStack(img, 360, 512, 512)
for it in range(3):
    V = conebp.Volume.zeros(256,256,256)
    t=time.perf_counter(); conebp.backproject_baseline(P, m, V); dt=time.perf_counter()-t
    print("cfg1 full", dt, 256**3*360/dt/1e9, "GUPS")
PY
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu --no-e2e
