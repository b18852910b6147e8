"""Time the host (numpy, pinned) path of config 1 for several chunk counts."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2104_13248_b200 import ProjectionStack, Volume, backproject_baseline, configs
spec = configs.get_config(1); geom = spec.geometry(); mats = spec.matrices(geom)
img_pin = torch.empty((geom.np, geom.nh, geom.nw), dtype=torch.float32, pin_memory=True)
img_pin.copy_(torch.rand((geom.np, geom.nh, geom.nw)))
vol_pin = torch.zeros((geom.nz, geom.ny, geom.nx), dtype=torch.float32, pin_memory=True)
proj = ProjectionStack(img_pin.numpy(), geom.np, geom.nh, geom.nw)
vol = Volume(vol_pin.numpy(), geom.nx, geom.ny, geom.nz)
for ch in sys.argv[1:]:
    os.environ["CBP_HOST_CHUNKS"] = ch
    for _ in range(2): backproject_baseline(proj, mats, vol)
    t = []
    for _ in range(5):
        t0 = time.perf_counter(); backproject_baseline(proj, mats, vol); t.append(time.perf_counter() - t0)
    print(f"chunks {ch}: {[round(x*1e3,2) for x in t]} ms")
