"""Profiling driver: N back-projections of one config through the device API (for ncu)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2104_13248_b200 import KernelVariant, configs
from paper_2104_13248_b200 import device as D

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--variant", default="baseline")
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--uniform", action="store_true", help="uniform inputs instead of the phantom (faster setup)")
ap.add_argument("--slab", default=None, help="k0:k1 -- back-project only this z-slab (global indices; for ncu on cfg4)")
ap.add_argument("--sha", action="store_true", help="print the sha256 of the resulting slab (A/B bit-equality checks)")
a = ap.parse_args()
spec = configs.get_config(a.config)
geom = spec.geometry()
mats = spec.matrices(geom)
torch.manual_seed(11)
if a.uniform:
    img = torch.rand((geom.np, geom.nh, geom.nw), device="cuda") * 2 - 1
else:
    img = spec.projections_device(geom, device="cuda")
st = D.StagedProjections(img, geom.np, geom.nh, geom.nw)
k0, k1 = (int(t) for t in a.slab.split(":")) if a.slab else (0, geom.nz)
vol = torch.zeros((k1 - k0, geom.ny, geom.nx), device="cuda")
v = KernelVariant.parse(a.variant)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.iters)]
for i in range(a.iters):
    ev[2 * i].record()
    D.backproject_staged(st, mats, vol, geom.nx, geom.ny, k1 - k0, v, k0=k0, nz_total=geom.nz, flags=a.flags)
    ev[2 * i + 1].record()
torch.cuda.synchronize()
ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(a.iters)]
print("plan", D.last_plan(), "stats", D.sync_status())
print("ms", [round(x, 3) for x in ms], "GUPS", [round(geom.nx * geom.ny * (k1 - k0) * geom.np / (x * 1e6), 1) for x in ms])
if a.sha:
    import hashlib
    print("sha", hashlib.sha256(vol.cpu().numpy().tobytes()).hexdigest())
