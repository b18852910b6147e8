"""Debug helper: run one small case through one library path in a fresh process."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

from conftest import load_golden
from paper_2104_13248_b200 import KernelVariant, Layout
from paper_2104_13248_b200 import device as D

flags = int(sys.argv[1])
case = sys.argv[2] if len(sys.argv) > 2 else "tiny"
g = load_golden(case)
img = torch.from_numpy(g["img"]).cuda()
vol = torch.from_numpy(g["vol0"].copy()).cuda()
nz, ny, nx = g["vol0"].shape
n, nh, nw = g["img"].shape
D.backproject_device(img, g["mats"], vol, n, nh, nw, nx, ny, nz, KernelVariant.BASELINE, Layout.NATURAL,
                     Layout.NATURAL, flags=flags)
print("plan", D.last_plan(), flush=True)
print("stats", D.sync_status(), flush=True)
out = vol.cpu().numpy()
print("bitwise", out.tobytes() == g["baseline"].tobytes(), "maxdiff", float(np.abs(out - g["baseline"]).max()))
