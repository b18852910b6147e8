"""Debug: TMA path with the caller's transposed buffer (no internal staging) vs staged copy."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np
import torch

from conftest import load_golden
from paper_2104_13248_b200 import KernelVariant, Layout
from paper_2104_13248_b200 import device as D

mode = sys.argv[1]
g = load_golden("tiny")
n, nh, nw = g["img"].shape
nz, ny, nx = g["vol0"].shape
vol = torch.from_numpy(g["vol0"].copy()).cuda()
if mode == "transposed":
    img_t = torch.from_numpy(np.ascontiguousarray(g["img"].transpose(0, 2, 1))).cuda()
    D.backproject_device(img_t, g["mats"], vol, n, nh, nw, nx, ny, nz, KernelVariant.BASELINE, Layout.TRANSPOSED,
                         Layout.NATURAL)
else:  # staged via torch memory
    img = torch.from_numpy(g["img"]).cuda()
    st = D.StagedProjections(img, n, nh, nw)
    D.backproject_staged(st, g["mats"], vol, nx, ny, nz)
print("plan", D.last_plan(), flush=True)
print("stats", D.sync_status(), flush=True)
out = vol.cpu().numpy()
print("bitwise", out.tobytes() == g["baseline"].tobytes())
