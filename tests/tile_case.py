"""Subprocess helper for test_gpu_parity.test_every_tile_shape_bitwise: back-projects a
full-size digest case with the tile shape forced by CBP_TILE_CFG (read at plan time)
and prints the sha256 of the volume.  Not a test module.

    CBP_TILE_CFG=1 python tests/tile_case.py cfg1|cfg2
"""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from conftest import GOLDEN, uniform  # noqa: E402
from paper_2104_13248_b200 import KernelVariant, Layout, configs  # noqa: E402
from paper_2104_13248_b200 import device as D  # noqa: E402

case = sys.argv[1]
if case == "cfg1":
    spec = configs.get_config(1)
    mats = spec.matrices(spec.geometry())
    img, n = uniform(360, 512, 512, 11), 256
else:
    mats = np.load(GOLDEN / "cfg2_mats.npy")
    img, n = uniform(496, 960, 1248, 12), 512
n_proj, nh, nw = img.shape
ti = torch.from_numpy(img).cuda()
tv = torch.zeros((n, n, n), device="cuda")
D.backproject_device(ti, mats, tv, n_proj, nh, nw, n, n, n, KernelVariant.BASELINE, Layout.NATURAL, Layout.NATURAL)
st = D.sync_status()
assert st["band_violations"] == 0
print(hashlib.sha256(tv.cpu().numpy().tobytes()).hexdigest(), D.last_plan()["tile_x"], D.last_plan()["tile_y"])
