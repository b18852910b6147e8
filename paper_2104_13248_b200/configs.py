"""The five BASELINE.json workloads as geometry + matrices + input recipes.

| cfg | volume | projections | geometry | inputs |
|---|---|---|---|---|
| 0 | 64^3, voxel 0.5 | 90 x 128x128, pitch 1.0 | d 1000, D 1500, 360 deg | uniform[-1,1) seed 0 |
| 1 | 256^3, voxel 1.0 | 360 x 512x512, pitch 0.8 | d 750, D 1200, 360 deg | 10 ellipsoids (seed 1), cosine + Ram-Lak |
| 2 | 512^3, voxel 0.5 | 496 x 960x1248 (nh x nw), pitch 0.32 | d 750, D 1200, 200 deg short scan, jitter sigma 0.5 (seed 2) | 10 ellipsoids (seed 2), cosine + Ram-Lak |
| 3 | 1024^3, voxel 0.25 | 1440 x 1536x1536, pitch 0.2 | d 1000, D 1500, 360 deg | 30 ellipsoids 2-30% (seed 3), cosine + Ram-Lak |
| 4 | 2048^3, voxel 0.125 | 2048 x 2048x2048, pitch 0.1 | d 1000, D 1500, 360 deg, u offset +16 px | uniform[-1,1) seed 7 |

Open items of SURVEY.md section 9, decided here: config 2's "1248x960" is
nw = 1248 (u) by nh = 960 (v); short-scan angles are s*200deg/496 (half
open); jitter perturbs source and detector centre per angle (geometry.
jittered_views); seeds as in the table.  Uniform inputs for configs 0 and 4
use numpy's default_rng on the host for config 0 and torch's device RNG for
config 4 (32 GiB: host generation would dominate the run).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import geometry as G
from . import phantom as P

__all__ = ["ConfigSpec", "CONFIGS", "get_config"]


@dataclass(frozen=True)
class ConfigSpec:
    index: int
    name: str
    geom_kwargs: dict
    angle_span: float = 2.0 * math.pi
    jitter_sigma: float = 0.0
    jitter_seed: int = 0
    u_offset_px: float = 0.0
    inputs: str = "uniform"        # "uniform" | "phantom"
    seed: int = 0
    n_ellipsoids: int = 0
    semi_frac: tuple = (0.05, 0.40)

    def geometry(self) -> G.ScanGeometry:
        n_proj = self.geom_kwargs["np"]
        angles = tuple(self.angle_span * s / n_proj for s in range(n_proj))
        return G.build_geometry(angles=angles, **self.geom_kwargs)

    def views(self, geom=None):
        geom = geom or self.geometry()
        if self.jitter_sigma > 0:
            return G.jittered_views(geom, self.jitter_sigma, self.jitter_seed)
        return G.circular_views(geom)

    def matrices(self, geom=None) -> np.ndarray:
        geom = geom or self.geometry()
        if self.jitter_sigma > 0:
            mats = G.view_matrices(geom, self.views(geom))
        else:
            mats = G.projection_matrices(geom)
        if self.u_offset_px:
            mats = G.u_offset(mats, self.u_offset_px)
        return mats

    @property
    def updates(self) -> int:
        k = self.geom_kwargs
        return k["nx"] * k["ny"] * k["nz"] * k["np"]

    def projections_host(self, geom=None) -> np.ndarray:
        """NATURAL (np, nh, nw) float32 projections on the host."""
        geom = geom or self.geometry()
        if self.inputs == "uniform":
            return P.uniform_projections(geom.np, geom.nh, geom.nw, self.seed)
        return self.projections_device(geom, device="cpu").numpy()

    def projections_device(self, geom=None, device="cuda"):
        """NATURAL (np, nh, nw) float32 torch tensor on ``device``."""
        import torch

        geom = geom or self.geometry()
        if self.inputs == "uniform":
            if self.index == 4:
                return P.uniform_projections_device(geom.np, geom.nh, geom.nw, self.seed, device=device)
            return torch.from_numpy(P.uniform_projections(geom.np, geom.nh, geom.nw, self.seed)).to(device)
        ell = P.random_ellipsoids(self.n_ellipsoids, geom, self.semi_frac, self.seed)
        return P.filtered_phantom_projections(geom, self.views(geom), ell, device=device)

    def describe(self) -> dict:
        k = self.geom_kwargs
        return {"workload": self.name, "volume": [k["nx"], k["ny"], k["nz"]], "np": k["np"], "nh": k["nh"],
                "nw": k["nw"], "inputs": self.inputs}


CONFIGS = (
    ConfigSpec(0, "cfg0_64cube_90x128sq", dict(nx=64, ny=64, nz=64, nw=128, nh=128, np=90, d=1000.0, D=1500.0,
                                                pixel_pitch_u=1.0, pixel_pitch_v=1.0, voxel_size=0.5),
               inputs="uniform", seed=0),
    ConfigSpec(1, "cfg1_256cube_360x512sq", dict(nx=256, ny=256, nz=256, nw=512, nh=512, np=360, d=750.0, D=1200.0,
                                                  pixel_pitch_u=0.8, pixel_pitch_v=0.8, voxel_size=1.0),
               inputs="phantom", seed=1, n_ellipsoids=10),
    ConfigSpec(2, "cfg2_512cube_496x960x1248_jitter", dict(nx=512, ny=512, nz=512, nw=1248, nh=960, np=496, d=750.0,
                                                            D=1200.0, pixel_pitch_u=0.32, pixel_pitch_v=0.32,
                                                            voxel_size=0.5),
               angle_span=math.radians(200.0), jitter_sigma=0.5, jitter_seed=2, inputs="phantom", seed=2,
               n_ellipsoids=10),
    ConfigSpec(3, "cfg3_1024cube_1440x1536sq", dict(nx=1024, ny=1024, nz=1024, nw=1536, nh=1536, np=1440, d=1000.0,
                                                     D=1500.0, pixel_pitch_u=0.2, pixel_pitch_v=0.2, voxel_size=0.25),
               inputs="phantom", seed=3, n_ellipsoids=30, semi_frac=(0.02, 0.30)),
    ConfigSpec(4, "cfg4_2048cube_2048x2048sq_uoff16", dict(nx=2048, ny=2048, nz=2048, nw=2048, nh=2048, np=2048,
                                                            d=1000.0, D=1500.0, pixel_pitch_u=0.1, pixel_pitch_v=0.1,
                                                            voxel_size=0.125),
               u_offset_px=16.0, inputs="uniform", seed=7),
)


def get_config(index: int) -> ConfigSpec:
    return CONFIGS[index]
