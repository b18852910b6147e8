"""Timings of the rows next to the hot path: f1 FDK pre-processing and f2 forward projector.

    python tools/time_f1_f2.py [--configs 1 3]

f1 ``cbp_fdk_filter_f32``: one fused kernel (weight, zero-padded shared-memory FFT of two rows
per complex transform, Ram-Lak spectrum, inverse, crop into the staging layout).  Reported
against HBM on its compulsory bytes = raw read + staged write (8 B per texel), which is all it
moves, and as FP32 work (10 N log2 N flops per complex transform pair forward + inverse).
f2 ``cbp_forward_project_f32`` (float64 ray marching, the reference's arithmetic): rays/s
on the config's grid (a subset of 32 angles).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2104_13248_b200 import _lib, configs
from paper_2104_13248_b200 import fdk as F
from paper_2104_13248_b200.device import stream_handle
from paper_2104_13248_b200.geometry import circular_views
from paper_2104_13248_b200.phantom import _views_array


def timed(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(iters):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return min(ms)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 3])
    ap.add_argument("--skip-f2", action="store_true")
    args = ap.parse_args()
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    out = {}
    for c in args.configs:
        spec = configs.get_config(c)
        geom = spec.geometry()
        n_proj, nh, nw = geom.np, geom.nh, geom.nw
        raw = torch.rand((n_proj, nh, nw), device="cuda")
        pitch = int(_lib.lib().cbp_staged_pitch(nw))
        staged = torch.empty((n_proj, nh, pitch), device="cuda")
        cu, cv = geom.detector_center

        def f1():
            _lib.check(_lib.lib().cbp_fdk_filter_f32(raw.data_ptr(), n_proj, nh, nw, float(geom.D),
                                                     float(geom.pixel_pitch_u), float(geom.pixel_pitch_v), float(cu),
                                                     float(cv), float(F.ramp_tau(geom)), staged.data_ptr(), pitch,
                                                     stream_handle()))

        ms1 = timed(f1)
        texels = n_proj * nh * nw
        nfft = 1
        while nfft < 2 * nw:
            nfft *= 2
        comp = 8.0 * texels
        logn = nfft.bit_length() - 1
        flops = 10.0 * nfft * logn * (n_proj * nh / 2.0)
        r1 = {"ms": ms1, "texels_per_s": texels / ms1 / 1e-3, "compulsory_gbs": comp / ms1 / 1e6,
              "hbm_peak_gbs": peaks.get("hbm_gbs"), "compulsory_frac": comp / ms1 / 1e6 / peaks.get("hbm_gbs", 6650.0),
              "transform_length": nfft, "fft_tflops": flops / ms1 / 1e9}
        del raw, staged
        # f2 on the config's grid (bounded: cfg3 is 1024^3 x 1440 x 1536^2 rays -> time a subset of angles)
        n_sub = min(n_proj, 32)
        vol = torch.rand((geom.nz, geom.ny, geom.nx), device="cuda")
        all_views = circular_views(geom)
        views = _views_array(all_views[::max(1, len(all_views) // n_sub)][:n_sub])  # evenly spaced over the orbit
        r2 = None
        if not args.skip_f2:
            outp = torch.empty((n_sub, nh, nw), device="cuda")

            def f2():
                _lib.check(_lib.lib().cbp_forward_project_f32(
                    vol.data_ptr(), geom.nx, geom.ny, geom.nz, float(geom.voxel_size),
                    views.ctypes.data_as(_lib.POINTER(_lib.ctypes.c_double)), n_sub, nh, nw,
                    float(geom.pixel_pitch_u), float(geom.pixel_pitch_v), float(cu), float(cv), outp.data_ptr(),
                    stream_handle()))

            ms2 = timed(f2, iters=2)
            os.environ["CBP_FWD_NATURAL_ONLY"] = "1"  # every ray reads the natural layout (round-2 first version)
            ms2_nat = timed(f2, iters=2)
            del os.environ["CBP_FWD_NATURAL_ONLY"]
            rays = n_sub * nh * nw
            r2 = {"ms": ms2, "ms_natural_layout_only": ms2_nat, "angles_timed": n_sub,
                  "angles": "evenly spaced over the orbit", "rays_per_s": rays / ms2 / 1e-3,
                  "note": "float64 ray marching (bitwise equal to the reference's numba _forward); rays that run "
                          "mostly along x read a y-contiguous copy of the volume (transpose inside the timed call)"}
        out[spec.name] = {"f1_fdk_filter": r1, "f2_forward_projector": r2}
        print(json.dumps({spec.name: out[spec.name]}), flush=True)
        del vol
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
