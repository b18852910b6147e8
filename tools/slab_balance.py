"""Slab load balance of the multi-GPU z-slab driver, projected on ONE GPU.

For config C and each N, plans the cost-balanced z-slabs (slabs.plan_slabs), then times
every rank's work -- its detector-row band staged in the device layout, its slab
back-projected over all angles -- one rank after another on the single GPU.  The ranks
of the real driver never wait on each other during compute (no collective after the
band distribution), so max over ranks of these times is the compute part of the N-GPU
step; T1 / (N * max) is the compute-only scaling efficiency.  The band bytes each rank
receives from rank 0 are printed as well (the copy-engine payload, not timed here).

    python tools/slab_balance.py --config 4 --ranks 2 4 8
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2104_13248_b200 import configs
from paper_2104_13248_b200 import device as D
from paper_2104_13248_b200 import slabs as SL


def time_slab(img, mats, plan, v0, rows, k0, k1, n_warm=64):
    if rows == 0 or k1 == k0:
        return 0.0
    band = torch.zeros((plan.np, rows, SL.pitch_of(plan.nw)), dtype=torch.float32, device="cuda")
    D.copy_band(img.data_ptr(), plan.np, plan.nh, plan.nw, 0, plan.np, v0, rows, band)
    staged = D.StagedProjections.wrap(band, plan.np, plan.nh, plan.nw, v0, rows)
    vol = torch.zeros((k1 - k0, plan.ny, plan.nx), dtype=torch.float32, device="cuda")
    D.backproject_staged(staged, mats, vol, plan.nx, plan.ny, k1 - k0, k0=k0, nz_total=plan.nz, s_end=min(n_warm, plan.np))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    D.backproject_staged(staged, mats, vol, plan.nx, plan.ny, k1 - k0, k0=k0, nz_total=plan.nz)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del band, vol, staged
    torch.cuda.empty_cache()
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--align", type=int, default=16, help="slab boundary granularity in slices (16 or 32)")
    args = ap.parse_args()
    spec = configs.get_config(args.config)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    img = torch.rand((geom.np, geom.nh, geom.nw), device="cuda") * 2 - 1
    updates = geom.nx * geom.ny * geom.nz * geom.np
    plan1 = SL.plan_slabs(mats, geom.nh, geom.nw, geom.nx, geom.ny, geom.nz, 1)
    t1 = time_slab(img, mats, plan1, *plan1.bands[0], *plan1.slab(0))
    out = {"config": args.config, "align": args.align, "updates": updates, "t1_ms": t1, "gups_1": updates / t1 / 1e6, "runs": []}
    print(f"cfg{args.config}: N=1 {t1:.1f} ms ({updates / t1 / 1e6:.0f} GUPS)", flush=True)
    for n in args.ranks:
        plan = SL.plan_slabs(mats, geom.nh, geom.nw, geom.nx, geom.ny, geom.nz, n, align=args.align)
        per = []
        for r in range(n):
            v0, rows = plan.bands[r]
            k0, k1 = plan.slab(r)
            ms = time_slab(img, mats, plan, v0, rows, k0, k1)
            per.append({"rank": r, "slab": [k0, k1], "band": [v0, rows], "ms": ms,
                        "band_bytes": geom.np * rows * SL.pitch_of(geom.nw) * 4})
        mx = max(p["ms"] for p in per)
        eff = t1 / (n * mx)
        out["runs"].append({"n": n, "per_rank": per, "max_ms": mx, "projected_gups": updates / mx / 1e6,
                            "compute_efficiency": eff})
        print(f"  N={n}: max {mx:.1f} ms, per rank " + " ".join(f"{p['ms']:.0f}" for p in per) +
              f"  -> {updates / mx / 1e6:.0f} GUPS, compute-only efficiency {eff:.3f}; band GB/rank " +
              " ".join(f"{p['band_bytes'] / 1e9:.1f}" for p in per), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
