"""Shared-memory bank-conflict model of the tiled kernel's texel gathers (CPU, numpy).

For sampled (tile, angle) pairs of a config, computes each lane's texel (ix, iy) per
slice with float32 arithmetic (reference op order is irrelevant here), the box
origin as the kernel does, and the wavefronts each warp-wide LDS.32 needs under a
candidate box row pitch / warp shape: wavefronts = max over banks of the number of
distinct words addressed in that bank.

    python tools/bank_sim.py --config 1 [--tiles 64 --angles 24]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2104_13248_b200.configs import get_config  # noqa: E402


def lane_coords(m, i, j, k):
    z = m[2, 0] * i + m[2, 1] * j + m[2, 2] * k + m[2, 3]
    f = 1.0 / z
    x = (m[0, 0] * i + m[0, 1] * j + m[0, 2] * k + m[0, 3]) * f
    y = (m[1, 0] * i + m[1, 1] * j + m[1, 2] * k + m[1, 3]) * f
    return x, y


def wavefronts(words):
    """words: (..., 32) int array of word addresses -> (...) wavefront count"""
    banks = words & 31
    out = np.zeros(words.shape[:-1], np.int64)
    flat_w = words.reshape(-1, 32)
    flat_b = banks.reshape(-1, 32)
    res = np.empty(flat_w.shape[0], np.int64)
    for r in range(flat_w.shape[0]):
        best = 1
        for b in np.unique(flat_b[r]):
            n = len(np.unique(flat_w[r][flat_b[r] == b]))
            best = max(best, n)
        res[r] = best
    return res.reshape(out.shape)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--tiles", type=int, default=48)
    ap.add_argument("--angles", type=int, default=16)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--transposed", action="store_true", help="box stored [u][v] (v contiguous)")
    ap.add_argument("--shapes", default="8x4,4x8,16x2")
    args = ap.parse_args()
    spec = get_config(args.config)
    geom = spec.geometry()
    mats = spec.matrices(geom).astype(np.float64).reshape(-1, 3, 4)
    nx, ny, nz, nw, nh = geom.nx, geom.ny, geom.nz, geom.nw, geom.nh
    rng = np.random.default_rng(args.seed)
    shapes = {sh: tuple(int(t) for t in sh.split("x")) for sh in args.shapes.split(",")}
    pitches = list(range(0, 32, 4)) + [2, 6, 10, 14, 18, 22, 26, 30, 1, 3, 5, 7, 9, 11, 13, 15, 17]
    res = {(sh, p): [0, 0] for sh in shapes for p in pitches}
    for _ in range(args.tiles):
        bx, by, bz = rng.integers(0, nx // 32), rng.integers(0, ny // 16), rng.integers(0, nz // 32)
        i0, j0, k0 = bx * 32, by * 16, bz * 32
        for s in rng.integers(0, mats.shape[0], args.angles):
            m = mats[s]
            for sh, (wx, wy) in shapes.items():
                # one warp at a random place in the tile
                ox = rng.integers(0, 32 // wx) * wx if wx <= 32 else 0
                oy = rng.integers(0, max(1, 16 // wy)) * wy
                li = np.arange(32) % wx
                lj = np.arange(32) // wx
                ii = (i0 + ox + li)[None, :].astype(np.float64)
                jj = (j0 + oy + lj)[None, :].astype(np.float64)
                kk = (k0 + np.arange(32))[:, None].astype(np.float64)
                x, y = lane_coords(m, ii, jj, kk)
                ok = (x >= 0) & (x < nw - 1) & (y >= 0) & (y < nh - 1)
                if not ok.all():
                    continue
                ix = np.floor(x).astype(np.int64)
                iy = np.floor(y).astype(np.int64)
                u0 = ix.min() & ~3
                v0 = iy.min()
                for p in pitches:
                    W = 96 + p + 32  # any base multiple of 32 plus the residue
                    base = (ix - u0) * W + (iy - v0) if args.transposed else (iy - v0) * W + (ix - u0)
                    wf = 0
                    for off in (0, 1, W, W + 1):
                        wf += wavefronts(base + off).sum()
                    res[(sh, p)][0] += wf
                    res[(sh, p)][1] += 4 * base.shape[0]
    print(f"config {args.config}: wavefronts per LDS.32 (1.00 = conflict free)")
    for sh in shapes:
        row = " ".join(f"{p}:{res[(sh, p)][0] / max(1, res[(sh, p)][1]):.3f}" for p in pitches)
        print(f"{sh:5s} {row}")


if __name__ == "__main__":
    main()
