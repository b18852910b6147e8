"""Multi-GPU z-slab driver: one process per GPU, torch.distributed (NCCL) plumbing.

The volume is split into contiguous z-slabs with cost-balanced boundaries
(``geometry.slab_plan``); every voxel has one writer, so no
reduction is needed.  Projections start on rank 0 (NATURAL layout, device);
rank r receives only the detector-row band [v0_r, v0_r + rows_r) its slab
samples, already in the staging layout [s][r][u], in angle chunks: chunk c+1
is in flight over NVLink while chunk c is back-projected (the kernel takes an
angle range and accumulates in ascending s, so chunking does not change a
single bit of the result).

The compute/staging calls go through a small backend object so the same
driver logic runs on CPU tensors over gloo in the tests (tests/
test_multigpu_gloo.py injects a CPU backend); the default backend is the
CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import geometry as G

__all__ = ["SlabPlan", "plan_slabs", "CudaBackend", "run_slabs", "gather_volume"]


@dataclass(frozen=True)
class SlabPlan:
    k_bounds: tuple      # n_ranks + 1 slice boundaries
    bands: tuple         # (v0, rows) per rank; rows == 0: slab samples nothing
    np: int
    nh: int
    nw: int
    nx: int
    ny: int
    nz: int
    variant: int = 0

    def slab(self, rank: int) -> tuple[int, int]:
        return self.k_bounds[rank], self.k_bounds[rank + 1]


def plan_slabs(mats: np.ndarray, nh: int, nw: int, nx: int, ny: int, nz: int, n_ranks: int, align: int = 32,
               variant: int = 0) -> SlabPlan:
    kb, bands = G.slab_plan(mats, nh, nw, nx, ny, nz, n_ranks, align=align, variant=variant)
    return SlabPlan(tuple(kb), tuple(bands), int(mats.shape[0]), nh, nw, nx, ny, nz, variant)


def pitch_of(nw: int) -> int:
    return (nw + 3) & ~3


class CudaBackend:
    """libconebp_b200 on the current CUDA device."""

    def __init__(self, torch):
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())

    def empty_band(self, n_proj, nw, rows):
        return self.torch.empty((n_proj, rows, pitch_of(nw)), dtype=self.torch.float32, device=self.device)

    def stage_band(self, img, plan: SlabPlan, v0, rows, out):
        from . import _lib
        from .device import stream_handle

        _lib.check(_lib.lib().cbp_stage_projections(img.data_ptr(), _lib.NATURAL, plan.np, plan.nh, plan.nw, v0, rows,
                                                    out.data_ptr(), out.shape[2], stream_handle()))

    def empty_slab(self, plan: SlabPlan, k0, k1):
        return self.torch.zeros((k1 - k0, plan.ny, plan.nx), dtype=self.torch.float32, device=self.device)

    def compute(self, band, plan: SlabPlan, v0, rows, k0, k1, s0, s1, mats, vol):
        from .device import StagedProjections, backproject_staged

        staged = StagedProjections.wrap(band, plan.np, plan.nh, plan.nw, v0, rows)
        backproject_staged(staged, mats, vol, plan.nx, plan.ny, k1 - k0, plan.variant, k0=k0, nz_total=plan.nz,
                           s_begin=s0, s_end=s1)


def _chunks(n_proj: int, n_chunks: int) -> list[tuple[int, int]]:
    n_chunks = max(1, min(n_chunks, n_proj))
    return [(n_proj * c // n_chunks, n_proj * (c + 1) // n_chunks) for c in range(n_chunks)]


def run_slabs(img, mats: np.ndarray, plan: SlabPlan, backend, dist, n_chunks: int = 4, vol=None):
    """Distribute bands from rank 0 and back-project this rank's slab.

    ``img`` is the NATURAL projection stack on rank 0 (ignored elsewhere).
    Returns this rank's slab volume [k1-k0][ny][nx] (accumulated into ``vol``
    when given).
    """
    rank, world = dist.get_rank(), dist.get_world_size()
    assert len(plan.k_bounds) == world + 1
    k0, k1 = plan.slab(rank)
    v0, rows = plan.bands[rank]
    if vol is None:
        vol = backend.empty_slab(plan, k0, k1)
    chunks = _chunks(plan.np, n_chunks)
    my_band = None
    if rows > 0 and k1 > k0:
        my_band = backend.empty_band(plan.np, plan.nw, rows)
    reqs = []
    if rank == 0:
        sends = []
        for r in range(1, world):
            rv0, rrows = plan.bands[r]
            if rrows == 0 or plan.k_bounds[r + 1] == plan.k_bounds[r]:
                continue
            buf = backend.empty_band(plan.np, plan.nw, rrows)
            backend.stage_band(img, plan, rv0, rrows, buf)
            sends.append((r, buf))
        if my_band is not None:
            backend.stage_band(img, plan, v0, rows, my_band)
        # angle-chunked sends: every rank's chunk c before any chunk c+1
        for s0, s1 in chunks:
            for r, buf in sends:
                reqs.append(dist.isend(buf[s0:s1], dst=r))
        recv_works = [None] * len(chunks)
    else:
        recv_works = []
        if my_band is not None:
            for s0, s1 in chunks:
                recv_works.append(dist.irecv(my_band[s0:s1], src=0))
        else:
            recv_works = [None] * len(chunks)
    if my_band is not None:
        for c, (s0, s1) in enumerate(chunks):
            if recv_works[c] is not None:
                recv_works[c].wait()
            backend.compute(my_band, plan, v0, rows, k0, k1, s0, s1, mats, vol)
    for w in reqs:
        w.wait()
    return vol


def gather_volume(vol_slab, plan: SlabPlan, dist, torch):
    """Validation only: collect every slab on rank 0 as one (nz, ny, nx) tensor."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank == 0:
        full = torch.empty((plan.nz, plan.ny, plan.nx), dtype=vol_slab.dtype, device=vol_slab.device)
        k0, k1 = plan.slab(0)
        full[k0:k1] = vol_slab
        for r in range(1, world):
            a, b = plan.slab(r)
            if b > a:
                dist.recv(full[a:b], src=r)
        return full
    k0, k1 = plan.slab(rank)
    if k1 > k0:
        dist.send(vol_slab.contiguous(), dst=0)
    return None
