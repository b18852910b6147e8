"""Multi-GPU z-slab driver: one process per GPU, torch.distributed for the plumbing.

The volume is split into contiguous z-slabs with cost-balanced boundaries
(``geometry.slab_plan``); every voxel has one writer
(/root/reference/pkg/src/conebp/_kernels.py:12-14), so no reduction is needed.
Projections start on rank 0 (NATURAL layout, device).  Rank r only ever holds
the detector-row band [v0_r, v0_r + rows_r) its slab samples, one angle chunk
at a time in a double buffer: chunk c+1 is in flight while chunk c is
back-projected (launches take an angle window and accumulate in ascending s,
so chunking does not change a single bit -- the ascending-s chain of
_kernels.py:38,61).

Two band transports:

* ``"ipc"`` (CUDA, one node, the default on GPUs): rank 0 exports its
  projection buffer through CUDA IPC; every other rank *pulls* its band chunks
  with the copy engines (``cbp_copy_band`` = cudaMemcpy3DPeerAsync over
  NVLink/NVSwitch) on a side stream.  Rank 0's SMs never touch another rank's
  data and nothing is staged on rank 0.
* ``"p2p"`` (any torch.distributed backend: NCCL, gloo): rank 0 stages chunk c
  of every rank's band into a per-rank double buffer and ``isend``s it.  This
  is what the CPU tests drive over gloo.

The compute calls go through a backend object, so the same driver runs on CPU
tensors over gloo in the tests (tests/test_multigpu_gloo.py); ``CudaBackend``
is the product.  Band violations are never silent: ``run_slabs`` checks the
device status counters before returning and raises ``CbpError`` (CBP_EBAND).
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

    def active(self, rank: int) -> bool:
        k0, k1 = self.slab(rank)
        return k1 > k0 and self.bands[rank][1] > 0


def plan_slabs(mats: np.ndarray, nh: int, nw: int, nx: int, ny: int, nz: int, n_ranks: int, align: int = 16,
               variant: int = 0) -> SlabPlan:
    kb, bands = G.slab_plan(mats, nh, nw, nx, ny, nz, n_ranks, align=align, variant=variant)
    return SlabPlan(tuple(kb), tuple(bands), int(mats.shape[0]), nh, nw, nx, ny, nz, variant)


def pitch_of(nw: int) -> int:
    return (nw + 3) & ~3


def _chunks(n_proj: int, n_chunks: int) -> list[tuple[int, int]]:
    n_chunks = max(1, min(n_chunks, n_proj))
    return [(n_proj * c // n_chunks, n_proj * (c + 1) // n_chunks) for c in range(n_chunks)]


class CudaBackend:
    """libconebp_b200 on the current CUDA device."""

    def __init__(self, torch):
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.copy_stream = None

    # buffers
    def empty_band(self, n_proj, nw, rows):
        # zeroed once: the pad columns [nw, pitch) are never written by the transports
        return self.torch.zeros((n_proj, rows, pitch_of(nw)), dtype=self.torch.float32, device=self.device)

    def empty_slab(self, plan: SlabPlan, k0, k1):
        return self.torch.zeros((k1 - k0, plan.ny, plan.nx), dtype=self.torch.float32, device=self.device)

    def direct(self, img, plan: SlabPlan):
        """Rank 0 reads the NATURAL stack in place when its rows are 16-byte aligned."""
        return img if plan.nw % 4 == 0 else None

    # transports
    def stage_chunk(self, img, plan: SlabPlan, v0, rows, s0, s1, out):
        """Angles [s0, s1) x rows [v0, v0+rows) of the local stack -> out[:s1-s0] (copy engines)."""
        from .device import copy_band

        copy_band(img.data_ptr(), plan.np, plan.nh, plan.nw, s0, s1, v0, rows, out)

    def ipc_share(self, img, dist):
        from .device import ipc_export

        obj = [ipc_export(img) if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def ipc_open(self, shared):
        from .device import ipc_open

        return ipc_open(*shared)

    def ipc_close(self, ptr, shared):
        from .device import ipc_close

        ipc_close(ptr, shared[1])

    def pull_chunk(self, src_ptr, plan: SlabPlan, v0, rows, s0, s1, out, after):
        """Copy-engine pull of a band chunk on a side stream; returns the event that marks it landed."""
        from .device import copy_band

        torch = self.torch
        if self.copy_stream is None:
            self.copy_stream = torch.cuda.Stream(device=self.device)
        if after is not None:
            self.copy_stream.wait_event(after)
        copy_band(src_ptr, plan.np, plan.nh, plan.nw, s0, s1, v0, rows, out, stream=self.copy_stream)
        ev = torch.cuda.Event()
        ev.record(self.copy_stream)
        return ev

    def wait(self, ev):
        if ev is not None:
            self.torch.cuda.current_stream().wait_event(ev)

    def record(self):
        ev = self.torch.cuda.Event()
        ev.record(self.torch.cuda.current_stream())
        return ev

    # compute
    def compute(self, band, s_base, plan: SlabPlan, v0, rows, k0, k1, s0, s1, mats, vol):
        from .device import backproject_window

        backproject_window(band, s_base, mats, vol, plan.np, plan.nh, plan.nw, v0, rows, plan.nx, plan.ny, k1 - k0,
                           plan.variant, k0=k0, nz_total=plan.nz, s_begin=s0, s_end=s1)

    def check(self):
        from .device import sync_status

        return sync_status()


def _run_p2p(img, mats, plan, backend, dist, chunks, vol):
    """Rank 0 stages and isends chunk c of every band; the others irecv into double buffers."""
    rank, world = dist.get_rank(), dist.get_world_size()
    k0, k1 = plan.slab(rank)
    v0, rows = plan.bands[rank]
    cap = max(s1 - s0 for s0, s1 in chunks)
    if rank == 0:
        dests = [r for r in range(1, world) if plan.active(r)]
        sbuf = {r: [backend.empty_band(cap, plan.nw, plan.bands[r][1]) for _ in range(2)] for r in dests}
        sends = {r: [None, None] for r in dests}
        own = backend.direct(img, plan) if plan.active(0) else None
        obuf = None
        if plan.active(0) and own is None:
            obuf = [backend.empty_band(cap, plan.nw, rows) for _ in range(2)]
        for c, (s0, s1) in enumerate(chunks):
            b = c & 1
            for r in dests:
                if sends[r][b] is not None:
                    sends[r][b].wait()  # chunk c-2 left this buffer
                rv0, rrows = plan.bands[r]
                backend.stage_chunk(img, plan, rv0, rrows, s0, s1, sbuf[r][b])
                sends[r][b] = dist.isend(sbuf[r][b][: s1 - s0], dst=r)
            if own is not None:
                backend.compute(own, 0, plan, 0, plan.nh, k0, k1, s0, s1, mats, vol)
            elif obuf is not None:
                backend.stage_chunk(img, plan, v0, rows, s0, s1, obuf[b])
                backend.compute(obuf[b], s0, plan, v0, rows, k0, k1, s0, s1, mats, vol)
        for r in dests:
            for w in sends[r]:
                if w is not None:
                    w.wait()
        return
    if not plan.active(rank):
        return
    rbuf = [backend.empty_band(cap, plan.nw, rows) for _ in range(2)]
    recvs = [None] * len(chunks)
    for c in range(min(2, len(chunks))):
        s0, s1 = chunks[c]
        recvs[c] = dist.irecv(rbuf[c & 1][: s1 - s0], src=0)
    for c, (s0, s1) in enumerate(chunks):
        recvs[c].wait()
        backend.compute(rbuf[c & 1], s0, plan, v0, rows, k0, k1, s0, s1, mats, vol)
        if c + 2 < len(chunks):  # the buffer is reused after this compute (stream-ordered on GPUs)
            n0, n1 = chunks[c + 2]
            recvs[c + 2] = dist.irecv(rbuf[c & 1][: n1 - n0], src=0)


def _run_ipc(img, mats, plan, backend, dist, chunks, vol, shared):
    """Every rank pulls its own band chunks from rank 0's memory with the copy engines."""
    rank = dist.get_rank()
    k0, k1 = plan.slab(rank)
    v0, rows = plan.bands[rank]
    if not plan.active(rank):
        return
    if rank == 0 and backend.direct(img, plan) is not None:
        for s0, s1 in chunks:
            backend.compute(img, 0, plan, 0, plan.nh, k0, k1, s0, s1, mats, vol)
        return
    src = img.data_ptr() if rank == 0 else backend.ipc_open(shared)
    try:
        cap = max(s1 - s0 for s0, s1 in chunks)
        buf = [backend.empty_band(cap, plan.nw, rows) for _ in range(2)]
        done = [None, None]
        landed = [None] * len(chunks)
        for c in range(min(2, len(chunks))):
            s0, s1 = chunks[c]
            landed[c] = backend.pull_chunk(src, plan, v0, rows, s0, s1, buf[c & 1], None)
        for c, (s0, s1) in enumerate(chunks):
            backend.wait(landed[c])
            backend.compute(buf[c & 1], s0, plan, v0, rows, k0, k1, s0, s1, mats, vol)
            done[c & 1] = backend.record()
            if c + 2 < len(chunks):  # the next pull into this buffer waits for this compute
                n0, n1 = chunks[c + 2]
                landed[c + 2] = backend.pull_chunk(src, plan, v0, rows, n0, n1, buf[c & 1], done[c & 1])
    finally:
        if rank != 0:
            # the mapping must outlive the copies that read it
            backend.torch.cuda.synchronize()
            backend.ipc_close(src, shared)


def run_slabs(img, mats: np.ndarray, plan: SlabPlan, backend, dist, n_chunks: int = 4, vol=None,
              transport: str = "p2p", shared=None, check: bool = True):
    """Move bands from rank 0 and back-project this rank's slab (accumulating into ``vol``).

    ``img`` is the NATURAL projection stack on rank 0 (ignored elsewhere).  With
    ``transport="ipc"``, ``shared`` is ``backend.ipc_share(img, dist)`` (collective; do it
    once, outside any timed region).  Returns this rank's slab [k1-k0][ny][nx].  Raises on
    samples outside the band when ``check`` (synchronises the rank's device).
    """
    rank, world = dist.get_rank(), dist.get_world_size()
    if len(plan.k_bounds) != world + 1:
        raise ValueError("the slab plan is for a different number of ranks")
    k0, k1 = plan.slab(rank)
    if vol is None:
        vol = backend.empty_slab(plan, k0, k1)
    chunks = _chunks(plan.np, n_chunks)
    if transport == "ipc":
        if shared is None:
            raise ValueError('transport="ipc" needs shared=backend.ipc_share(img, dist)')
        _run_ipc(img, mats, plan, backend, dist, chunks, vol, shared)
    elif transport == "p2p":
        _run_p2p(img, mats, plan, backend, dist, chunks, vol)
    else:
        raise ValueError(f"unknown band transport {transport!r}")
    if check:
        backend.check()
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
