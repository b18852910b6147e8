"""Loopback harness for the multi-rank z-slab driver on ONE GPU (test infrastructure).

``run_loopback`` drives the product driver ``slabs.run_slabs`` with the real
``CudaBackend`` for every rank of an N-rank plan, one rank after another in
this process, all on the current GPU.  ``LoopbackDist`` stands in for
torch.distributed: ``isend`` deposits a device copy of the chunk in a mailbox
and ``irecv`` takes it out (rank 0 runs first, so every message a rank waits
for has been sent), ``broadcast_object_list`` hands rank 0's object to the
others.  For the IPC transport, ``LoopbackBackend`` maps "rank 0's buffer" to
the local pointer (a process cannot open its own IPC handle); everything else --
the copy-engine band pulls, the angle-window launches on double buffers, the
slab offsets k0 / nz_total, the band status check -- is the product code path.

Ranks never wait on one another's kernels here (each rank's work is complete
before the next starts), so nothing depends on concurrent GPUs; this is a
correctness harness, not a timing one.
"""

from __future__ import annotations

from collections import defaultdict, deque

from paper_2104_13248_b200 import slabs


class _Done:
    def wait(self):
        return None


class LoopbackDist:
    def __init__(self, world: int):
        self.world = world
        self.rank = 0
        self.mail = defaultdict(deque)
        self.objects = None
        self.sent_bytes = 0

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.world

    def isend(self, t, dst):
        self.mail[(self.rank, dst)].append(t.clone())
        self.sent_bytes += t.numel() * t.element_size()
        return _Done()

    def irecv(self, t, src):
        t.copy_(self.mail[(src, self.rank)].popleft())
        return _Done()

    def broadcast_object_list(self, obj, src=0):
        if self.rank == src:
            self.objects = list(obj)
        else:
            obj[:] = self.objects


class LoopbackBackend(slabs.CudaBackend):
    def ipc_share(self, img, dist):
        return ("loopback", 0) if dist.get_rank() == 0 else None

    def ipc_open(self, shared):
        return self._img_ptr

    def ipc_close(self, ptr, shared):
        return None


def run_loopback(torch, img, mats, plan, n_chunks=4, transport="p2p"):
    """Run every rank of ``plan`` in turn; returns the list of slab tensors (rank order)."""
    world = len(plan.k_bounds) - 1
    dist = LoopbackDist(world)
    backend = LoopbackBackend(torch)
    backend._img_ptr = img.data_ptr()
    shared = None
    out = []
    for r in range(world):
        dist.rank = r
        if transport == "ipc":
            obj = [backend.ipc_share(img, dist) if r == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            shared = obj[0]
        vol = slabs.run_slabs(img if r == 0 else None, mats, plan, backend, dist, n_chunks=n_chunks,
                              transport=transport, shared=shared)
        out.append(vol)
    torch.cuda.synchronize()
    return out, dist
