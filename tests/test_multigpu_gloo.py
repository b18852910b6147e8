"""Multi-rank z-slab driver on CPU: torch.distributed gloo, world size 2 and 3.

The product driver (paper_2104_13248_b200/slabs.py: cost-balanced slabs, per-rank
detector-row bands sent from rank 0 in angle chunks, chunked accumulation) runs
unchanged; only its compute backend is swapped for the CPU oracle (test
infrastructure).  The gathered volume must equal the single-process reference
result bit for bit, and no rank may sample a row outside its band.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleBackend:
    """CPU stand-in for slabs.CudaBackend (same interface, p2p transport)."""

    def __init__(self, torch):
        self.torch = torch
        self.violations = 0

    def empty_band(self, n_proj, nw, rows):
        from paper_2104_13248_b200.slabs import pitch_of

        return self.torch.zeros((n_proj, rows, pitch_of(nw)), dtype=self.torch.float32)

    def empty_slab(self, plan, k0, k1):
        return self.torch.zeros((k1 - k0, plan.ny, plan.nx), dtype=self.torch.float32)

    def direct(self, img, plan):
        return img if plan.nw % 4 == 0 else None

    def stage_chunk(self, img, plan, v0, rows, s0, s1, out):
        out[: s1 - s0, :, : plan.nw] = img[s0:s1, v0:v0 + rows, :]

    def compute(self, band, s_base, plan, v0, rows, k0, k1, s0, s1, mats, vol):
        import oracle

        img = np.ascontiguousarray(band[s0 - s_base:s1 - s_base, :, : plan.nw].numpy())
        self.violations += oracle.baseline(img, mats[s0:s1], vol.numpy(), threads=1, nh=plan.nh, v0=v0, k_lo=k0)

    def check(self):
        if self.violations:
            raise RuntimeError(f"{self.violations} samples outside the band")


def worker(rank, world, port, case, n_chunks, result_q):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "oracle"))
    sys.path.insert(0, str(REPO / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from conftest import load_golden
    from paper_2104_13248_b200 import slabs

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden(case)
        img, mats = g["img"], g["mats"]
        n_proj, nh, nw = img.shape
        nz, ny, nx = g["vol0"].shape
        plan = slabs.plan_slabs(mats, nh, nw, nx, ny, nz, world, align=2)
        backend = OracleBackend(torch)
        k0, k1 = plan.slab(rank)
        vol = torch.from_numpy(g["vol0"][k0:k1].copy())
        slabs.run_slabs(torch.from_numpy(img) if rank == 0 else None, mats, plan, backend, dist, n_chunks=n_chunks,
                        vol=vol)
        full = slabs.gather_volume(vol, plan, dist, torch)
        if rank == 0:
            result_q.put(("ok", full.numpy().tobytes() == g["baseline"].tobytes(), backend.violations,
                          list(plan.k_bounds), list(plan.bands)))
        else:
            result_q.put(("rank", rank, backend.violations))
    except Exception as exc:  # pragma: no cover - surfaced through the queue
        result_q.put(("error", rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case,n_chunks", [(2, "uoffset", 3), (3, "tilted", 2), (2, "ragged", 4)])
def test_zslab_driver_over_gloo_is_bitwise(world, case, n_chunks):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, case, n_chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errors = [r for r in results if r[0] == "error"]
    assert not errors, errors
    head = [r for r in results if r[0] == "ok"][0]
    _, bitwise, viol0, k_bounds, bands = head
    assert bitwise, f"gathered slabs differ from the reference (k_bounds {k_bounds}, bands {bands})"
    assert viol0 == 0 and all(r[2] == 0 for r in results if r[0] == "rank")
