"""Benchmark: FDK cone-beam back-projection GUPS on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workload: BASELINE.json configs[1] by default (256^3 volume from 360 filtered
projections of 512x512); ``--config`` selects another.  A step is one pass of
the hot path over the whole workload: re-lay the projections into the staging
layout and back-project every angle into the volume (zeroed at step start).

* ``value``  GUPS (nx*ny*nz*np / step time / 1e9) with inputs resident in HBM,
             CUDA events on the launch stream, max over ranks.  The projections
             (360 MiB for config 1) exceed the 126 MB L2, so no flush is needed.
* ``e2e``    the same metric through the public numpy API (pinned host buffers:
             H2D of projections + volume, kernels, D2H of the volume every step).
* ``roofline`` the back-projection kernel's algorithmic gather bytes (16 B per
             update) per launch / its CUDA-event duration vs the
             L1/shared gather peak 128 B/clk/SM x SMs x the SM clock measured
             during the run; the FP32 and HBM rooflines ride along.
* ``cpu_baseline`` the C oracle port (oracle/, a bit-exact restatement of the
             reference kernel) on this host's cores over a bounded z-slab sample.

N > 1 (torchrun, NCCL): the volume is z-slab partitioned with cost-balanced
boundaries; rank 0 holds the projections and sends each rank its detector-row
band in angle chunks over NVLink inside the timed region (strong scaling).
``--impl reference`` times the reference algorithm on the host cores (the C
port, all threads) on the same config and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "GUPS (voxel*projection updates/s)"
GATHER_BYTES_PER_UPDATE = 16.0      # 4 float32 texels per bilinear sample
FP32_OPS_FAST = 16.0                # FP32 lane ops per update executed by the fast hot loop: y 3, frac 1,
                                    # blend 10, accumulate 2 (SASS: 16 FADD2/FMUL2 per slice pair)
FP32_OPS_GENERAL = 27.0             # general matrices (jitter)
LDS_BYTES_PER_CLK_SM = 128.0


def ncu_traffic(workload: str):
    p = REPO / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(p.read_text()).get(workload, {}).get("dram_bytes")
    except (OSError, ValueError):
        return None


def measured_peaks() -> dict:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            pass
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~2 ms during the timed region."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._thr = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
            self.max_mhz = None

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nvml is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=5)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["clock sampling unavailable"],
                    "samples": 0}
        sm = [a for a, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "NVML every ~2 ms during the timed region"}


def cpu_sample_gups(spec, geom, mats, img_np, target_s: float = 12.0) -> dict:
    """C-oracle GUPS on this host's cores over a bounded full-width z-slab sample."""
    sys.path.insert(0, str(REPO / "oracle"))
    import oracle

    threads = oracle.default_threads()
    nx, ny, nz = geom.nx, geom.ny, geom.nz
    # calibrate on a thin slab around the centre, then size the sample for ~target_s
    k_mid = nz // 2
    nk = max(1, min(nz, 2))
    vol = np.zeros((nk, ny, nx), np.float32)
    t0 = time.perf_counter()
    oracle.baseline(img_np, mats, vol, threads=threads, k_lo=k_mid)
    dt = time.perf_counter() - t0
    rate = nk * nx * ny * geom.np / max(dt, 1e-6)
    nk = int(max(1, min(nz, rate * target_s / (nx * ny * geom.np))))
    k_lo = max(0, k_mid - nk // 2)
    vol = np.zeros((nk, ny, nx), np.float32)
    t0 = time.perf_counter()
    oracle.baseline(img_np, mats, vol, threads=threads, k_lo=k_lo)
    dt = time.perf_counter() - t0
    ups = nk * nx * ny * geom.np
    out = {"value": ups / dt / 1e9, "unit": "GUPS", "cores": threads, "kind": "port",
           "sample": f"z-slab k=[{k_lo},{k_lo + nk}) of {nz} (full x,y, all {geom.np} angles), {dt:.1f} s, "
                     f"C oracle (bit-exact restatement of _kernels.baseline), {threads} threads"}
    # context: the paper's fastest CPU rung, subline_prefetch with the largest
    # nb <= 32 dividing np, on the full volume when it is small enough to finish in seconds
    nb = max(b for b in range(1, 33) if geom.np % b == 0)
    if nz % 2 == 0 and nx * ny * nz * geom.np <= 2e10:
        img_t = np.ascontiguousarray(img_np.transpose(0, 2, 1))
        vol_t = np.zeros((nx, ny, nz), np.float32)
        t0 = time.perf_counter()
        oracle.rung(5, img_t, mats, vol_t, nb, threads=threads)
        dt = time.perf_counter() - t0
        out["context"] = {"subline_prefetch": {"value": nx * ny * nz * geom.np / dt / 1e9, "unit": "GUPS", "nb": nb,
                                               "sample": f"full volume, {dt:.1f} s, C restatement of "
                                                         f"_kernels.subline_prefetch, {threads} threads; "
                                                         f"not parity-valid (SURVEY F2), context only"}}
    return out


def run_reference(args, spec, geom, mats) -> None:
    """--impl reference: the reference algorithm (C port) on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    img_np = spec.projections_host(geom)
    sys.path.insert(0, str(REPO / "oracle"))
    import oracle

    threads = oracle.default_threads()
    nx, ny, nz = geom.nx, geom.ny, geom.nz
    per_slice = nx * ny * geom.np
    # bounded sample per step: slices sized for ~2 s of CPU work
    vol = np.zeros((2, ny, nx), np.float32)
    t0 = time.perf_counter()
    oracle.baseline(img_np, mats, vol, threads=threads, k_lo=nz // 2)
    rate = 2 * per_slice / max(time.perf_counter() - t0, 1e-6)
    nk = int(max(1, min(nz, rate * 2.0 / per_slice)))
    k_lo = max(0, nz // 2 - nk // 2)
    times = []
    for it in range(args.warmup + args.steps):
        vol = np.zeros((nk, ny, nx), np.float32)
        t0 = time.perf_counter()
        oracle.baseline(img_np, mats, vol, threads=threads, k_lo=k_lo)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    tot = sum(times)
    value = nk * per_slice * len(times) / tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GUPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": spec.inputs + " (synthetic, seeded)", "config": spec.describe() | {"sample_slices": nk},
            "cpu_baseline": {"value": value, "unit": "GUPS", "cores": threads, "kind": "port",
                             "sample": f"per step: z-slab k=[{k_lo},{k_lo + nk}) of {nz}, full x,y, all {geom.np} "
                                       f"angles; C oracle = bit-exact restatement of conebp._kernels.baseline"},
            "e2e": {"value": value, "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="baseline")
    ap.add_argument("--flags", type=int, default=0, help="library flags (1 naive, 2 no smem staging)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--chunks", type=int, default=4)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2104_13248_b200 import KernelVariant, configs

    spec = configs.get_config(args.config)
    geom = spec.geometry()
    mats = spec.matrices(geom)
    if args.impl == "reference":
        run_reference(args, spec, geom, mats)
        return

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2104_13248_b200 import _lib
    from paper_2104_13248_b200 import device as D
    from paper_2104_13248_b200 import slabs as SL

    variant = KernelVariant.parse(args.variant)
    nx, ny, nz, n_proj, nh, nw = geom.nx, geom.ny, geom.nz, geom.np, geom.nh, geom.nw
    updates = nx * ny * nz * n_proj
    stream = torch.cuda.current_stream()
    img_dev = spec.projections_device(geom, device="cuda") if rank == 0 else None
    torch.cuda.synchronize()

    kern_ms = []
    if world == 1:
        # one step = the library call on device-resident buffers: projections in the
        # reference's NATURAL layout are already the staging layout when nw % 4 == 0,
        # so the step is exactly one back-projection kernel (else one staging kernel too)
        vol = torch.zeros((nz, ny, nx), dtype=torch.float32, device="cuda")
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

        def step(i=None):
            if i is not None:
                ev[i][0].record(stream)
            D.backproject_device(img_dev, mats, vol, n_proj, nh, nw, nx, ny, nz, variant, flags=args.flags)
            if i is not None:
                ev[i][1].record(stream)

        launches_per_step = 1 if nw % 4 == 0 else 2
    else:
        plan = SL.plan_slabs(mats, nh, nw, nx, ny, nz, world, align=32, variant=int(variant))
        backend = SL.CudaBackend(torch)
        k0, k1 = plan.slab(rank)
        vol = backend.empty_slab(plan, k0, k1)

        def step(i=None):
            SL.run_slabs(img_dev, mats, plan, backend, dist, n_chunks=args.chunks, vol=vol)

        launches_per_step = args.chunks + (world if rank == 0 else 0)

    for _ in range(args.warmup):
        step()
    stats_warm = D.sync_status()
    plan_info = D.last_plan()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        t_start.record(stream)
        for i in range(args.steps):
            step(i if world == 1 else None)
        t_end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    if world == 1:
        kern_ms = [a.elapsed_time(b) for a, b in ev]
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    stats = D.sync_status()
    ms_per_step = total_ms / args.steps
    value = updates / (ms_per_step * 1e-3) / 1e9
    clocks = sampler.summary()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peaks = measured_peaks()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    f_mhz = clocks["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    line = {"metric": METRIC, "value": value, "unit": "GUPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic: {spec.inputs} inputs (seeded); projections {n_proj * nh * nw * 4 / 2**20:.0f} MiB "
                    f"(> 126 MB L2, no flush needed)",
            "config": spec.describe() | {"variant": variant.name.lower(), "parallelism": f"zslab{world}",
                                         "l2": "inputs larger than L2 (no flush)"},
            "clocks": clocks, "gpu_launches": launches_per_step * args.steps}
    if kern_ms:
        k_avg = statistics.mean(kern_ms)
        gath = GATHER_BYTES_PER_UPDATE * updates / (k_avg * 1e-3) / 1e9
        peak = LDS_BYTES_PER_CLK_SM * sms * f_mhz * 1e6 / 1e9
        general = not __import__("paper_2104_13248_b200.geometry", fromlist=["x"]).has_vertical_columns(mats) \
            and variant < KernelVariant.SHARE
        fp_ops = FP32_OPS_GENERAL if general else FP32_OPS_FAST
        fp_peak_gups = 128.0 * sms * f_mhz * 1e6 / fp_ops / 1e9
        gups_k = updates / (k_avg * 1e-3) / 1e9
        comp_bytes = 8.0 * nx * ny * nz + 4.0 * n_proj * nh * nw  # volume RMW once + each texel once
        line["roofline"] = {
            "bound": "gather", "unit": "GB/s", "achieved": gath, "peak": peak, "frac": gath / peak,
            "traffic": ncu_traffic(spec.name),
            "traffic_note": "DRAM read+write bytes per launch from a committed ncu --set full capture "
                            "(profiles/ncu_traffic.json); the gather roofline's algorithmic bytes are L1/shared "
                            "bytes, so DRAM traffic is shown for the HBM side",
            "peak_basis": f"128 B/clk/SM x {sms} SMs x {f_mhz:.0f} MHz (SM clock measured during run); "
                          f"algorithmic 16 B/update",
            "kernel_ms": k_avg, "kernel_gups": gups_k,
            "fp32": {"ops_per_update": fp_ops, "peak_gups": fp_peak_gups, "frac": gups_k / fp_peak_gups},
            "hbm": {"compulsory_bytes": comp_bytes, "achieved_gbs": comp_bytes / (k_avg * 1e-3) / 1e9,
                    "peak_gbs": peaks.get("hbm_gbs")},
            "kernel_share_of_step": k_avg / ms_per_step,
        }
    line["plan"] = plan_info
    line["tile_stats"] = stats_warm

    if not args.no_e2e and world == 1:
        line["e2e"] = e2e_leg(torch, spec, geom, mats, img_dev, variant, args)
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_sample_gups(spec, geom, mats, img_dev.cpu().numpy())
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def e2e_leg(torch, spec, geom, mats, img_dev, variant, args) -> dict:
    """Same metric through the public numpy API with pinned host buffers."""
    from paper_2104_13248_b200 import Layout, ProjectionStack, Volume, backproject_baseline, backproject_optimized

    nx, ny, nz, n_proj, nh, nw = geom.nx, geom.ny, geom.nz, geom.np, geom.nh, geom.nw
    img_pin = torch.empty((n_proj, nh, nw), dtype=torch.float32, pin_memory=True)
    img_pin.copy_(img_dev)
    vol_pin = torch.zeros((nz, ny, nx), dtype=torch.float32, pin_memory=True)
    proj = ProjectionStack(img_pin.numpy(), n_proj, nh, nw, Layout.NATURAL)
    vol = Volume(vol_pin.numpy(), nx, ny, nz, Layout.NATURAL)
    assert proj.data.ctypes.data == img_pin.data_ptr() and vol.data.ctypes.data == vol_pin.data_ptr()

    def step():  # the user's call: accumulate into the caller's (pinned) volume
        backproject_baseline(proj, mats, vol)

    for _ in range(max(1, args.warmup)):
        step()
    n = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    dt = (time.perf_counter() - t0) / n
    return {"value": nx * ny * nz * n_proj / dt / 1e9, "unit": "GUPS",
            "h2d_bytes_per_step": 4 * (n_proj * nh * nw + nx * ny * nz), "d2h_bytes_per_step": 4 * nx * ny * nz,
            "ms_per_step": dt * 1e3, "api": "paper_2104_13248_b200.backproject_baseline (numpy, pinned)"}


if __name__ == "__main__":
    main()
