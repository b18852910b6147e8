"""Benchmark: FDK cone-beam back-projection GUPS on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Workload: BASELINE.json configs[4] by default (2048^3 volume from 2048
projections of 2048x2048 with a +16 px u offset; 32 GiB + 32 GiB, the largest
configuration, which fits one B200); ``--config`` selects another.  A step is
one pass of the hot path over the whole workload: one library call that
back-projects every angle into the (resident) volume.  The NATURAL projections
with nw % 4 == 0 already are the staging layout, so a step is exactly one
kernel launch (a staging kernel too when nw % 4 != 0); the volume accumulates
across steps, as the reference's ``+=`` does.

* ``value``  GUPS (nx*ny*nz*np / step time / 1e9, every voxel-angle pair counted,
             guard-skipped ones included, as /root/reference/pkg/src/conebp/
             bench.py:150-154), inputs resident in HBM, CUDA events on the launch
             stream, max over ranks.  Inputs (>= 360 MiB) exceed the 126 MB L2.
* ``e2e``    the same metric through the public numpy API (``backproject_baseline``
             on pinned host buffers: H2D of projections + volume, kernels, D2H of
             the volume inside every step).
* ``roofline`` the back-projection kernel against the L1/shared gather roofline
             (16 algorithmic bytes per update; 128 B/clk/SM x SMs x
             the SM clock measured during the run).  ``achieved``/``frac`` use the
             reference-defined update count; ``executed`` uses the updates the kernel
             actually runs (queued tile-angle pairs x tile voxels, from the device
             counters) -- tiles whose footprint misses the detector are never queued
             (the reference's guard rejects every voxel of them), so on configs 3-4
             the reference count exceeds what any kernel must execute.
* ``cpu_baseline`` the live reference (``conebp.backproject_baseline`` from
             baseline/_ref, numba, all host threads) on a bounded sample of the same
             workload; the C port (oracle/) if the reference cannot be imported.

``--impl reference`` times the reference's own CPU implementation (the live numba
kernel, all host cores) on the same config: per step a stratified sample of z-slices
evenly spaced over the whole volume (the full volume on configs 0-1).

N > 1 (torchrun, one process per GPU): the volume is z-slab partitioned with
cost-balanced boundaries; rank 0 holds the projections and every other rank pulls
its detector-row band in angle chunks with the copy engines over NVLink (CUDA IPC,
no SM work on rank 0), inside the timed region (strong scaling).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "GUPS (voxel*projection updates/s)"
GATHER_BYTES_PER_UPDATE = 16.0      # 4 float32 texels per bilinear sample
FP32_OPS_FAST = 16.0                # FP32 lane ops per update executed by the exact fast hot loop (SURVEY's
                                    # algorithmic count is 13 with FMA lerps; the reference's separately rounded
                                    # ops are y 3, frac 1, 1-ay 1, lerps 9, weight+accumulate 2)
FP32_OPS_GENERAL = 27.0             # general matrices (jitter), SURVEY.md 8(d)
LDS_BYTES_PER_CLK_SM = 128.0
REF_PATH = REPO / "baseline" / "_ref"


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


# ------------------------------------------------------------------ the reference on the host cores
def import_reference():
    """The live reference package (pip-installed into baseline/_ref), numba threads = all host cores."""
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/conebp_numba_cache")
    if not (REF_PATH / "conebp").is_dir():
        raise ImportError(f"{REF_PATH} has no reference install")
    if str(REF_PATH) not in sys.path:
        sys.path.insert(0, str(REF_PATH))
    import conebp  # noqa: F401
    import numba

    return conebp, numba


def reference_sample(geom, mats: np.ndarray, n_threads: int, full_limit: float = 2e10):
    """A stratified z-slice sample the reference times in a few seconds: the full volume when
    U <= full_limit, else ``n_slices`` slices evenly spaced over z (a multiple of the thread
    count: the reference parallelises over slices, _kernels.py:42).  Evenly spaced slices are
    an affine relabelling of k, fed to the unmodified reference as a thin volume with matrices
    m[:, :, 2] *= stride, m[:, :, 3] += m[:, :, 2] * k_first (timing only: values are compared
    elsewhere, and the relabelled products round differently)."""
    nx, ny, nz, n_proj = geom.nx, geom.ny, geom.nz, geom.np
    if nx * ny * nz * n_proj <= full_limit:
        return mats, nz, f"full volume ({nz} slices)"
    n_slices = max(n_threads, 1)
    stride = nz // n_slices
    k_first = stride // 2
    m = mats.astype(np.float64)
    m2 = m.copy()
    m2[:, :, 2] = m[:, :, 2] * stride
    m2[:, :, 3] = m[:, :, 3] + m[:, :, 2] * k_first
    ks = f"k = {k_first} + {stride}*q, q < {n_slices}"
    return m2.astype(np.float32), n_slices, f"{n_slices} z-slices evenly spaced over all {nz} ({ks}), full x,y, " \
                                            f"all {n_proj} angles"


def reference_step(conebp, img_np, mats_s, nx, ny, nk):
    P = conebp.ProjectionStack(img_np, img_np.shape[0], img_np.shape[1], img_np.shape[2])
    V = conebp.Volume.zeros(nx, ny, nk)
    t0 = time.perf_counter()
    conebp.backproject_baseline(P, mats_s, V)
    return time.perf_counter() - t0


def reference_warm(conebp) -> None:
    """Compile the reference kernel (numba JIT / cache load) outside any timed region."""
    img = np.zeros((2, 4, 4), np.float32)
    mats = np.zeros((2, 3, 4), np.float32)
    mats[:, 2, 3] = 1.0
    conebp.backproject_baseline(conebp.ProjectionStack(img, 2, 4, 4), mats, conebp.Volume.zeros(4, 4, 4))


def cpu_baseline_leg(geom, mats, img_np) -> dict:
    """cpu_baseline: the live reference on the host cores over a bounded sample."""
    try:
        conebp, numba = import_reference()
    except Exception as exc:  # the C port of _kernels.baseline (oracle/) stands in
        return cpu_port_leg(geom, mats, img_np, reason=f"reference import failed: {exc!r}")
    threads = numba.get_num_threads()
    mats_s, nk, sample = reference_sample(geom, mats, threads, full_limit=7e9)
    reference_warm(conebp)
    dt = reference_step(conebp, img_np, mats_s, geom.nx, geom.ny, nk)
    ups = geom.nx * geom.ny * nk * geom.np
    return {"value": ups / dt / 1e9, "unit": "GUPS", "cores": threads, "kind": "reference",
            "sample": f"{sample}, {dt:.1f} s; conebp.backproject_baseline (live reference, numba "
                      f"{numba.__version__}, {threads} threads, baseline/_ref)"}


def cpu_port_leg(geom, mats, img_np, reason: str) -> dict:
    sys.path.insert(0, str(REPO / "oracle"))
    import oracle

    threads = oracle.default_threads()
    nx, ny, nz = geom.nx, geom.ny, geom.nz
    nk = max(1, min(nz, threads))
    k_lo = max(0, nz // 2 - nk // 2)
    vol = np.zeros((nk, ny, nx), np.float32)
    t0 = time.perf_counter()
    oracle.baseline(img_np, mats, vol, threads=threads, k_lo=k_lo)
    dt = time.perf_counter() - t0
    return {"value": nk * nx * ny * geom.np / dt / 1e9, "unit": "GUPS", "cores": threads, "kind": "port",
            "sample": f"z-slab k=[{k_lo},{k_lo + nk}) of {nz}, {dt:.1f} s, C port of _kernels.baseline ({reason})"}


def reference_inputs(spec, geom) -> np.ndarray:
    """The same projection bytes our arm uses (config 4 is drawn by torch's CUDA RNG)."""
    if spec.index == 4:
        try:
            import torch

            if torch.cuda.is_available():
                return spec.projections_device(geom, device="cuda").cpu().numpy()
        except Exception:
            pass
    return spec.projections_host(geom)


def run_reference(args, spec, geom, mats) -> None:
    """--impl reference: the reference's own CPU implementation on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    img_np = reference_inputs(spec, geom)
    nx, ny = geom.nx, geom.ny
    try:
        conebp, numba = import_reference()
        threads = numba.get_num_threads()
        kind = "reference"
        mats_s, nk, sample = reference_sample(geom, mats, threads)
        desc = f"conebp.backproject_baseline (live reference from baseline/_ref, numba {numba.__version__})"

        def step():
            return reference_step(conebp, img_np, mats_s, nx, ny, nk)
        reference_warm(conebp)
    except Exception as exc:
        sys.path.insert(0, str(REPO / "oracle"))
        import oracle

        threads = oracle.default_threads()
        kind = "port"
        nk = max(threads, 1)
        k_lo = geom.nz // 2 - nk // 2
        sample = f"z-slab k=[{k_lo},{k_lo + nk}) of {geom.nz}"
        desc = f"C port of _kernels.baseline (reference import failed: {exc!r})"

        def step():
            vol = np.zeros((nk, ny, nx), np.float32)
            t0 = time.perf_counter()
            oracle.baseline(img_np, mats, vol, threads=threads, k_lo=k_lo)
            return time.perf_counter() - t0
    times = []
    for it in range(args.warmup + args.steps):
        dt = step()
        if it >= args.warmup:
            times.append(dt)
    tot = sum(times)
    per_step = nx * ny * nk * geom.np
    value = per_step * len(times) / tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GUPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": spec.inputs + " (synthetic, seeded; the same bytes as --impl ours)",
            # the same workload as --impl ours; a step covers a bounded sample of it (the contract's
            # "bounded sample of that workload"), described here and in cpu_baseline.sample
            "config": spec.describe() | {"variant": "baseline", "parallelism": f"host threads x{threads}",
                                         "arithmetic": "bit-exact (reference float32 op order)",
                                         "step_sample": {"z_slices": nk, "of": geom.nz,
                                                         "whole_volume": nk == geom.nz}},
            "cpu_baseline": {"value": value, "unit": "GUPS", "cores": threads, "kind": kind,
                             "sample": f"per step: {sample}; {desc}, {threads} threads"},
            "e2e": {"value": value, "unit": "GUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", default="baseline")
    ap.add_argument("--flags", type=int, default=0, help="library flags (1 naive, 2 no smem staging, 4 FMA lerps)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-pageable", action="store_true", help="also time the numpy API on pageable buffers")
    ap.add_argument("--chunks", type=int, default=8, help="angle chunks of the band transport (N > 1)")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "p2p"])
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
        plan = SL.plan_slabs(mats, nh, nw, nx, ny, nz, world, align=16, variant=int(variant))
        backend = SL.CudaBackend(torch)
        k0, k1 = plan.slab(rank)
        vol = backend.empty_slab(plan, k0, k1)
        shared = backend.ipc_share(img_dev, dist) if args.transport == "ipc" else None

        def step(i=None):
            SL.run_slabs(img_dev, mats, plan, backend, dist, n_chunks=args.chunks, vol=vol,
                         transport=args.transport, shared=shared, check=False)

        launches_per_step = args.chunks if plan.active(rank) else 0

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
    stats = D.sync_status()  # raises CBP_EBAND if a slab sampled outside its band
    ms_per_step = total_ms / args.steps
    value = updates / (ms_per_step * 1e-3) / 1e9
    clocks = sampler.summary()

    if rank != 0:
        if dist:
            dist.barrier()
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
                                         "arithmetic": "fma_lerp (tolerance mode)" if args.flags & 4 else
                                         "bit-exact (reference float32 op order)",
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
        # executed work: queued (tile, angle) pairs x tile voxels (every BASELINE config is a whole
        # number of tiles), per launch, from the device counters of the timed steps
        pairs = (stats["smem_pairs"] + stats["global_pairs"]) / args.steps
        tile_vox = plan_info["tile_x"] * plan_info["tile_y"] * plan_info["tile_z"]
        exec_updates = pairs * tile_vox if plan_info["kernel_kind"] else float(updates)
        exec_gath = GATHER_BYTES_PER_UPDATE * exec_updates / (k_avg * 1e-3) / 1e9
        line["roofline"] = {
            "bound": "gather", "unit": "GB/s", "achieved": gath, "peak": peak, "frac": gath / peak,
            "traffic": ncu_traffic(spec.name),
            "traffic_note": "DRAM read+write bytes per launch from a committed ncu --set full capture "
                            "(profiles/ncu_traffic.json); the gather roofline's algorithmic bytes are L1/shared "
                            "bytes, so DRAM traffic is shown for the HBM side",
            "peak_basis": f"128 B/clk/SM x {sms} SMs x {f_mhz:.0f} MHz (SM clock measured during run); "
                          f"algorithmic 16 B/update",
            "executed": {"achieved": exec_gath, "frac": exec_gath / peak, "updates_per_launch": exec_updates,
                         "fraction_of_reference_updates": exec_updates / updates,
                         "gups": exec_updates / (k_avg * 1e-3) / 1e9,
                         "basis": "queued (tile, angle) pairs x tile voxels; tiles whose detector footprint "
                                  "misses the detector are never queued (the reference guard rejects all their "
                                  "voxels)"},
            "kernel_ms": k_avg, "kernel_gups": gups_k,
            "fp32": {"ops_per_update": fp_ops, "ops_basis": "executed (reference's separately rounded ops)",
                     "peak_gups": fp_peak_gups, "frac": gups_k / fp_peak_gups,
                     "executed_frac": exec_updates / (k_avg * 1e-3) / 1e9 / fp_peak_gups},
            "hbm": {"compulsory_bytes": comp_bytes, "achieved_gbs": comp_bytes / (k_avg * 1e-3) / 1e9,
                    "peak_gbs": peaks.get("hbm_gbs")},
            "kernel_share_of_step": k_avg / ms_per_step,
        }
    line["plan"] = plan_info
    line["tile_stats_per_launch"] = {k: v / args.steps for k, v in stats.items()}

    img_pin = None
    if not args.no_e2e and world == 1:
        line["e2e"], img_pin = e2e_leg(torch, spec, geom, mats, img_dev, vol, variant, args)
    if not args.no_cpu and world == 1:
        img_np = img_pin.numpy() if img_pin is not None else img_dev.cpu().numpy()
        del img_dev, vol
        line["cpu_baseline"] = cpu_baseline_leg(geom, mats, img_np)
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def e2e_leg(torch, spec, geom, mats, img_dev, vol_dev, variant, args):
    """Same metric through the public numpy API with pinned host buffers (H2D + D2H every step)."""
    from paper_2104_13248_b200 import Layout, ProjectionStack, Volume, backproject_baseline

    nx, ny, nz, n_proj, nh, nw = geom.nx, geom.ny, geom.nz, geom.np, geom.nh, geom.nw
    img_pin = torch.empty((n_proj, nh, nw), dtype=torch.float32, pin_memory=True)
    img_pin.copy_(img_dev)
    vol_pin = torch.zeros((nz, ny, nx), dtype=torch.float32, pin_memory=True)
    proj = ProjectionStack(img_pin.numpy(), n_proj, nh, nw, Layout.NATURAL)
    vol = Volume(vol_pin.numpy(), nx, ny, nz, Layout.NATURAL)
    assert proj.data.ctypes.data == img_pin.data_ptr() and vol.data.ctypes.data == vol_pin.data_ptr()
    big = n_proj * nh * nw > 2 ** 30
    if big:  # make room on the device for the call's own copies (64 GiB on config 4)
        vol_dev.resize_(0)
        torch.cuda.empty_cache()

    def step():  # the user's call: accumulate into the caller's (pinned) volume
        backproject_baseline(proj, mats, vol)

    step()
    n = max(2, min(args.steps, 3 if big else 10))
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    dt = (time.perf_counter() - t0) / n
    out = {"value": nx * ny * nz * n_proj / dt / 1e9, "unit": "GUPS",
           "h2d_bytes_per_step": 4 * (n_proj * nh * nw + nx * ny * nz), "d2h_bytes_per_step": 4 * nx * ny * nz,
           "ms_per_step": dt * 1e3, "steps": n,
           "api": "paper_2104_13248_b200.backproject_baseline (numpy, pinned host buffers; angle-chunked H2D "
                  "overlapped with the kernels)"}
    if args.e2e_pageable:
        img_pg = img_pin.numpy().copy()
        vol_pg = np.zeros((nz, ny, nx), np.float32)
        p2, v2 = ProjectionStack(img_pg, n_proj, nh, nw), Volume(vol_pg, nx, ny, nz)
        backproject_baseline(p2, mats, v2)
        t0 = time.perf_counter()
        backproject_baseline(p2, mats, v2)
        dtp = time.perf_counter() - t0
        out["pageable"] = {"value": nx * ny * nz * n_proj / dtp / 1e9, "unit": "GUPS", "ms_per_step": dtp * 1e3}
        del img_pg, vol_pg, p2, v2
    del vol_pin
    return out, img_pin


if __name__ == "__main__":
    main()
