"""Benchmark harness with the reference's report schema, timing the GPU path (row f4).

Mirrors ``conebp.bench`` (/root/reference/pkg/src/conebp/bench.py:50-312): the desk and
full-scale problem catalogs, ``gups``, ``BenchReport`` (CSV columns and JSON schema v1,
plus GPU columns appended), ``run_bench`` / ``sweep_nb`` / ``verify_variants`` and the
report writers.  Differences, all deliberate:

* timing covers the back-projection on device-resident buffers (CUDA events, median
  of ``repeats`` after one warm-up), the analogue of the reference's kernel-only
  timing that excludes layout transposes (bench.py:224-246);
* ``nb`` is validated and recorded exactly as the reference does but does not change
  the GPU schedule (outputs are bitwise identical for every nb);
* ``verify_variants`` reports RMSE against the GPU BASELINE result; the GPU rungs are
  bit-exact reproductions of the reference rungs, so the values equal the
  reference's own ladder RMSEs.
"""

from __future__ import annotations

import csv
import json
import statistics
from dataclasses import dataclass

from .backprojector import BatchConfig, KernelVariant, OpCounters, count_ops
from .geometry import ScanGeometry, build_geometry

__all__ = ["Problem", "BenchReport", "DESK_LABELS", "desk_catalog", "fullscale_catalog", "find_problem",
           "geometry_for", "problem_data", "clear_data_cache", "gups", "run_bench", "sweep_nb", "verify_variants",
           "write_reports_csv", "write_reports_json", "CSV_COLUMNS", "SCHEMA_VERSION"]

SCHEMA_VERSION = 1
CSV_COLUMNS = ["label", "variant", "nb", "threads", "seconds", "gups", "dot_ops", "vol_words", "proj_words",
               "transpose_seconds", "gpus", "device", "sm_mhz"]


@dataclass(frozen=True)
class Problem:
    """Detector (nh, nw, np) -> volume (nx, ny, nz), as in bench.py:66-80."""

    label: str
    proj: tuple
    vol: tuple
    note: str = ""

    @property
    def updates(self) -> int:
        nx, ny, nz = self.vol
        return nx * ny * nz * self.proj[2]


_DESK = (
    Problem("D1", (64, 64, 128), (64, 64, 64), note="P1 at 1/4 linear scale"),
    Problem("D2", (128, 128, 128), (128, 128, 128), note="P5 at 1/4 linear scale"),
    Problem("D3", (128, 128, 256), (256, 256, 256), note="P2 at 1/2 linear scale"),
)
_FULL = tuple(Problem(lbl, (n, n, 512), (v, v, v)) for lbl, n, v in (
    ("P1", 256, 256), ("P2", 256, 512), ("P3", 256, 1024), ("P4", 512, 256), ("P5", 512, 512),
    ("P6", 512, 1024), ("P7", 1024, 256), ("P8", 1024, 512), ("P9", 1024, 1024), ("P10", 1024, 1300)))
DESK_LABELS = tuple(p.label for p in _DESK)


def desk_catalog() -> tuple:
    return _DESK


def fullscale_catalog() -> tuple:
    return _FULL


def find_problem(label: str) -> Problem:
    for p in _DESK + _FULL:
        if p.label.lower() == label.lower():
            return p
    raise ValueError(f"unknown problem label {label!r}")


def geometry_for(problem: Problem) -> ScanGeometry:
    nh, nw, n_proj = problem.proj
    nx, ny, nz = problem.vol
    return build_geometry(nx=nx, ny=ny, nz=nz, nw=nw, nh=nh, np=n_proj)


_cache: dict = {}


def problem_data(problem: Problem):
    """(geometry, truth, projections, matrices) from the GPU make_dataset, cached."""
    from .phantom import make_dataset

    key = (problem.proj, problem.vol)
    if key not in _cache:
        geom = geometry_for(problem)
        _cache[key] = (geom, *make_dataset(geom))
    return _cache[key]


def clear_data_cache() -> None:
    _cache.clear()


def gups(nx: int, ny: int, nz: int, np_: int, seconds: float) -> float:
    """Giga voxel updates per second: nx*ny*nz*np / t / 1e9 (bench.py:150-154)."""
    if seconds <= 0:
        raise ValueError(f"seconds must be positive, got {seconds}")
    return nx * ny * nz * np_ / seconds / 1e9


@dataclass(frozen=True)
class BenchReport:
    label: str
    variant: str
    nb: int
    threads: int
    wall_seconds: float
    gups: float
    counters: OpCounters
    transpose_seconds: float
    gpus: int = 1
    device: str = ""
    sm_mhz: float = 0.0

    def to_csv_row(self) -> list:
        c = self.counters
        return [self.label, self.variant, self.nb, self.threads, repr(self.wall_seconds), repr(self.gups), c.dot_ops,
                c.vol_word_accesses, c.proj_word_accesses, repr(self.transpose_seconds), self.gpus, self.device,
                repr(self.sm_mhz)]

    def to_json_dict(self) -> dict:
        c = self.counters
        return {"schema_version": SCHEMA_VERSION, "label": self.label, "variant": self.variant, "nb": self.nb,
                "threads": self.threads, "seconds": self.wall_seconds, "gups": self.gups, "dot_ops": c.dot_ops,
                "vol_words": c.vol_word_accesses, "proj_words": c.proj_word_accesses,
                "transpose_seconds": self.transpose_seconds, "gpus": self.gpus, "device": self.device,
                "sm_mhz": self.sm_mhz}


def _sm_mhz() -> float:
    try:
        import pynvml

        pynvml.nvmlInit()
        import torch

        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        return float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
    except Exception:
        return 0.0


def run_bench(problem: Problem, variant: KernelVariant, nb: int = 32, threads: int | None = None,
              repeats: int = 5) -> BenchReport:
    """Median-of-N device timing of one back-projection after one discarded warm-up."""
    import torch

    from . import device as D
    from .tensors import Layout

    variant = KernelVariant(variant)
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    nh, nw, n_proj = problem.proj
    nx, ny, nz = problem.vol
    if variant is KernelVariant.BASELINE:
        nb = 1
    BatchConfig(nb).check_divides(n_proj)
    geom, truth, proj, mats = problem_data(problem)
    img = torch.from_numpy(proj.data).cuda()
    layout = Layout.NATURAL if variant is KernelVariant.BASELINE else Layout.TRANSPOSED
    transpose_seconds = 0.0
    if layout is Layout.TRANSPOSED:  # the reference transposes on the host and times it separately
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        img = img.transpose(1, 2).contiguous()
        t1.record()
        torch.cuda.synchronize()
        transpose_seconds = t0.elapsed_time(t1) * 1e-3
    shape = (nz, ny, nx) if layout is Layout.NATURAL else (nx, ny, nz)

    def once() -> float:
        vol = torch.zeros(shape, dtype=torch.float32, device="cuda")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        D.backproject_device(img, mats, vol, n_proj, nh, nw, nx, ny, nz, variant, layout, layout)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e-3

    once()
    seconds = statistics.median(once() for _ in range(repeats))
    return BenchReport(label=problem.label, variant=variant.name.lower(), nb=nb, threads=0, wall_seconds=seconds,
                       gups=gups(nx, ny, nz, n_proj, seconds), counters=count_ops(variant, nx, ny, nz, n_proj, nb=nb,
                                                                                   nh=nh),
                       transpose_seconds=transpose_seconds, gpus=1, device=torch.cuda.get_device_name(),
                       sm_mhz=_sm_mhz())


def sweep_nb(problem: Problem, variant: KernelVariant, nb_values=(1, 2, 4, 8, 16, 32), threads: int | None = None,
             repeats: int = 5) -> list:
    return [run_bench(problem, variant, nb=nb, threads=threads, repeats=repeats) for nb in nb_values]


def verify_variants(problem: Problem, variants=None, nb: int = 32, threads: int | None = None) -> dict:
    """RMSE of each optimized rung against the BASELINE volume (bench.py:276-298)."""
    from .backprojector import backproject_baseline, backproject_optimized
    from .phantom import rmse
    from .tensors import Layout, Volume, transpose_projections, transpose_volume

    if variants is None:
        variants = [v for v in KernelVariant if v is not KernelVariant.BASELINE]
    nx, ny, nz = problem.vol
    geom, truth, proj, mats = problem_data(problem)
    base = backproject_baseline(proj, mats, Volume.zeros(nx, ny, nz))
    img_t = transpose_projections(proj)
    out = {}
    for variant in variants:
        variant = KernelVariant(variant)
        if variant is KernelVariant.BASELINE:
            continue
        vol_t = Volume.zeros(nx, ny, nz, Layout.TRANSPOSED)
        backproject_optimized(img_t, mats, vol_t, variant, batch=BatchConfig(nb))
        out[variant.name.lower()] = rmse(base, transpose_volume(vol_t))
    return out


def write_reports_csv(path, reports) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(CSV_COLUMNS)
        for r in reports:
            w.writerow(r.to_csv_row())


def write_reports_json(path, reports) -> None:
    with open(path, "w") as fh:
        json.dump([r.to_json_dict() for r in reports], fh, indent=2)
        fh.write("\n")
