"""Instrumented builds over assignment-function variants on the device.

Mirrors pilothash.analysis.measure_work / WorkReport / work_csv
(analysis.py:160-290), the work measurement behind the paper's Figure-4/5
sweeps: for every assignment variant, the keys' buckets are redistributed and
the full seed search runs, reporting the reference's trial counts (per bucket
index, per partition, total), the bucket-size histogram and the space of the
encoded result. Here each variant is one instrumented device build pass
(BuildEngine.run(instrument=True): K1-K5 with the search writing per-bucket
trials), so the counts are the reference's exactly (tests/test_gpu_analysis.py
checks them against the reference's own measure_work outputs).

The paper-math helpers of the reference module (chain models, expected
bucket sizes) are analysis of the method, not the construction path, and
are out of scope.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .assignment import AssignmentSpec
from .builder import BuildConfig, SeedExhausted
from .keygen import to_device
from .mphf import BuildEngine

CSV_HEADER = "assignment,lambda,partition_size,trials_per_key,bits_per_key,wall_seconds"


@dataclass
class WorkReport:
    """analysis.py:160-180."""

    assignment: str
    lambda_: float
    partition_size: float
    n: int
    per_bucket_trials: np.ndarray  # summed over partitions, by bucket index
    per_partition_trials: np.ndarray
    total_trials: int
    trials_per_key: float
    size_histogram: dict
    bits_per_key: float
    wall_seconds: float

    def csv_row(self) -> str:
        return (
            f"{self.assignment},{self.lambda_},{self.partition_size},"
            f"{self.trials_per_key:.3f},{self.bits_per_key:.4f},{self.wall_seconds:.3f}"
        )


def measure_work(keys, variants, config: BuildConfig | None = None) -> list[WorkReport]:
    """analysis.py:185-249. `variants`: AssignmentSpec or kind names (a bare
    name means epsilon 0, as in the reference). wall_seconds is the device
    time of the variant's build pass (CUDA events)."""
    config = config or BuildConfig()
    dev = _native.require_device()
    dk = to_device(keys, dev)
    reports = []
    for spec in variants:
        if not isinstance(spec, AssignmentSpec):
            spec = AssignmentSpec(str(spec))
        cfg = dataclasses.replace(config, assignment=spec)
        engine = BuildEngine(cfg, dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = engine.run(dk, config.global_seed, instrument=True)
        e1.record()
        if isinstance(res, tuple):  # build_all_partitions raises (builder.py:273-276)
            bad, code = res
            reason = "unseparable duplicate hashes" if code == 1 else "seed cap hit"
            raise SeedExhausted(f"partition {bad}: {reason}")
        torch.cuda.synchronize()
        B, nparts = res.bcount, res.nparts
        trials = res.trials.view(B, nparts)
        per_bucket = trials.sum(dim=1).cpu().numpy()
        per_part = res.part_trials.cpu().numpy()
        sizes = torch.bincount(res.bucket_sizes).cpu().numpy()
        hist = {int(s): int(c) for s, c in enumerate(sizes) if s > 0 and c > 0}
        total = int(per_bucket.sum())
        reports.append(WorkReport(
            assignment=spec.kind, lambda_=config.lambda_, partition_size=config.partition_size,
            n=dk.n, per_bucket_trials=per_bucket, per_partition_trials=per_part,
            total_trials=total, trials_per_key=total / dk.n, size_histogram=hist,
            bits_per_key=(res.total_bytes + 8 - 16) * 8 / dk.n,
            wall_seconds=e0.elapsed_time(e1) / 1e3))
    return reports


def work_csv(reports: list[WorkReport]) -> str:
    return "\n".join([CSV_HEADER] + [r.csv_row() for r in reports]) + "\n"
