"""Build configuration and the per-partition construction entry point.

Mirrors pilothash.builder (builder.py:1-277): ``BuildConfig`` keeps the
reference's fields, defaults and validation (builder.py:43-76);
``build_all_partitions`` keeps its signature and result
(seeds, per-bucket trials as [nparts, B] arrays, ``SeedExhausted`` on any
failing partition, builder.py:224-277) but runs the whole partition range
as one device launch (C-ABI ``phb_build_partition_range``, replacing
_kernels.build_partition_range on a thread pool). ``threads`` is accepted
and ignored: the device search is thread-count invariant by construction.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .assignment import AssignmentSpec, AssignmentTable, bucket_count, default_epsilon

DEFAULT_SEED_CAP = 1 << 40


class SeedExhausted(RuntimeError):
    """No seed below the cap places a bucket; the input may contain duplicates."""


class InvalidConfig(ValueError):
    pass


def parse_encoder(name: str) -> tuple[str, int | None]:
    """Encoder preset -> (family, compact prefix) (builder.py:79-88)."""
    if name in ("ic-r", "ic-c", "mono-r", "mono-c"):
        return name, None
    if name.startswith("mixed:"):
        try:
            t = int(name.split(":", 1)[1])
        except ValueError as exc:
            raise InvalidConfig(f"bad mixed preset {name!r}") from exc
        if t < 0:
            raise InvalidConfig("mixed:<t> needs t >= 0")
        return "mixed", t
    raise InvalidConfig(f"unknown encoder preset {name!r}")


@dataclass(frozen=True)
class BuildConfig:
    lambda_: float = 8.0
    partition_size: float = 2500.0
    assignment: AssignmentSpec | None = None  # None: beta_eps with the default epsilon
    seed_cap: int = DEFAULT_SEED_CAP
    global_seed: int = 0
    encoder: str = "ic-r"  # ic-r | ic-c | mixed:<t> | mono-r | mono-c
    tie_break: str = "asc-expected"
    threads: int = 1

    def __post_init__(self):
        if self.lambda_ <= 0:
            raise InvalidConfig("lambda must be > 0")
        if self.partition_size < 1:
            raise InvalidConfig("partition size must be >= 1")
        if self.seed_cap < self.partition_size:
            raise InvalidConfig("seed cap must allow one full displacement sweep")
        if self.tie_break not in ("asc-expected", "desc-expected"):
            raise InvalidConfig("tie_break must be asc-expected or desc-expected")
        if self.threads < 1:
            raise InvalidConfig("threads must be >= 1")
        parse_encoder(self.encoder)

    def resolved_assignment(self) -> AssignmentSpec:
        if self.assignment is not None:
            return self.assignment
        return AssignmentSpec("beta_eps", default_epsilon(self.lambda_, self.partition_size))

    @property
    def bucket_count(self) -> int:
        return bucket_count(self.partition_size, self.lambda_)

    @property
    def tie_desc(self) -> int:
        """The reference kernel's flag: 1 for "asc-expected" (builder.py:241)."""
        return 1 if self.tie_break == "asc-expected" else 0

    def compact_prefix(self) -> tuple[int, int]:
        """(mono flag, compact prefix t) of the encoder preset."""
        fam, t = parse_encoder(self.encoder)
        B = self.bucket_count
        if fam == "ic-r":
            return 0, 0
        if fam == "ic-c":
            return 0, B
        if fam == "mixed":
            return 0, min(int(t), B)
        return 1, (1 if fam == "mono-c" else 0)


def _dev_u64(a, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(dev).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(dev)


def device_table(table: AssignmentTable, dev) -> torch.Tensor:
    return torch.from_numpy(np.array(table.entries, dtype=np.float64)).to(dev)


def build_partition_range(his, los, key_offsets, p_lo: int, p_hi: int, table: AssignmentTable,
                          config: BuildConfig, seeds_out=None, trials_out=None, status_out=None):
    """Device equivalent of _kernels.build_partition_range over [p_lo, p_hi).

    his/los grouped by partition (any in-partition order). Returns device
    tensors (seeds u64 [nparts*B], trials i64, status u8) in the reference's
    row-major layout.
    """
    dev = _native.require_device()
    B = config.bucket_count
    d_his, d_los = _dev_u64(his, dev), _dev_u64(los, dev)
    d_off = torch.as_tensor(np.ascontiguousarray(key_offsets, np.int64)).to(dev)
    nparts = d_off.numel() - 1
    seeds = seeds_out if seeds_out is not None else torch.zeros(nparts * B, dtype=torch.int64, device=dev)
    trials = trials_out if trials_out is not None else torch.zeros(nparts * B, dtype=torch.int64, device=dev)
    status = status_out if status_out is not None else torch.zeros(nparts, dtype=torch.uint8, device=dev)
    entries = device_table(table, dev)
    _native.call("phb_build_partition_range", _native.ptr(d_his), _native.ptr(d_los),
                 _native.ptr(d_off), p_lo, p_hi, _native.ptr(entries), B, config.seed_cap,
                 config.tie_desc, _native.ptr(seeds), _native.ptr(trials), _native.ptr(status),
                 _native.stream())
    return seeds, trials, status


def build_all_partitions(his, los, key_offsets, table: AssignmentTable, config: BuildConfig):
    """(seed matrix [nparts, B] uint64, per-bucket trials [nparts, B] int64);
    raises SeedExhausted if any partition fails (builder.py:224-277)."""
    nparts = len(key_offsets) - 1
    B = config.bucket_count
    seeds, trials, status = build_partition_range(his, los, key_offsets, 0, nparts, table, config)
    st = status.cpu().numpy()
    if np.any(st != 0):
        bad = int(np.flatnonzero(st)[0])
        reason = "unseparable duplicate hashes" if st[bad] == 1 else "seed cap hit"
        raise SeedExhausted(f"partition {bad}: {reason}")
    s = seeds.cpu().numpy().view(np.uint64).reshape(nparts, B)
    return s, trials.cpu().numpy().reshape(nparts, B)
