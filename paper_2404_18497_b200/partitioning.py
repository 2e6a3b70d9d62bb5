"""Partition layout: counts, offsets and the stored offset deltas.

Mirrors pilothash.partitioning (partitioning.py:1-152). The device pipeline
(csrc/hash.cu K1, csrc/layout.cu K2) produces counts, key offsets and
deltas; ``PartitionLayout`` keeps the host copy of the deltas that the
serialized format and ``offset`` need. ``pack_deltas`` / ``unpack_deltas``
are linear-time here (the reference's big-int version is O(nparts^2),
SURVEY.md §6.2); the build path packs deltas on the device instead.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class DegenerateConfig(ValueError):
    pass


def num_partitions_for(n: int, partition_size: float) -> int:
    """max(1, round(n / P)), Python half-even rounding (partitioning.py:62-65)."""
    if partition_size < 1:
        raise ValueError("partition size must be >= 1")
    return max(1, round(n / partition_size))


def expected_offset(j: int, n: int, nparts: int) -> int:
    """Round-half-up of j * n / nparts in exact integers (partitioning.py:68-70)."""
    return (2 * j * n + nparts) // (2 * nparts)


def expected_offsets(n: int, nparts: int) -> np.ndarray:
    j = np.arange(nparts + 1, dtype=object)
    return ((2 * j * n + nparts) // (2 * nparts)).astype(np.int64)


@dataclass(frozen=True)
class PartitionLayout:
    n: int
    num_partitions: int
    deltas: np.ndarray  # int64[num_partitions + 1]; first and last are 0

    def offset(self, j: int) -> int:
        return offset(self, j)

    def size(self, j: int) -> int:
        return offset(self, j + 1) - offset(self, j)

    @property
    def delta_width(self) -> int:
        return delta_width(self.deltas)

    def key_offsets(self) -> np.ndarray:
        return expected_offsets(self.n, self.num_partitions) + self.deltas


def offset(layout: PartitionLayout, j: int) -> int:
    if not 0 <= j <= layout.num_partitions:
        raise IndexError(f"partition index {j} out of range")
    return expected_offset(j, layout.n, layout.num_partitions) + int(layout.deltas[j])


def delta_width(deltas: np.ndarray) -> int:
    """bitlen(max |delta|) + 1 (partitioning.py:125-128)."""
    peak = int(np.max(np.abs(deltas))) if len(deltas) else 0
    return peak.bit_length() + 1


def pack_deltas(deltas: np.ndarray) -> tuple[int, bytes]:
    """Fixed-width LSB-first packing with bias 2^(w-1) (partitioning.py:131-142)."""
    d = np.asarray(deltas, dtype=np.int64)
    w = delta_width(d)
    v = (d + (1 << (w - 1))).astype(np.uint64)
    if np.any(v >> np.uint64(w) if w < 64 else False):
        raise ValueError("delta out of range for computed width")
    nbits = len(d) * w
    bits = ((v[:, None] >> np.arange(w, dtype=np.uint64)) & np.uint64(1)).astype(np.uint8)
    packed = np.packbits(bits.reshape(-1), bitorder="little")
    return w, packed.tobytes()[: (nbits + 7) // 8]


def unpack_deltas(width: int, data: bytes, count: int) -> np.ndarray:
    """Inverse of pack_deltas (partitioning.py:145-152)."""
    if width < 1:
        raise ValueError("delta width must be >= 1")
    need = (count * width + 7) // 8
    if len(data) < need:
        raise ValueError("truncated delta section")
    bits = np.unpackbits(np.frombuffer(data[:need], np.uint8), bitorder="little")
    bits = bits[: count * width].reshape(count, width).astype(np.uint64)
    vals = (bits << np.arange(width, dtype=np.uint64)).sum(axis=1, dtype=np.uint64)
    return vals.astype(np.int64) - np.int64(1 << (width - 1)) if width < 64 else (
        (vals - np.uint64(1 << 63)).astype(np.int64))
