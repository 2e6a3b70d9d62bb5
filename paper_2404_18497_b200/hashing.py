"""Key hashing: the 128-bit master hash and its derived indices.

Mirrors pilothash.hashing (hashing.py:1-202). Bulk hashing runs on the
device (csrc/hash.cu, C-ABI ``phb_murmur3_many`` / ``phb_murmur3_u64``,
replacing _kernels.murmur3_many). The scalar helpers below (mix64,
to_unit, position_hash, ...) are reference-compatible formula helpers for
hand-built test cases; the build and query paths never call them.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np
import torch

from . import _native
from .keygen import as_corpus, to_device

MASK64 = (1 << 64) - 1
BUCKET_SALT = 0xC2B2AE3D27D4EB4F    # hashing.py:29 / _kernels.py:29
POSITION_SALT = 0x9E3779B97F4A7C15  # hashing.py:31 / _kernels.py:30


class MasterHash(NamedTuple):
    hi: int
    lo: int


def mix64(z: int) -> int:
    """splitmix64 finalizer (hashing.py:42-50)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def to_unit(bits: int) -> float:
    """(bits + 1) / 2^64 in float64 (hashing.py:96-103)."""
    return (float(bits & MASK64) + 1.0) * 2.0**-64


def bucket_bits(h: MasterHash) -> int:
    return mix64(h.hi ^ BUCKET_SALT)


def normalized_hash(h: MasterHash) -> float:
    return to_unit(bucket_bits(h))


def partition_index(h: MasterHash, num_partitions: int) -> int:
    """floor(hi * nparts / 2^64) (hashing.py:115-117)."""
    return ((h.hi & MASK64) * num_partitions) >> 64


def position_hash(h: MasterHash, s: int, m: int) -> int:
    """floor(mix64(lo ^ mix64(s ^ SALT)) * m / 2^64) (hashing.py:120-130)."""
    if m < 1:
        raise ValueError("partition size must be >= 1")
    return (mix64(h.lo ^ mix64(s ^ POSITION_SALT)) * m) >> 64


def master_hash_device(keys, seed: int):
    """Device his/los (torch uint64 tensors) of any accepted key container."""
    dev = _native.require_device()
    dk = to_device(keys, dev)
    hi = torch.empty(dk.n, dtype=torch.uint64, device=dev)
    lo = torch.empty(dk.n, dtype=torch.uint64, device=dev)
    if dk.n:
        if dk.is_u64:
            _native.call("phb_murmur3_u64", _native.ptr(dk.keys64), dk.n, seed & MASK64,
                         _native.ptr(hi), _native.ptr(lo), _native.stream())
        else:
            _native.call("phb_murmur3_many", _native.ptr(dk.buf), _native.ptr(dk.offsets), dk.n,
                         seed & MASK64, _native.ptr(hi), _native.ptr(lo), _native.stream())
    return hi, lo


def _host_u64(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int64).cpu().numpy().view(np.uint64)


def master_hash_many(buf: np.ndarray, offsets: np.ndarray, seed: int):
    """Bulk master hash over concatenated keys -> (his, los) uint64 arrays
    (hashing.py:65-76), computed on the device."""
    from .keygen import KeyCorpus

    hi, lo = master_hash_device(KeyCorpus(np.asarray(buf, np.uint8), np.asarray(offsets, np.int64)),
                                seed)
    return _host_u64(hi), _host_u64(lo)


def master_hash(key, seed: int) -> MasterHash:
    """128-bit master hash of one key (hashing.py:53-62), on the device."""
    if isinstance(key, str):
        key = key.encode("utf-8")
    his, los = master_hash_many(np.frombuffer(bytes(key), np.uint8).copy(),
                                np.array([0, len(key)], np.int64), seed)
    return MasterHash(int(his[0]), int(los[0]))


def master_hash_corpus(keys, seed: int):
    """Host (his, los) for any key container accepted by ``build``."""
    if isinstance(keys, (np.ndarray, torch.Tensor)):
        hi, lo = master_hash_device(keys, seed)
        return _host_u64(hi), _host_u64(lo)
    c = as_corpus(keys)
    return master_hash_many(c.buf, c.offsets, seed)
