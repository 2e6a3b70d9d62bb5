"""ORACLE — test infrastructure only; never part of the product path.

Python side of the CPU restatement of the reference's PHOBIC construction
(pilothash 0.1.0). The arithmetic lives in ``phobic_oracle.c`` (compiled to
``oracle/build/liboracle.so`` by ``__graft_entry__.build()`` /
``oracle/Makefile``); this module adds the host-side pieces the reference
computes in Python: the assignment table (assignment.py:48-121), the
partition count (partitioning.py:62-65), the retry loop (mphf.py:236-290)
and the fixed header + checksum (mphf.py:156-175, :231-233).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` leg may import this module. Parity of the
restatement is pinned against golden vectors produced by the reference
itself (``tests/golden/make_golden.py``, checked by
``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import struct
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"
SRC = HERE / "phobic_oracle.c"

GRID = 2048
KINDS = ("uniform", "skew", "beta_star", "beta_eps")
MAX_ATTEMPTS = 4
DEFAULT_SEED_CAP = 1 << 40

_lib = None


def build_lib() -> Path:
    """Compile the restatement (no FMA contraction: -ffp-contract=off)."""
    LIB_PATH.parent.mkdir(exist_ok=True)
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
             "-o", str(LIB_PATH), str(SRC), "-lm"],
            check=True,
        )
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build_lib()
        L = ctypes.CDLL(str(LIB_PATH))
        P, I64, U64, INT = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        L.orc_murmur3_many.argtypes = [P, P, I64, U64, P, P]
        L.orc_murmur3_u64.argtypes = [P, I64, U64, P, P]
        L.orc_bucket_ids.argtypes = [P, I64, P, I64, P]
        L.orc_partition.argtypes = [P, P, I64, I64, P, P, P, P]
        L.orc_build_partition_range.argtypes = [P, P, P, I64, I64, P, I64, I64, INT, P, P, P, INT]
        L.orc_query_many.argtypes = [P, P, I64, I64, I64, P, P, I64, P, P]
        L.orc_encode_body.argtypes = [P, I64, I64, INT, I64, P, ctypes.POINTER(ctypes.c_size_t)]
        L.orc_encode_body.restype = ctypes.c_void_p
        L.orc_free.argtypes = [P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a.size else None


# ---- host-side config math (assignment.py, partitioning.py, builder.py) ----

def beta_star(x: float) -> float:  # assignment.py:48-54
    if x == 1.0:
        return 1.0
    return x + (1.0 - x) * math.log1p(-x)


def curve(kind: str, eps: float):  # assignment.py:87-94
    if kind == "uniform":
        return lambda x: x
    if kind == "skew":  # assignment.py:71-77
        return lambda x: 0.5 * x if x <= 0.6 else 1.75 * x - 0.75
    if kind == "beta_star":
        return beta_star
    return lambda x: eps * x + (1.0 - eps) * beta_star(x)  # assignment.py:57-61


def tabulate(kind: str = "beta_eps", eps: float = 0.0) -> np.ndarray:  # assignment.py:115-121
    g = curve(kind, eps)
    return np.array([g(k / GRID) for k in range(GRID + 1)], dtype=np.float64)


def default_epsilon(lam: float, P: float) -> float:  # assignment.py:64-68
    return min(0.99, max(0.0, lam / (5.0 * math.sqrt(P))))


def bucket_count(P: float, lam: float) -> int:  # assignment.py:80-84
    return max(1, round(P / lam))


def num_partitions_for(n: int, P: float) -> int:  # partitioning.py:62-65
    return max(1, round(n / P))


def parse_encoder(name: str):  # builder.py:79-88
    if name in ("ic-r", "ic-c", "mono-r", "mono-c"):
        return name, None
    if name.startswith("mixed:"):
        return "mixed", int(name.split(":", 1)[1])
    raise ValueError(name)


# ---- stage wrappers ----

def murmur3_many(buf: np.ndarray, offsets: np.ndarray, seed: int):
    n = len(offsets) - 1
    hi = np.empty(n, np.uint64)
    lo = np.empty(n, np.uint64)
    buf = np.ascontiguousarray(buf, np.uint8)
    offsets = np.ascontiguousarray(offsets, np.int64)
    if n:
        lib().orc_murmur3_many(_p(buf) if buf.size else None, _p(offsets), n,
                               seed & (2**64 - 1), _p(hi), _p(lo))
    return hi, lo


def murmur3_u64(keys: np.ndarray, seed: int):
    keys = np.ascontiguousarray(keys, np.uint64)
    hi = np.empty(len(keys), np.uint64)
    lo = np.empty(len(keys), np.uint64)
    if len(keys):
        lib().orc_murmur3_u64(_p(keys), len(keys), seed & (2**64 - 1), _p(hi), _p(lo))
    return hi, lo


def bucket_ids(his: np.ndarray, table: np.ndarray, bcount: int) -> np.ndarray:
    his = np.ascontiguousarray(his, np.uint64)
    out = np.empty(len(his), np.int64)
    if len(his):
        lib().orc_bucket_ids(_p(his), len(his), _p(np.ascontiguousarray(table)), bcount, _p(out))
    return out


def partition(his: np.ndarray, los: np.ndarray, P: float):
    n = len(his)
    nparts = num_partitions_for(n, P)
    hs = np.empty(n, np.uint64)
    ls = np.empty(n, np.uint64)
    key_off = np.empty(nparts + 1, np.int64)
    deltas = np.empty(nparts + 1, np.int64)
    lib().orc_partition(_p(np.ascontiguousarray(his, np.uint64)),
                        _p(np.ascontiguousarray(los, np.uint64)), n, nparts,
                        _p(hs), _p(ls), _p(key_off), _p(deltas))
    return hs, ls, key_off, deltas


def build_partition_range(his, los, key_off, p_lo, p_hi, table, bcount, seed_cap, tie_desc,
                          threads=1):
    nparts = len(key_off) - 1
    seeds = np.zeros(nparts * bcount, np.uint64)
    trials = np.zeros(nparts * bcount, np.int64)
    status = np.zeros(nparts, np.uint8)
    lib().orc_build_partition_range(
        _p(np.ascontiguousarray(his, np.uint64)), _p(np.ascontiguousarray(los, np.uint64)),
        _p(np.ascontiguousarray(key_off, np.int64)), p_lo, p_hi,
        _p(np.ascontiguousarray(table)), bcount, seed_cap, int(tie_desc),
        _p(seeds), _p(trials), _p(status), threads)
    return seeds.reshape(nparts, bcount), trials.reshape(nparts, bcount), status


def query_many(his, los, n, nparts, deltas, table, bcount, seed_mat):
    out = np.empty(len(his), np.int64)
    if len(his):
        lib().orc_query_many(_p(np.ascontiguousarray(his, np.uint64)),
                             _p(np.ascontiguousarray(los, np.uint64)), len(his), n, nparts,
                             _p(np.ascontiguousarray(deltas, np.int64)),
                             _p(np.ascontiguousarray(table)), bcount,
                             _p(np.ascontiguousarray(seed_mat, np.uint64).reshape(-1)), _p(out))
    return out


def encode_body(seed_mat: np.ndarray, deltas: np.ndarray, encoder: str) -> bytes:
    nparts, bcount = seed_mat.shape
    fam, t = parse_encoder(encoder)
    mono = fam.startswith("mono")
    if fam == "ic-r":
        prefix = 0
    elif fam == "ic-c":
        prefix = bcount
    elif fam == "mixed":
        prefix = min(t, bcount)
    else:
        prefix = 1 if fam == "mono-c" else 0
    n_out = ctypes.c_size_t(0)
    sm = np.ascontiguousarray(seed_mat, np.uint64)
    ptr = lib().orc_encode_body(_p(sm), nparts, bcount, int(mono), prefix,
                                _p(np.ascontiguousarray(deltas, np.int64)), ctypes.byref(n_out))
    data = ctypes.string_at(ptr, n_out.value)
    lib().orc_free(ptr)
    return data


# ---- end to end (mphf.build, mphf.py:236-290) ----

@dataclass
class OracleMphf:
    n: int
    nparts: int
    bcount: int
    lambda_: float
    P: float
    kind: str
    eps: float
    global_seed: int
    attempts: int
    deltas: np.ndarray
    seeds: np.ndarray       # [nparts, B]
    trials: np.ndarray      # [nparts, B]
    table: np.ndarray
    encoder: str

    def body(self) -> bytes:
        return encode_body(self.seeds, self.deltas, self.encoder)

    def serialize(self) -> bytes:  # mphf.py:156-175
        head = (b"PHOB" + struct.pack("<I", 1) + struct.pack("<Q", self.n)
                + struct.pack("<Q", self.nparts) + struct.pack("<d", self.lambda_)
                + struct.pack("<d", self.P) + struct.pack("<B", KINDS.index(self.kind))
                + struct.pack("<d", self.eps) + struct.pack("<Q", self.global_seed & (2**64 - 1)))
        body = head + self.body()
        return body + struct.pack("<Q", checksum(body))

    def query_hashes(self, his, los):
        return query_many(his, los, self.n, self.nparts, self.deltas, self.table, self.bcount,
                          self.seeds)


def checksum(payload: bytes) -> int:  # mphf.py:231-233
    return int.from_bytes(hashlib.blake2b(payload, digest_size=8).digest(), "little")


def hash_keys(keys, seed: int):
    """keys: np.uint64 array (8-byte LE contract) or (buf, offsets)."""
    if isinstance(keys, tuple):
        return murmur3_many(keys[0], keys[1], seed)
    return murmur3_u64(keys, seed)


def build(keys, lambda_=8.0, P=2500.0, encoder="ic-r", tie_break="asc-expected",
          seed_cap=DEFAULT_SEED_CAP, global_seed=0, threads=None, kind="beta_eps",
          eps=None) -> OracleMphf:
    threads = threads or os.cpu_count() or 1
    if eps is None:
        eps = default_epsilon(lambda_, P) if kind == "beta_eps" else 0.0
    table = tabulate(kind, eps)
    B = bucket_count(P, lambda_)
    tie_desc = tie_break == "asc-expected"
    for attempt in range(MAX_ATTEMPTS):
        seed = global_seed + attempt
        his, los = hash_keys(keys, seed)
        n = len(his)
        hs, ls, key_off, deltas = partition(his, los, P)
        nparts = len(key_off) - 1
        seeds, trials, status = build_partition_range(hs, ls, key_off, 0, nparts, table, B,
                                                      seed_cap, tie_desc, threads)
        if np.any(status != 0):
            continue
        return OracleMphf(n, nparts, B, lambda_, P, kind, eps, seed, attempt + 1, deltas, seeds,
                          trials, table, encoder)
    raise RuntimeError("oracle: duplicate keys")
