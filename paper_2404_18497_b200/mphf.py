"""The queryable minimal perfect hash function and its device build.

Mirrors pilothash.mphf (mphf.py:1-306): ``build(keys, config) -> Mphf``
with the reference's retry policy (global_seed + attempt, 4 attempts, then
``DuplicateKeys``, mphf.py:236-290), ``Mphf.query / query_many /
is_bijection_on / bits_per_key / serialize / save / deserialize / load`` and
the versioned little-endian format with a blake2b-8 checksum
(mphf.py:156-233).

The construction path is the device pipeline of ``BuildEngine``:
  K1 phb_hash_count   murmur3 + partition index + per-partition counts
  K2 phb_layout       key offsets, offset deltas, max |delta|, max size
  K3 phb_scatter      re-hash, bucket id, scatter (lo, bucket) by partition
  K4 phb_search       per-partition bucket order + bit-parallel seed search
  K5 phb_encode_*     interleaved / mono Compact-Rice seeds + packed deltas
                      assembled as the serialized body (from byte 57)
Host work per attempt: two small synchronisations (max partition size for
the search's shared-memory plan, and the status/size summary), the 57-byte
fixed header and, for ``serialize``, blake2b over the body.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import struct
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .assignment import KIND_CODES, KINDS, AssignmentSpec, AssignmentTable, tabulate
from .builder import BuildConfig, InvalidConfig, SeedExhausted, device_table
from .encoders import MonoSeeds, SeedStore, parse_section
from .keygen import DeviceKeys, to_device, to_device_chunked
from .partitioning import PartitionLayout, num_partitions_for, unpack_deltas

MAGIC = b"PHOB"
VERSION = 1
HEADER_BYTES = 16  # magic + version + n; excluded from bits/key (mphf.py:56)
HEADER_FIXED = 57  # everything before the delta-width byte
MAX_ATTEMPTS = 4   # mphf.py:58


class DuplicateKeys(ValueError):
    pass


class FormatError(ValueError):
    pass


@dataclass
class BuildStats:
    attempts: int
    trials_total: int
    trials_per_key: float
    build_seconds: float


def _checksum(payload) -> int:
    return int.from_bytes(hashlib.blake2b(payload, digest_size=8).digest(), "little")


_ck_pool = None


def _checksum_async(payload):
    """blake2b of a freshly built body on a host thread (hashlib releases the
    GIL), overlapped with whatever the caller does next (query / verify);
    serialize() joins it. ~40 ms for the 27 MB body at C2."""
    global _ck_pool
    if _ck_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _ck_pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="phb-blake2b")
    return _ck_pool.submit(_checksum, payload)


def _header(n: int, nparts: int, lambda_: float, psize: float, spec: AssignmentSpec,
            global_seed: int) -> bytes:
    return (MAGIC + struct.pack("<IQQdd", VERSION, n, nparts, lambda_, psize)
            + struct.pack("<Bd", KIND_CODES[spec.kind], spec.epsilon)
            + struct.pack("<Q", global_seed & 0xFFFFFFFFFFFFFFFF))


@dataclass
class DeviceBuild:
    """Device-resident result of one successful pipeline pass."""

    n: int
    nparts: int
    bcount: int
    global_seed: int
    key_off: torch.Tensor   # int64 [nparts + 1]
    deltas: torch.Tensor    # int64 [nparts + 1]
    seeds: torch.Tensor     # int64 view of u64, column-major [B][nparts]
    blob: torch.Tensor      # uint8, serialized body (bytes [57, total) valid)
    total_bytes: int
    seed_section: int
    trials_total: int
    # instrumented builds only (BuildEngine.run(..., instrument=True)):
    trials: torch.Tensor | None = None        # int64 column-major [B][nparts] per-bucket trials
    part_trials: torch.Tensor | None = None   # int64 [nparts]
    bucket_sizes: torch.Tensor | None = None  # int64 [nparts * B]: keys per (partition, bucket)


class BuildEngine:
    """One device build pass at a time; buffers come from torch's caching allocator."""

    def __init__(self, config: BuildConfig, device: torch.device | None = None):
        self.config = config
        self.device = device or _native.require_device()
        self.spec = config.resolved_assignment()
        self.table: AssignmentTable = tabulate(self.spec)
        self.entries = device_table(self.table, self.device)
        self.bcount = config.bucket_count
        self.mono, self.prefix = config.compact_prefix()
        self._pinned = torch.zeros(2, dtype=torch.int64).pin_memory()
        self._pinned3 = torch.zeros(3, dtype=torch.int64).pin_memory()
        self._summary = np.zeros(8, np.int64)
        self.last_launches = 0

    def padded_capacity(self, n: int) -> int:
        """Record slots per partition for the fixed-capacity grouping: the
        mean size plus 12 standard deviations (Poisson) and a small margin;
        0 when the layout would not fit u32 cursors."""
        nparts = num_partitions_for(n, self.config.partition_size)
        mean = n / nparts
        cap = int(math.ceil(mean + 12.0 * math.sqrt(mean) + 16))
        return cap if nparts * cap < 2**32 and cap < 65536 else 0

    def _group_padded(self, dk: DeviceKeys, seed: int, nparts: int, cap: int, chunks):
        """K3 into fixed-capacity slots (one launch per arriving chunk), counts
        from the cursors, K2 layout. None if a partition overflowed."""
        dev, B = self.device, self.bcount
        n = dk.n
        st = _native.stream()
        P = _native.ptr
        L = _native.lib()
        cursor = torch.empty(nparts, dtype=torch.int32, device=dev)
        # 16-byte (lo, bucket id) records: one scattered store per key
        lo = torch.empty(2 * nparts * cap, dtype=torch.int64, device=dev)
        bid = None
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        base = P(dk.keys64)
        cur = torch.cuda.current_stream(dev)
        for i, (a, b, ev) in enumerate(chunks or [(0, n, None)]):
            if ev is not None:
                cur.wait_event(ev)  # this chunk's host-to-device copy is done
            _native.check(L.phb_scatter_padded(base + 8 * a, b - a, seed, nparts,
                                               P(self.entries), B, cap, int(i == 0), P(cursor),
                                               P(lo), P(bid), P(flag), st), "phb_scatter_padded")
        counts = torch.empty(nparts, dtype=torch.int32, device=dev)
        _native.check(L.phb_padded_counts(P(cursor), nparts, cap, P(counts), P(flag), st),
                      "phb_padded_counts")
        key_off = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
        deltas = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
        stats = torch.empty(3, dtype=torch.int64, device=dev)
        _native.check(L.phb_layout(P(counts), nparts, 0, 0, n, nparts, P(key_off), P(deltas),
                                   P(stats), st), "phb_layout")
        stats[2:3].copy_(flag)
        self._pinned3.copy_(stats, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        if int(self._pinned3[2]):
            return None  # a partition exceeded its slots: use the counted layout
        return lo, bid, key_off, deltas, stats[:2], int(self._pinned3[1])

    def run(self, dk: DeviceKeys, seed: int, instrument: bool = False,
            chunks=None) -> DeviceBuild | tuple[int, int]:
        """One attempt. Returns DeviceBuild, or (first_bad, code) on failure.
        instrument: also keep per-bucket trials, per-partition trials and the
        (partition, bucket) key counts (analysis.measure_work).
        chunks: [(begin, end, cuda event)] of u64 keys still being copied to
        the device; the grouping pass consumes each chunk once it has landed."""
        cfg, dev, B = self.config, self.device, self.bcount
        n = dk.n
        nparts = num_partitions_for(n, cfg.partition_size)
        st = _native.stream()
        P = _native.ptr
        L = _native.lib()
        seed &= 0xFFFFFFFFFFFFFFFF
        k64 = P(dk.keys64) if dk.is_u64 else None
        buf = None if dk.is_u64 else P(dk.buf)
        offs = None if dk.is_u64 else P(dk.offsets)

        # u64 keys still arriving from the host: fixed-capacity grouping, no
        # counting pass, each chunk grouped as soon as it lands (the copy and
        # the grouping overlap). Keys already in HBM, byte keys, or an
        # overflow: count, lay out, scatter (the counted pair is 0.25 ms faster
        # than the fixed-capacity pass when there is no copy to hide).
        grouped = None
        cap = self.padded_capacity(n) if chunks and dk.is_u64 and not instrument else 0
        if cap and k64 % 16 == 0:
            grouped = self._group_padded(dk, seed, nparts, cap, chunks)
        elif chunks:
            for _, _, ev in chunks:
                torch.cuda.current_stream(dev).wait_event(ev)
        if grouped is not None:
            lo, bid, key_off, deltas, stats, m_max = grouped
            seeds = torch.zeros(B * nparts, dtype=torch.int64, device=dev)
            part_trials = torch.empty(nparts, dtype=torch.int64, device=dev)
            status = torch.empty(nparts, dtype=torch.uint8, device=dev)
            glo = torch.empty(nparts * cap, dtype=torch.int64, device=dev)
            queue = torch.empty(1, dtype=torch.int32, device=dev)
            _native.check(L.phb_search_strided(P(lo), P(bid), P(key_off), 0, nparts, 0, B,
                                               cfg.seed_cap, cfg.tie_desc, m_max, P(seeds), 1,
                                               nparts, None, P(part_trials), P(status), P(glo),
                                               P(queue), cap, st), "phb_search_strided")
            return self._encode(n, nparts, seed, key_off, deltas, stats, seeds, status,
                                part_trials)

        counts = torch.zeros(nparts, dtype=torch.int32, device=dev)
        # byte keys: K1 keeps the 128-bit hashes so K3 does not hash the bytes again
        hashes = None
        if not dk.is_u64 and not instrument:
            hashes = torch.empty(2 * n, dtype=torch.int64, device=dev)
            _native.check(L.phb_hash_count_store(buf, offs, n, seed, nparts, P(counts), P(hashes),
                                                 st), "phb_hash_count_store")
        else:
            _native.check(L.phb_hash_count(buf, offs, k64, n, seed, nparts, P(counts), st),
                          "phb_hash_count")
        key_off = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
        deltas = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
        stats = torch.empty(2, dtype=torch.int64, device=dev)
        _native.check(L.phb_layout(P(counts), nparts, 0, 0, n, nparts, P(key_off), P(deltas),
                                   P(stats), st), "phb_layout")
        self._pinned.copy_(stats, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        # counts is reused as the scatter cursors (phb_scatter initialises them);
        # 16-byte (lo, bucket id) records (one scattered store per key) unless
        # the instrumented build needs the bucket ids on their own
        if instrument:
            lo = torch.empty(n, dtype=torch.int64, device=dev)
            bid = torch.empty(n, dtype=torch.int16, device=dev)
        else:
            lo = torch.empty(2 * n, dtype=torch.int64, device=dev)
            bid = None
        if hashes is not None:
            _native.check(L.phb_scatter_hashed(P(hashes), n, nparts, P(self.entries), B,
                                               P(key_off), P(counts), P(lo), st),
                          "phb_scatter_hashed")
            del hashes
        else:
            _native.check(L.phb_scatter(buf, offs, k64, n, seed, nparts, P(self.entries), B,
                                        P(key_off), P(counts), P(lo), P(bid), st), "phb_scatter")
        seeds = torch.zeros(B * nparts, dtype=torch.int64, device=dev)
        trials = torch.zeros(B * nparts, dtype=torch.int64, device=dev) if instrument else None
        sizes = None
        if instrument:  # keys per (partition, bucket): analysis only, torch is plumbing here
            part = torch.repeat_interleave(
                torch.arange(nparts, device=dev), key_off[1:] - key_off[:-1], output_size=n)
            sizes = torch.bincount(part * B + (bid.long() & 0xFFFF) - 1, minlength=nparts * B)
        part_trials = torch.empty(nparts, dtype=torch.int64, device=dev)
        status = torch.empty(nparts, dtype=torch.uint8, device=dev)
        glo = torch.empty(n, dtype=torch.int64, device=dev)
        queue = torch.empty(1, dtype=torch.int32, device=dev)
        ev.synchronize()
        m_max = int(self._pinned[1])
        _native.check(L.phb_search(P(lo), P(bid), P(key_off), 0, nparts, 0, B, cfg.seed_cap,
                                   cfg.tie_desc, m_max, P(seeds), 1, nparts,
                                   P(trials) if instrument else None,
                                   P(part_trials), P(status), P(glo), P(queue), st),
                      "phb_search")
        return self._encode(n, nparts, seed, key_off, deltas, stats, seeds, status, part_trials,
                            trials, part_trials if instrument else None, sizes)

    def _encode(self, n, nparts, seed, key_off, deltas, stats, seeds, status, part_trials,
                trials=None, keep_part_trials=None, sizes=None):
        """K5: plan (status / trials reduction, sizes) and the serialized body."""
        dev, B = self.device, self.bcount
        st = _native.stream()
        P = _native.ptr
        L = _native.lib()
        ws = torch.empty(int(L.phb_encode_workspace_bytes(nparts, B, self.mono)),
                         dtype=torch.uint8, device=dev)
        summ = self._summary
        _native.check(L.phb_encode_plan(P(seeds), nparts, B, self.mono, self.prefix, P(deltas),
                                        nparts, P(stats), P(status), P(part_trials), P(ws),
                                        summ.ctypes.data_as(ctypes.c_void_p), st),
                      "phb_encode_plan")
        if summ[3] >= 0:
            return int(summ[3]), int(summ[4])
        total = int(summ[0])
        blob = torch.empty((total + 16 + 3) // 4 * 4, dtype=torch.uint8, device=dev)
        _native.check(L.phb_encode_write(P(seeds), nparts, B, self.mono, self.prefix, P(deltas),
                                         nparts, P(stats), P(ws), P(blob), blob.numel(), st),
                      "phb_encode_write")
        return DeviceBuild(n, nparts, B, seed, key_off, deltas, seeds, blob, total,
                           int(summ[1]), int(summ[2]), trials, keep_part_trials, sizes)


class Mphf:
    def __init__(self, global_seed: int, layout: PartitionLayout | None, table: AssignmentTable,
                 bcount: int, seeds: SeedStore | None, lambda_: float, partition_size: float,
                 stats: BuildStats | None = None):
        self.global_seed = global_seed
        self._layout = layout
        self.table = table
        self.bcount = bcount
        self._seeds = seeds
        self.lambda_ = lambda_
        self.partition_size = partition_size
        self.stats = stats
        self._body = None  # serialized body without checksum (bytes-like)
        self._dev = None   # DeviceBuild backing a freshly built structure
        self._dev_key_off: torch.Tensor | None = None
        self._dev_entries: torch.Tensor | None = None

    # ---- construction from a device build -------------------------------
    @classmethod
    def _from_device(cls, db: DeviceBuild, config: BuildConfig, engine: BuildEngine,
                     stats: BuildStats) -> "Mphf":
        """Wrap a device build. The only eager host work is one D2H of the
        encoded body into pinned memory (the build's result); the layout and
        the seed-store views over the bytes are materialised on first use."""
        host = torch.empty(db.total_bytes, dtype=torch.uint8, pin_memory=True)
        host.copy_(db.blob[: db.total_bytes], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        body = host.numpy()
        body[:HEADER_FIXED] = np.frombuffer(
            _header(db.n, db.nparts, config.lambda_, config.partition_size, engine.spec,
                    db.global_seed), np.uint8)
        f = cls(db.global_seed, None, engine.table, db.bcount, None, config.lambda_,
                config.partition_size, stats)
        f._body = body
        f._body_owner = host
        f._ck_future = _checksum_async(body)  # the body is final: header written above
        f._dev = db
        f._dev_key_off = db.key_off
        f._dev_entries = engine.entries
        return f

    @property
    def layout(self) -> PartitionLayout:
        if self._layout is None:
            db = self._dev
            deltas = db.deltas.cpu().numpy()
            deltas.setflags(write=False)
            self._layout = PartitionLayout(db.n, db.nparts, deltas)
        return self._layout

    @layout.setter
    def layout(self, value: PartitionLayout) -> None:
        self._layout = value

    @property
    def seeds(self) -> SeedStore:
        if self._seeds is None:
            db = self._dev
            store, _ = parse_section(memoryview(self._body), db.seed_section, db.nparts,
                                     db.bcount)
            if db.seeds is not None:  # a sharded multi-GPU build keeps no seed matrix
                store._device = db.seeds.view(db.bcount, db.nparts)
            # encoded blocks for query_encoded_device come from the device body
            store._dev_source = (db.blob, db.seed_section + 4, db.total_bytes)
            self._seeds = store
        return self._seeds

    @seeds.setter
    def seeds(self, value: SeedStore) -> None:
        self._seeds = value

    # ---- properties -----------------------------------------------------
    @property
    def n(self) -> int:
        return self._dev.n if self._layout is None else self._layout.n

    @property
    def encoder_name(self) -> str:
        if isinstance(self.seeds, MonoSeeds):
            return "mono-c" if self.seeds.compact_prefix else "mono-r"
        t = self.seeds.compact_prefix
        if t == 0:
            return "ic-r"
        if t >= self.bcount:
            return "ic-c"
        return f"mixed:{t}"

    # ---- query ----------------------------------------------------------
    def _device_state(self, matrix: bool = True):
        dev = _native.require_device()
        if self._dev is not None:
            seeds = self._dev.seeds
            if seeds is None and matrix:
                seeds = self.seeds.device_matrix()  # decoded once from the device body
            return self._dev_key_off, self._dev_entries, seeds
        if self._dev_key_off is None:
            d = torch.from_numpy(np.array(self.layout.deltas, np.int64)).to(dev)  # (a writable copy)
            key_off = torch.empty(self.layout.num_partitions + 1, dtype=torch.int64, device=dev)
            _native.call("phb_offsets_from_deltas", _native.ptr(d), self.n,
                         self.layout.num_partitions, _native.ptr(key_off), _native.stream())
            self._dev_key_off = key_off
        if self._dev_entries is None:
            self._dev_entries = device_table(self.table, dev)
        return (self._dev_key_off, self._dev_entries,
                self.seeds.device_matrix() if matrix else None)

    @property
    def num_partitions(self) -> int:
        return self._dev.nparts if self._layout is None else self._layout.num_partitions

    def _query_tables32(self, seeds: torch.Tensor, key_off: torch.Tensor):
        """The compact tables phb_query32 reads, built once per structure:
        (s << 16) | d per seed (phb_seed_table32) and (offset, end) u32
        partition pairs (phb_part_table32). None if an entry does not fit or
        n >= 2^32 (phb_query on the u64 matrix then)."""
        cached = getattr(self, "_tables32", None)
        if cached is not None and cached[0] is seeds:
            return cached[1]
        tables = None
        if self.n < 2**32:
            t32 = torch.empty(seeds.numel(), dtype=torch.int32, device=seeds.device)
            flag = torch.zeros(1, dtype=torch.int32, device=seeds.device)
            nparts = self.num_partitions
            _native.call("phb_seed_table32", _native.ptr(seeds), _native.ptr(key_off), nparts,
                         seeds.numel(), _native.ptr(t32), _native.ptr(flag), _native.stream())
            part2 = torch.empty(2 * nparts, dtype=torch.int32, device=seeds.device)
            _native.call("phb_part_table32", _native.ptr(key_off), nparts, _native.ptr(part2),
                         _native.stream())
            if not int(flag.item()):
                tables = (t32, part2)
        self._tables32 = (seeds, tables)
        return tables

    def query_device(self, keys) -> torch.Tensor:
        """Batched device query -> int64 CUDA tensor (query_many_kernel, _kernels.py:379-397)."""
        dev = _native.require_device()
        key_off, entries, seeds = self._device_state()
        dk = keys if isinstance(keys, DeviceKeys) else to_device(keys, dev)
        out = torch.empty(dk.n, dtype=torch.int64, device=dev)
        P = _native.ptr
        tables = self._query_tables32(seeds, key_off)
        if tables is not None and (not dk.is_u64 or dk.keys64.data_ptr() % 16 == 0):
            t32, part2 = tables
            _native.call("phb_query32", None if dk.is_u64 else P(dk.buf),
                         None if dk.is_u64 else P(dk.offsets),
                         P(dk.keys64) if dk.is_u64 else None, dk.n,
                         self.global_seed & 0xFFFFFFFFFFFFFFFF, self.n, self.num_partitions,
                         P(key_off), P(part2), P(entries), self.bcount, P(t32), P(out),
                         _native.stream())
            return out
        _native.call("phb_query", None if dk.is_u64 else P(dk.buf),
                     None if dk.is_u64 else P(dk.offsets), P(dk.keys64) if dk.is_u64 else None,
                     dk.n, self.global_seed & 0xFFFFFFFFFFFFFFFF, self.n,
                     self.num_partitions, P(key_off), P(entries), self.bcount, P(seeds),
                     1, self.num_partitions, P(out), _native.stream())
        return out

    def query_encoded_device(self, keys) -> torch.Tensor:
        """Batched device query that reads the seeds straight from the encoded
        section (CompactVector.get / RiceVector.get with sampled select,
        encoders.py:89-99, :224-230) instead of a decoded seed matrix."""
        dev = _native.require_device()
        key_off, entries, _ = self._device_state(matrix=False)
        blob, info, num_enc, mono, dsel, dstride = self.seeds.device_encoded()
        dk = keys if isinstance(keys, DeviceKeys) else to_device(keys, dev)
        out = torch.empty(dk.n, dtype=torch.int64, device=dev)
        P = _native.ptr
        _native.call("phb_query_encoded", None if dk.is_u64 else P(dk.buf),
                     None if dk.is_u64 else P(dk.offsets), P(dk.keys64) if dk.is_u64 else None,
                     dk.n, self.global_seed & 0xFFFFFFFFFFFFFFFF, self.n, self.num_partitions,
                     P(key_off), P(entries), self.bcount, P(blob), P(info), num_enc, mono,
                     None if dsel is None else P(dsel), dstride, P(out), _native.stream())
        return out

    def query_many(self, keys) -> np.ndarray:
        return self.query_device(keys).cpu().numpy()

    def query(self, key) -> int:
        if isinstance(key, str):
            key = key.encode("utf-8")
        return int(self.query_many([bytes(key)])[0])

    def verify_device(self, out: torch.Tensor) -> bool:
        """Bijection of device outputs onto [0, n) (K8, replaces mphf.py:147-151)."""
        if out.numel() != self.n:
            return False
        dev = out.device
        bitmap = torch.zeros((self.n + 31) // 32, dtype=torch.int32, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        _native.call("phb_verify", _native.ptr(out), out.numel(), self.n, _native.ptr(bitmap),
                     _native.ptr(bad), _native.stream())
        return int(bad.item()) == 0

    def is_bijection_on(self, keys) -> bool:
        return self.verify_device(self.query_device(keys))

    # ---- format ---------------------------------------------------------
    def _serialized_body(self) -> bytes:
        if self._body is None:
            from .partitioning import pack_deltas

            width, packed = pack_deltas(self.layout.deltas)
            spec = self.table.spec
            self._body = (_header(self.n, self.layout.num_partitions, self.lambda_,
                                  self.partition_size, spec, self.global_seed)
                          + struct.pack("<B", width) + packed + struct.pack("<I", self.bcount)
                          + self.seeds.section())
        return self._body

    def bits_per_key(self) -> float:
        return (len(self._serialized_body()) + 8 - HEADER_BYTES) * 8 / self.n

    def serialize(self) -> bytes:
        body = self._serialized_body()
        fut = getattr(self, "_ck_future", None)
        ck = fut.result() if fut is not None else _checksum(body)
        return bytes(body) + struct.pack("<Q", ck)

    def save(self, path) -> None:
        with open(path, "wb") as f:
            f.write(self.serialize())

    @classmethod
    def deserialize(cls, data: bytes) -> "Mphf":
        """mphf.py:181-223: validate magic, version, checksum, then parse."""
        data = bytes(data)
        if len(data) < HEADER_BYTES + 8:
            raise FormatError("input shorter than any valid structure")
        if data[:4] != MAGIC:
            raise FormatError("bad magic")
        (version,) = struct.unpack_from("<I", data, 4)
        if version != VERSION:
            raise FormatError(f"unsupported version {version}")
        (stored,) = struct.unpack_from("<Q", data, len(data) - 8)
        body = memoryview(data)[:-8]  # zero-copy: checksum, parse and body share the bytes
        if _checksum(body) != stored:
            raise FormatError("checksum mismatch")
        try:
            n, nparts, lambda_, psize, kind_code, epsilon, global_seed, width = struct.unpack_from(
                "<QQddBdQB", data, 8)
            at = HEADER_FIXED + 1
            nbytes = ((nparts + 1) * width + 7) // 8
            deltas = unpack_deltas(width, data[at: at + nbytes], nparts + 1)
            at += nbytes
            (bcount,) = struct.unpack_from("<I", data, at)
            at += 4
            if kind_code >= len(KINDS):
                raise FormatError("unknown assignment kind")
            store, at = parse_section(data, at, nparts, bcount)
            if at != len(data) - 8:
                raise FormatError("trailing bytes after seed section")
        except (struct.error, ValueError, IndexError) as exc:
            if isinstance(exc, FormatError):
                raise
            raise FormatError(f"malformed structure: {exc}") from exc
        deltas.setflags(write=False)
        layout = PartitionLayout(n=n, num_partitions=nparts, deltas=deltas)
        table = tabulate(AssignmentSpec(KINDS[kind_code], epsilon))
        f = cls(global_seed, layout, table, bcount, store, lambda_, psize)
        f._body = body
        return f

    @classmethod
    def load(cls, path) -> "Mphf":
        with open(path, "rb") as f:
            return cls.deserialize(f.read())


def build(keys, config: BuildConfig | None = None) -> Mphf:
    """Construct an Mphf over distinct keys on the device (mphf.py:236-290).

    keys: a KeyCorpus, an iterable of bytes/str, or a uint64 array / tensor
    (host or CUDA; 64-bit keys hash as their 8-byte little-endian string).
    """
    config = config or BuildConfig()
    if hasattr(keys, "__len__") and len(keys) == 0:  # host-side, like the reference (mphf.py:245)
        raise InvalidConfig("need at least one key")
    dev = _native.require_device()
    t0 = time.perf_counter()
    dk, chunks = to_device_chunked(keys, dev)
    if dk.n < 1:
        raise InvalidConfig("need at least one key")
    engine = BuildEngine(config, dev)
    last: str | None = None
    for attempt in range(MAX_ATTEMPTS):
        seed = config.global_seed + attempt
        res = engine.run(dk, seed, chunks=chunks)
        chunks = None  # a retry finds every key on the device
        if isinstance(res, tuple):
            bad, code = res
            reason = "unseparable duplicate hashes" if code == 1 else "seed cap hit"
            last = f"partition {bad}: {reason}"
            continue
        stats = BuildStats(attempts=attempt + 1, trials_total=res.trials_total,
                           trials_per_key=res.trials_total / dk.n, build_seconds=0.0)
        f = Mphf._from_device(res, config, engine, stats)
        stats.build_seconds = time.perf_counter() - t0
        return f
    raise DuplicateKeys(
        f"construction failed after {MAX_ATTEMPTS} seeds ({SeedExhausted(last)}); "
        "input most likely contains duplicate keys")


def query(f: Mphf, key) -> int:
    return f.query(key)


def serialize(f: Mphf) -> bytes:
    return f.serialize()


def deserialize(data: bytes) -> Mphf:
    return Mphf.deserialize(data)


def bits_per_key(f: Mphf) -> float:
    return f.bits_per_key()
