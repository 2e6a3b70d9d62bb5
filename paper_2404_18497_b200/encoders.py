"""Seed stores: the encoded per-bucket seeds, their byte format and decode.

Mirrors pilothash.encoders (encoders.py:1-381). Encoding runs on the device
(csrc/encode.cu: per-column Compact width / exact Golomb-Rice parameter,
LSB-first fields, unary highs, every-1024th-one select samples, block
headers); decoding back to the seed matrix runs on the device too
(csrc/decode.cu). This module holds the host-side views over the encoded
bytes: block parsing (``deserialize_seeds``, encoders.py:258-280 /
:358-376), scalar random access (``get`` / ``seed_at``, encoders.py:89-99,
:224-230, :305-307) and the store containers.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native

SELECT_SAMPLE = 1024
KIND_COMPACT = 0
KIND_RICE = 1
FULL64 = (1 << 64) - 1


def _bits(data: bytes, pos: int, width: int) -> int:
    if width == 0:
        return 0
    a, b = pos >> 3, (pos + width + 7) >> 3
    return (int.from_bytes(data[a:b], "little") >> (pos & 7)) & ((1 << width) - 1)


@dataclass
class CompactVector:
    width: int
    count: int
    data: bytes  # ceil(count * width / 8) payload bytes

    @classmethod
    def encode(cls, values: np.ndarray) -> "CompactVector":
        store = _encode_single(values, rice=False)
        return store.encoders[0]

    def get(self, i: int) -> int:
        if not 0 <= i < self.count:
            raise IndexError("compact index out of range")
        return _bits(self.data, i * self.width, self.width)

    def decode_all(self) -> np.ndarray:
        return InterleavedSeeds([self], self.count, 1).decode_matrix()[:, 0]

    @property
    def payload_bits(self) -> int:
        return self.count * self.width

    def block(self) -> bytes:
        return struct.pack("<BBQ", KIND_COMPACT, self.width, self.count) + self.data


@dataclass
class RiceVector:
    b: int
    count: int
    lows: bytes          # ceil(count * b / 8) bytes
    highs: bytes         # ceil(highs_nbits / 8) bytes, unary stream
    highs_nbits: int
    samples: np.ndarray  # int64 positions of every 1024th one
    _words: np.ndarray | None = field(default=None, repr=False)

    @classmethod
    def encode(cls, values: np.ndarray) -> "RiceVector":
        store = _encode_single(values, rice=True)
        return store.encoders[0]

    def _highs_words(self) -> np.ndarray:
        if self._words is None:
            nw = (self.highs_nbits + 63) >> 6
            self._words = np.frombuffer(bytes(self.highs).ljust(nw * 8, b"\0"),
                                        "<u8").astype(np.uint64)
        return self._words

    def select1(self, k: int) -> int:
        """Position of the (k+1)-th one via the sampled index (encoders.py:129-145)."""
        if k < 0 or (k >> 10) >= len(self.samples):
            raise IndexError("select rank out of range")
        words = self._highs_words()
        spos = int(self.samples[k >> 10])
        need = k - ((k >> 10) << 10) + 1
        w = spos >> 6
        word = int(words[w]) & (FULL64 << (spos & 63)) & FULL64
        while True:
            c = word.bit_count()
            if c >= need:
                for _ in range(need - 1):
                    word &= word - 1
                return (w << 6) + ((word & -word).bit_length() - 1)
            need -= c
            w += 1
            word = int(words[w])

    def next_one(self, pos: int) -> int:
        words = self._highs_words()
        w = pos >> 6
        word = int(words[w]) & (FULL64 << (pos & 63)) & FULL64
        while word == 0:
            w += 1
            word = int(words[w])
        return (w << 6) + ((word & -word).bit_length() - 1)

    def get(self, i: int) -> int:
        if not 0 <= i < self.count:
            raise IndexError("rice index out of range")
        prev = self.select1(i - 1) if i > 0 else -1
        pos = self.next_one(prev + 1)
        return ((pos - prev - 1) << self.b) | _bits(self.lows, i * self.b, self.b)

    def decode_all(self) -> np.ndarray:
        return InterleavedSeeds([self], self.count, 0).decode_matrix()[:, 0]

    @property
    def payload_bits(self) -> int:
        return self.count * self.b + self.highs_nbits

    def block(self) -> bytes:
        return (struct.pack("<BBQ", KIND_RICE, self.b, self.count)
                + struct.pack("<QI", self.highs_nbits, len(self.samples))
                + np.asarray(self.samples, "<i8").tobytes() + self.lows + self.highs)


Encoder = CompactVector | RiceVector


def _parse_encoder(data: bytes, at: int) -> tuple[Encoder, int, tuple]:
    """One block (encoders.py:258-280); also returns its payload geometry."""
    kind, param, count = struct.unpack_from("<BBQ", data, at)
    at += 10
    if kind == KIND_COMPACT:
        nbytes = (count * param + 7) // 8
        if at + nbytes > len(data):
            raise ValueError("truncated compact payload")
        enc = CompactVector(param, count, memoryview(data)[at: at + nbytes])
        return enc, at + nbytes, (0, param, count, at, 0, 0)
    if kind != KIND_RICE:
        raise ValueError(f"unknown encoder kind {kind}")
    if param > 64:
        raise ValueError("rice parameter out of range")
    highs_nbits, nsamples = struct.unpack_from("<QI", data, at)
    at += 12
    if at + 8 * nsamples > len(data):
        raise ValueError("truncated select samples")
    samples = np.frombuffer(data[at: at + 8 * nsamples], dtype="<i8").astype(np.int64)
    at += 8 * nsamples
    low_bytes = (count * param + 7) // 8
    high_bytes = (highs_nbits + 7) // 8
    if at + low_bytes + high_bytes > len(data):
        raise ValueError("truncated rice payload")
    lows = memoryview(data)[at: at + low_bytes]  # zero-copy views of the parsed bytes
    highs = memoryview(data)[at + low_bytes: at + low_bytes + high_bytes]
    geo = (1, param, count, at, at + low_bytes, highs_nbits)
    return RiceVector(param, count, lows, highs, highs_nbits, samples), at + low_bytes + high_bytes, geo


def _col_info(encs, geo_at0=None) -> np.ndarray:
    """8 int64 per encoder for phb_decode_seeds / phb_query_encoded: kind,
    width or b, count, payload byte, highs byte, highs_nbits, samples byte,
    nsamples, relative to a blob holding the encoder blocks back to back."""
    rows = []
    at = 0
    for e in encs:
        if isinstance(e, CompactVector):
            rows.append([0, e.width, e.count, at + 10, 0, 0, 0, 0])
        else:
            pay = at + 22 + 8 * len(e.samples)
            rows.append([1, e.b, e.count, pay, pay + len(e.lows), e.highs_nbits, at + 22,
                         len(e.samples)])
        at += _block_len(e)
    return np.ascontiguousarray(np.array(rows, dtype=np.int64).reshape(-1, 8))


def _block_len(e) -> int:
    if isinstance(e, CompactVector):
        return 10 + len(e.data)
    return 22 + 8 * len(e.samples) + len(e.lows) + len(e.highs)


def _blocks_bytes(store) -> memoryview:
    """The encoder blocks back to back = the serialized section minus its u32 count."""
    return memoryview(store.section())[4:]


def _device_blocks(store):
    """Device copy of the encoder blocks (8-byte aligned, zero tail: the
    kernels read whole aligned u64 words past the last field) + col_info.
    A freshly built structure copies them from its device body; a loaded one
    uploads them once through the pinned staging path. Cached on the store."""
    if store._dev_blocks is None:
        from .keygen import staged_h2d

        dev = _native.require_device()
        encs = store.encoders if isinstance(store, InterleavedSeeds) else [store.encoder]
        src = store._dev_source
        if src is not None:  # (device body, first block byte, end byte)
            body, a, b = src
            d_blob = torch.zeros(b - a + 32, dtype=torch.uint8, device=body.device)
            d_blob[: b - a].copy_(body[a:b])
        else:
            blocks = np.frombuffer(_blocks_bytes(store), dtype=np.uint8)
            d_blob = staged_h2d(blocks, dev, pad=32)
        info = _col_info(encs)
        store._dev_blocks = (d_blob, torch.from_numpy(info).to(dev), info)
    return store._dev_blocks


def _select_dir(d_blob, d_info, hinfo: np.ndarray):
    """(dense select directory, stride) for the Rice encoders (phb_select_index),
    or (None, 1) when the section has none."""
    rice = hinfo[:, 0] == 1
    if not rice.any():
        return None, 1
    stride = int((hinfo[rice, 2].max() + 63) // 64) + 1
    dsel = torch.zeros(len(hinfo) * stride, dtype=torch.int32, device=d_blob.device)
    _native.call("phb_select_index", _native.ptr(d_blob), _native.ptr(d_info), len(hinfo), stride,
                 _native.ptr(dsel), _native.stream())
    return dsel, stride


def _decode(store, nparts: int, bcount: int, mono: bool) -> torch.Tensor:
    """Device decode -> column-major u64 matrix [bcount][nparts] (torch int64 view)."""
    dev = _native.require_device()
    d_blob, _, hinfo = _device_blocks(store)
    out = torch.zeros(bcount * nparts, dtype=torch.int64, device=dev)
    _native.call("phb_decode_seeds", _native.ptr(d_blob), len(hinfo),
                 hinfo.ctypes.data_as(__import__("ctypes").c_void_p), nparts, bcount, int(mono),
                 _native.ptr(out), _native.stream())
    return out.view(bcount, nparts)


@dataclass
class InterleavedSeeds:
    """Encoder i holds the seed of bucket i+1 from every partition (encoders.py:283-311)."""

    encoders: list
    num_partitions: int
    compact_prefix: int
    _section: bytes | None = field(default=None, repr=False)
    _device: torch.Tensor | None = field(default=None, repr=False)
    _encoded: tuple | None = field(default=None, repr=False)
    _dev_blocks: tuple | None = field(default=None, repr=False)
    _dev_source: tuple | None = field(default=None, repr=False)

    @classmethod
    def build(cls, seed_matrix: np.ndarray, compact_prefix: int) -> "InterleavedSeeds":
        m = np.asarray(seed_matrix, dtype=np.uint64)
        nparts, B = m.shape
        return encode_matrix(m, 0, min(compact_prefix, B))

    @property
    def bucket_count(self) -> int:
        return len(self.encoders)

    def seed_at(self, j: int, i: int) -> int:
        return self.encoders[i - 1].get(j)

    def device_matrix(self) -> torch.Tensor:
        """Column-major [B][nparts] u64 seeds on the device (cached)."""
        if self._device is None:
            self._device = _decode(self, self.num_partitions, self.bucket_count, False)
        return self._device

    def device_encoded(self):
        """(section blob, col_info, num encoders, mono) on the device, cached."""
        if self._encoded is None:
            blob, info, hinfo = _device_blocks(self)
            self._encoded = (blob, info, len(self.encoders), 0) + _select_dir(blob, info, hinfo)
        return self._encoded

    def decode_matrix(self) -> np.ndarray:
        if not self.encoders:
            return np.zeros((self.num_partitions, 0), np.uint64)
        return self.device_matrix().t().contiguous().cpu().numpy().view(np.uint64)

    def section(self) -> bytes:
        if self._section is None:
            self._section = struct.pack("<I", len(self.encoders)) + b"".join(
                e.block() for e in self.encoders)
        return self._section


@dataclass
class MonoSeeds:
    """One encoder over all seeds in partition-major order (encoders.py:314-341)."""

    encoder: Encoder
    num_partitions: int
    bucket_count: int
    _section: bytes | None = field(default=None, repr=False)
    _device: torch.Tensor | None = field(default=None, repr=False)
    _encoded: tuple | None = field(default=None, repr=False)
    _dev_blocks: tuple | None = field(default=None, repr=False)
    _dev_source: tuple | None = field(default=None, repr=False)

    @classmethod
    def build(cls, seed_matrix: np.ndarray, rice: bool) -> "MonoSeeds":
        return encode_matrix(np.asarray(seed_matrix, np.uint64), 1, 0 if rice else 1)

    @property
    def encoders(self) -> list:
        return [self.encoder]

    @property
    def compact_prefix(self) -> int:
        return self.bucket_count if isinstance(self.encoder, CompactVector) else 0

    def seed_at(self, j: int, i: int) -> int:
        return self.encoder.get(j * self.bucket_count + (i - 1))

    def device_matrix(self) -> torch.Tensor:
        if self._device is None:
            self._device = _decode(self, self.num_partitions, self.bucket_count, True)
        return self._device

    def device_encoded(self):
        if self._encoded is None:
            blob, info, hinfo = _device_blocks(self)
            self._encoded = (blob, info, 1, 1) + _select_dir(blob, info, hinfo)
        return self._encoded

    def decode_matrix(self) -> np.ndarray:
        return self.device_matrix().t().contiguous().cpu().numpy().view(np.uint64)

    def section(self) -> bytes:
        if self._section is None:
            self._section = struct.pack("<I", 1) + self.encoder.block()
        return self._section


SeedStore = InterleavedSeeds | MonoSeeds


def parse_section(data: bytes, at: int, num_partitions: int, bcount: int):
    """deserialize_seeds (encoders.py:358-376): parse, validate, build the store."""
    (num_enc,) = struct.unpack_from("<I", data, at)
    start = at
    at += 4
    encs = []
    for _ in range(num_enc):
        enc, at, _geo = _parse_encoder(data, at)
        encs.append(enc)
    section = memoryview(data)[start:at]
    if num_enc == 1 and bcount > 1:
        if encs[0].count != num_partitions * bcount:
            raise ValueError("mono encoder count does not match layout")
        store: SeedStore = MonoSeeds(encs[0], num_partitions, bcount, _section=section)
    else:
        if num_enc != bcount or any(e.count != num_partitions for e in encs):
            raise ValueError("interleaved encoder shape does not match layout")
        t = 0
        while t < num_enc and isinstance(encs[t], CompactVector):
            t += 1
        store = InterleavedSeeds(encs, num_partitions, t, _section=section)
    return store, at


def deserialize_seeds(data: bytes, at: int, num_partitions: int, bcount: int):
    return parse_section(data, at, num_partitions, bcount)


def serialize_seeds(store: SeedStore) -> bytes:
    return store.section()


def total_bits(store: SeedStore) -> int:
    return 8 * len(serialize_seeds(store))


def interleave(partition_seeds, compact_prefix: int) -> InterleavedSeeds:
    matrix = np.stack([np.asarray(s, dtype=np.uint64) for s in partition_seeds])
    return InterleavedSeeds.build(matrix, compact_prefix)


# ---- device encode of an arbitrary host matrix (standalone encoder API) ----

def encode_colmajor(seeds_cm: torch.Tensor, nparts: int, bcount: int, mono: int, prefix: int):
    """Encode a device column-major seed matrix; returns (section bytes, store)."""
    dev = seeds_cm.device
    stats = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(int(_native.load().phb_encode_workspace_bytes(nparts, bcount, mono)),
                     dtype=torch.uint8, device=dev)
    summ = np.zeros(8, np.int64)
    import ctypes

    _native.call("phb_encode_plan", _native.ptr(seeds_cm), nparts, bcount, mono, prefix, None,
                 nparts, _native.ptr(stats), None, None, _native.ptr(ws),
                 summ.ctypes.data_as(ctypes.c_void_p), _native.stream())
    total, sec0 = int(summ[0]), int(summ[1])
    blob = torch.empty(((total + 16) + 3) // 4 * 4, dtype=torch.uint8, device=dev)
    _native.call("phb_encode_write", _native.ptr(seeds_cm), nparts, bcount, mono, prefix, None,
                 nparts, _native.ptr(stats), _native.ptr(ws), _native.ptr(blob), blob.numel(),
                 _native.stream())
    section = blob[sec0:total].cpu().numpy().tobytes()
    store, _ = parse_section(section, 0, nparts, bcount)
    store._device = seeds_cm.view(bcount, nparts)
    return section, store


def encode_matrix(matrix: np.ndarray, mono: int, prefix: int) -> SeedStore:
    dev = _native.require_device()
    nparts, B = matrix.shape
    cm = torch.from_numpy(np.ascontiguousarray(matrix.T).view(np.int64).reshape(-1)).to(dev)
    if nparts == 0 or B == 0:
        raise ValueError("empty seed matrix")
    _, store = encode_colmajor(cm, nparts, B, mono, prefix)
    return store


def _encode_single(values: np.ndarray, rice: bool) -> InterleavedSeeds:
    v = np.asarray(values, dtype=np.uint64).reshape(-1, 1)
    return encode_matrix(v, 0, 0 if rice else 1)
