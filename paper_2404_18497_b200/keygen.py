"""Key containers: the input ABI of the construction path.

``KeyCorpus`` mirrors pilothash.keygen.KeyCorpus (keygen.py:25-57): one
flat uint8 buffer plus int64 offsets[n+1]. In addition, 64-bit keys are
accepted directly (numpy / torch uint64 or int64 arrays, host or CUDA):
key i is defined as its 8-byte little-endian string, which is exactly what
the reference hashes for ``KeyCorpus(keys.view(uint8), 8 * arange(n+1))``
(SURVEY.md §0 finding 4). Such arrays take the u64 fast path on device.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator

import threading

import numpy as np
import torch

MIN_LEN = 10
MAX_LEN = 50
CHAR_LO = 33
CHAR_HI = 126
_DEDUP_SEED = 0x5EEDC0DE


@dataclass(frozen=True)
class KeyCorpus:
    buf: np.ndarray      # uint8, keys back to back
    offsets: np.ndarray  # int64, len(keys) + 1

    def __len__(self) -> int:
        return len(self.offsets) - 1

    def __getitem__(self, i: int) -> bytes:
        return self.buf[self.offsets[i]: self.offsets[i + 1]].tobytes()

    def __iter__(self) -> Iterator[bytes]:
        return (self[i] for i in range(len(self)))

    @classmethod
    def from_keys(cls, keys: Iterable[bytes | str]) -> "KeyCorpus":
        blobs = [k.encode("utf-8") if isinstance(k, str) else bytes(k) for k in keys]
        offsets = np.zeros(len(blobs) + 1, dtype=np.int64)
        if blobs:
            np.cumsum(np.fromiter((len(b) for b in blobs), np.int64, len(blobs)), out=offsets[1:])
        buf = np.frombuffer(b"".join(blobs), dtype=np.uint8).copy()
        return cls(buf, offsets)

    @classmethod
    def from_u64(cls, keys: np.ndarray) -> "KeyCorpus":
        """The reference's byte-string view of 64-bit keys (8-byte LE each)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        return cls(keys.view(np.uint8).copy(), np.arange(len(keys) + 1, dtype=np.int64) * 8)

    def save(self, path) -> None:
        with open(path, "wb") as f:
            for key in self:
                f.write(key)
                f.write(b"\n")

    @classmethod
    def load(cls, path) -> "KeyCorpus":
        with open(path, "rb") as f:
            return cls.from_keys(f.read().splitlines())


def as_corpus(keys) -> KeyCorpus:
    if isinstance(keys, KeyCorpus):
        return keys
    if isinstance(keys, (np.ndarray, torch.Tensor)):
        return KeyCorpus.from_u64(np.asarray(keys.cpu() if isinstance(keys, torch.Tensor) else keys))
    return KeyCorpus.from_keys(keys)


@dataclass
class DeviceKeys:
    """Keys resident on the device: either u64 (keys64) or bytes (buf, offsets)."""

    n: int
    keys64: torch.Tensor | None = None
    buf: torch.Tensor | None = None
    offsets: torch.Tensor | None = None
    h2d_bytes: int = 0

    @property
    def is_u64(self) -> bool:
        return self.keys64 is not None


def _as_u64_tensor(t: torch.Tensor) -> torch.Tensor:
    if t.dtype in (torch.uint64, torch.int64):
        return t.contiguous()
    raise TypeError(f"64-bit key arrays must be uint64/int64, got {t.dtype}")


# ---- host ingestion: pageable host arrays reach the device through pinned
# staging buffers, with the host-side copy (threaded) of chunk i+1 overlapped
# with the DMA of chunk i. torch's pageable .to(device) runs at ~11 GB/s on
# the B200 boxes (800 MB in 71 ms); staged, the copy approaches the PCIe rate.
_STAGE_BYTES = 64 << 20
_STAGE_SLOTS = 3
_stage = {"bufs": None, "events": None, "pool": None}
_stage_lock = threading.Lock()  # the staging buffers are shared: one copy at a time


def _stage_init():
    if _stage["bufs"] is None:
        import os
        from concurrent.futures import ThreadPoolExecutor

        _stage["bufs"] = [torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True)
                          for _ in range(_STAGE_SLOTS)]
        _stage["events"] = [None] * _STAGE_SLOTS
        _stage["pool"] = ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1)))
    return _stage


def staged_h2d(host: np.ndarray, device: torch.device, pad: int = 0) -> torch.Tensor:
    """Copy a C-contiguous host array to a new uint8 device tensor (its bytes),
    followed by `pad` zero bytes."""
    src = np.ascontiguousarray(host).reshape(-1).view(np.uint8)
    nbytes = src.size
    out = torch.empty(max(nbytes + pad, 1), dtype=torch.uint8, device=device)
    if pad:
        out[nbytes:].zero_()
    if nbytes == 0:
        return out[: nbytes + pad]
    with _stage_lock:
        _staged_copy(src, out, nbytes, device)
    return out if pad else out[:nbytes]


def _staged_copy(src: np.ndarray, out: torch.Tensor, nbytes: int, device) -> None:
    for _ in _staged_chunks(src, out, nbytes, device, torch.cuda.current_stream(device)):
        pass


def _staged_chunks(src: np.ndarray, out: torch.Tensor, nbytes: int, device, stream):
    """Generator: per staging chunk, the threaded host copy into a pinned slot
    and the DMA into out on `stream`; yields (byte begin, byte end, event)."""
    st = _stage_init()
    pool = st["pool"]
    workers = pool._max_workers
    for k, a in enumerate(range(0, nbytes, _STAGE_BYTES)):
        b = min(a + _STAGE_BYTES, nbytes)
        slot = k % _STAGE_SLOTS
        ev = st["events"][slot]
        if ev is not None:
            ev.synchronize()  # the DMA that last read this staging buffer is done
        dst = st["bufs"][slot].numpy()[: b - a]
        step = -(-(b - a) // workers)
        futs = [pool.submit(np.copyto, dst[o: o + step], src[a + o: a + o + step])
                for o in range(0, b - a, step)]
        for fu in futs:
            fu.result()
        with torch.cuda.stream(stream):
            out[a:b].copy_(st["bufs"][slot][: b - a], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        st["events"][slot] = ev
        yield a, b, ev


_COPY_CHUNK_KEYS = 8 << 20  # 64 MB of u64 keys per chunk (even: 16-byte aligned chunk starts)
_copy_streams: dict = {}


def to_device_chunked(keys, device: torch.device):
    """(DeviceKeys, chunks) for pinned host u64 tensors: the copy is issued as
    chunks on a side stream, chunks = [(begin, end, event)], so the grouping
    pass can consume each chunk as soon as it lands (BuildEngine.run). Any
    other input: (to_device(keys), None)."""
    if (isinstance(keys, torch.Tensor) and not keys.is_cuda and keys.is_pinned()
            and keys.dtype in (torch.int64, torch.uint64) and keys.dim() == 1
            and keys.is_contiguous() and keys.numel() > _COPY_CHUNK_KEYS):
        n = keys.numel()
        out = torch.empty(n, dtype=torch.int64, device=device)
        src = keys.view(torch.int64)
        cs = _copy_streams.get(device)
        if cs is None:
            cs = _copy_streams[device] = torch.cuda.Stream(device)
        cs.wait_stream(torch.cuda.current_stream(device))  # `out` is allocated on the compute stream
        chunks = []
        with torch.cuda.stream(cs):
            for a in range(0, n, _COPY_CHUNK_KEYS):
                b = min(a + _COPY_CHUNK_KEYS, n)
                out[a:b].copy_(src[a:b], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                chunks.append((a, b, ev))
        out.record_stream(cs)
        return DeviceKeys(n, keys64=out, h2d_bytes=n * 8), chunks
    host = None
    if isinstance(keys, np.ndarray) and keys.dtype in (np.uint64, np.int64) and keys.ndim == 1:
        host = np.ascontiguousarray(keys)
    elif (isinstance(keys, torch.Tensor) and not keys.is_cuda and not keys.is_pinned()
          and keys.dtype in (torch.int64, torch.uint64) and keys.dim() == 1):
        host = keys.contiguous().view(torch.int64).numpy()
    if host is not None and host.size > _COPY_CHUNK_KEYS:
        # pageable keys: the staged copy runs chunk by chunk as the build pulls
        # the chunks, so the host copy of chunk k+1 overlaps chunk k's DMA and
        # grouping pass
        n = host.size
        out = torch.empty(n, dtype=torch.int64, device=device)
        cs = _copy_streams.get(device)
        if cs is None:
            cs = _copy_streams[device] = torch.cuda.Stream(device)
        cs.wait_stream(torch.cuda.current_stream(device))
        out.record_stream(cs)

        def chunks():
            with _stage_lock:
                src = host.view(np.uint8)
                for a, b, ev in _staged_chunks(src, out.view(torch.uint8), n * 8, device, cs):
                    yield a // 8, b // 8, ev
        return DeviceKeys(n, keys64=out, h2d_bytes=n * 8), chunks()
    return to_device(keys, device), None


def _host_to_device_u64(t: torch.Tensor, device: torch.device) -> torch.Tensor:
    if t.is_cuda:
        return t.to(device)
    if t.is_pinned():
        return t.to(device, non_blocking=True)
    return staged_h2d(t.numpy(), device).view(torch.int64)


def to_device(keys, device: torch.device) -> DeviceKeys:
    """Stage keys on the device. u64 arrays -> fast path; everything else -> bytes."""
    if isinstance(keys, DeviceKeys):
        return keys
    if isinstance(keys, torch.Tensor):
        t = _as_u64_tensor(keys.reshape(-1))
        moved = 0 if t.is_cuda else t.numel() * 8
        return DeviceKeys(int(t.numel()), keys64=_host_to_device_u64(t, device), h2d_bytes=moved)
    if isinstance(keys, np.ndarray):
        if keys.dtype not in (np.uint64, np.int64):
            raise TypeError(f"64-bit key arrays must be uint64/int64, got {keys.dtype}")
        host = np.ascontiguousarray(keys).reshape(-1)
        return DeviceKeys(len(host), keys64=staged_h2d(host, device).view(torch.int64),
                          h2d_bytes=int(host.nbytes))
    corpus = as_corpus(keys)
    buf = corpus.buf if corpus.buf.size else np.zeros(8, dtype=np.uint8)
    off = np.ascontiguousarray(corpus.offsets, dtype=np.int64)
    return DeviceKeys(len(corpus), buf=staged_h2d(buf, device),
                      offsets=staged_h2d(off, device).view(torch.int64),
                      h2d_bytes=int(corpus.buf.nbytes + corpus.offsets.nbytes))


def synth_u64(n: int, offset: int = 0) -> np.ndarray:
    """Distinct synthetic 64-bit keys mix64(offset + i) (host restatement of
    phb_synth_keys; mix64 is a bijection, so no dedup is needed)."""
    z = (np.arange(n, dtype=np.uint64) + np.uint64(offset & 0xFFFFFFFFFFFFFFFF))
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def synth_u64_device(n: int, offset: int = 0, device=None) -> torch.Tensor:
    """phb_synth_keys on the device -> int64 view of u64 keys."""
    from . import _native

    dev = device or _native.require_device()
    out = torch.empty(n, dtype=torch.int64, device=dev)
    _native.call("phb_synth_keys", _native.ptr(out), n, offset & 0xFFFFFFFFFFFFFFFF,
                 _native.stream())
    return out


def gen_keys(n: int, prng_seed: int) -> KeyCorpus:
    """n distinct random printable keys, lengths in [10, 50] (keygen.py:78-111).

    Same generator stream as the reference; distinctness is enforced on a
    128-bit device fingerprint (seed 0x5EEDC0DE) like keygen.py:66-75.
    """
    from .hashing import master_hash_many

    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.default_rng(prng_seed)
    lengths = rng.integers(MIN_LEN, MAX_LEN + 1, size=n, dtype=np.int64)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lengths, out=offsets[1:])
    buf = rng.integers(CHAR_LO, CHAR_HI + 1, size=int(offsets[-1]), dtype=np.uint8)
    while True:
        his, los = master_hash_many(buf, offsets, _DEDUP_SEED)
        order = np.lexsort((los, his))
        same = (his[order][1:] == his[order][:-1]) & (los[order][1:] == los[order][:-1])
        dups = np.sort(order[1:][same])
        if len(dups) == 0:
            return KeyCorpus(buf, offsets)
        new_lengths = lengths.copy()
        for i in dups:
            new_lengths[i] = rng.integers(MIN_LEN, MAX_LEN + 1)
        pieces = []
        at = 0
        for i in range(n):
            if at < len(dups) and dups[at] == i:
                pieces.append(rng.integers(CHAR_LO, CHAR_HI + 1, size=int(new_lengths[i]),
                                           dtype=np.uint8))
                at += 1
            else:
                pieces.append(buf[offsets[i]: offsets[i + 1]])
        buf = np.concatenate(pieces)
        lengths = new_lengths
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lengths, out=offsets[1:])
