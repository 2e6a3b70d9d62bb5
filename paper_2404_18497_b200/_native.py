"""ctypes binding of libphobic_b200.so (the C-ABI declared in include/phobic.h).

There is no fallback: if the library is missing or no CUDA device is
visible, every entry point raises. PyTorch is used only for device buffers
and the current stream.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import torch

import os

LIB_PATH = Path(os.environ.get("PHB_LIB") or Path(__file__).resolve().parent / "libphobic_b200.so")

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
SZ = ctypes.c_size_t
INT = ctypes.c_int

# name -> argtypes (restype int unless noted)
SIGNATURES = {
    "phb_murmur3_many": [P, P, I64, U64, P, P, P],
    "phb_murmur3_u64": [P, I64, U64, P, P, P],
    "phb_build_partition_range": [P, P, P, I64, I64, P, I32, I64, I32, P, P, P, P],
    "phb_query_many": [P, P, I64, I64, I64, P, P, I32, P, P, P],
    "phb_bucket_ids": [P, I64, P, I32, P, P],
    "phb_hash_count": [P, P, P, I64, U64, I64, P, P],
    "phb_layout": [P, I64, I64, I64, I64, I64, P, P, P, P],
    "phb_hash_count_store": [P, P, I64, U64, I64, P, P, P],
    "phb_scatter_hashed": [P, I64, I64, P, I32, P, P, P, P],
    "phb_scatter": [P, P, P, I64, U64, I64, P, I32, P, P, P, P, P],
    "phb_scatter_padded": [P, I64, U64, I64, P, I32, I32, I32, P, P, P, P, P],
    "phb_padded_counts": [P, I64, I32, P, P, P],
    "phb_search_strided": [P, P, P, I64, I64, I64, I32, I64, I32, I64, P, I64, I64, P, P, P, P, P,
                           I64, P],
    "phb_search": [P, P, P, I64, I64, I64, I32, I64, I32, I64, P, I64, I64, P, P, P, P, P, P],
    "phb_encode_plan": [P, I64, I32, I32, I32, P, I64, P, P, P, P, P, P],
    "phb_encode_write": [P, I64, I32, I32, I32, P, I64, P, P, P, SZ, P],
    "phb_decode_seeds": [P, I64, P, I64, I32, I32, P, P],
    "phb_encode_shard_stats": [P, I64, I32, I32, P, P],
    "phb_encode_shard_plan": [P, I64, I64, I64, I32, I32, I32, P, P, P, P, P, P],
    "phb_encode_shard_write": [P, I64, I64, I64, I32, I32, I32, P, P, P, I32, P, P, SZ, P],
    "phb_query": [P, P, P, I64, U64, I64, I64, P, P, I32, P, I64, I64, P, P],
    "phb_query32": [P, P, P, I64, U64, I64, I64, P, P, P, I32, P, P, P],
    "phb_seed_table32": [P, P, I64, I64, P, P, P],
    "phb_part_table32": [P, I64, P, P],
    "phb_query_encoded": [P, P, P, I64, U64, I64, I64, P, P, I32, P, P, I32, I32, P, I64, P, P],
    "phb_select_index": [P, P, I64, I64, P, P],
    "phb_verify": [P, I64, I64, P, P, P],
    "phb_offsets_from_deltas": [P, I64, I64, P, P],
    "phb_device_sms": [],
    "phb_synth_keys": [P, I64, U64, P],
    "phb_regroup": [P, P, P, I64, I64, P, P, P, P],
    "phb_scatter_p2p": [P, P, P, I64, U64, I64, P, I32, P, P, P, P, I32, P, P],
    "phb_ipc_alloc": [SZ, P],
    "phb_ipc_free": [P],
    "phb_ipc_handle": [P, P],
    "phb_ipc_open": [P, P],
    "phb_ipc_close": [P],
    "phb_sync": [P],
    "phb_search_stats": [P, INT],
}
OTHER = {
    "phb_version": ([], ctypes.c_char_p),
    "phb_error_string": ([INT], ctypes.c_char_p),
    "phb_encode_workspace_bytes": ([I64, I32, I32], SZ),
    "phb_launch_count": ([], ctypes.c_ulonglong),
}

_lib = None


class NativeError(RuntimeError):
    """A CUDA / launch error reported by the native layer."""


def load():
    """Load the shared library (no CUDA context needed)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = INT
        for name, (args, res) in OTHER.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def require_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2404_18497_b200 runs its construction path on a CUDA device (B200); "
            "no CUDA device is visible and there is no CPU fallback"
        )
    return torch.device("cuda", torch.cuda.current_device())


def lib():
    require_device()
    return load()


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().phb_error_string(rc).decode()
        raise NativeError(f"{what} failed: {msg} (code {rc})")


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def launch_count() -> int:
    """Kernel launches issued by libphobic_b200.so so far in this process."""
    return int(load().phb_launch_count())


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
