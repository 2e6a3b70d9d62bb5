"""Drop-in replacement for ``pilothash._kernels`` (the reference's numba
operator module, pkg/src/pilothash/_kernels.py), backed by libphobic_b200.so.

Same names, argument meaning and in-place output semantics as the
reference's three entry points; host numpy arrays in and out, staged on the
device around each call. Installing this file as ``pilothash/_kernels.py``
 runs the reference package on the B200 kernels.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native

POSITION_SALT = np.uint64(0x9E3779B97F4A7C15)  # _kernels.py:30, read by builder.py:132
BUCKET_SALT = np.uint64(0xC2B2AE3D27D4EB4F)    # _kernels.py:29


def _dev(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(a).to(_native.require_device())


def murmur3_many(buf, offsets, seed, out_hi, out_lo) -> None:
    """_kernels.py:89-146."""
    n = len(offsets) - 1
    if n <= 0:
        return
    b = _dev(buf if len(buf) else np.zeros(8, np.uint8))
    o = _dev(np.asarray(offsets, np.int64))
    hi = torch.empty(n, dtype=torch.int64, device=o.device)
    lo = torch.empty_like(hi)
    _native.call("phb_murmur3_many", _native.ptr(b), _native.ptr(o), n, int(seed) & (2**64 - 1),
                 _native.ptr(hi), _native.ptr(lo), _native.stream())
    out_hi[:] = hi.cpu().numpy().view(np.uint64)
    out_lo[:] = lo.cpu().numpy().view(np.uint64)


def build_partition_range(his, los, key_off, p_lo, p_hi, entries, bcount, seed_cap, tie_desc,
                          seeds_out, trials_out, status_out) -> None:
    """_kernels.py:221-371 (outputs written in place, like the reference).

    Only the rows this call owns are staged and written back: keys
    [key_off[p_lo], key_off[p_hi]) go up, seeds / trials rows [p_lo, p_hi)
    and status[p_lo:p_hi] come back. builder.build_all_partitions
    (builder.py:260-271) calls this concurrently from a thread pool with
    disjoint partition ranges over shared output arrays; the native call and
    the copies release the GIL, so writing back whole arrays would clobber
    the other threads' rows."""
    p_lo, p_hi, bcount = int(p_lo), int(p_hi), int(bcount)
    if p_hi <= p_lo:
        return
    key_off = np.asarray(key_off, np.int64)
    k0, k1 = int(key_off[p_lo]), int(key_off[p_hi])
    dev = _native.require_device()
    ko = _dev(key_off)
    h = _dev(np.asarray(his[k0:k1] if k1 > k0 else np.zeros(1, np.uint64)))
    l = _dev(np.asarray(los[k0:k1] if k1 > k0 else np.zeros(1, np.uint64)))
    e = _dev(np.asarray(entries, np.float64))
    rows = p_hi - p_lo
    s = torch.zeros(rows * bcount, dtype=torch.int64, device=dev)
    t = torch.zeros(rows * bcount, dtype=torch.int64, device=dev)
    st = torch.zeros(rows, dtype=torch.uint8, device=dev)
    # the C-ABI indexes keys by key_off and outputs by partition j: shift the
    # base pointers so that index k0 / row p_lo land on element 0
    _native.call("phb_build_partition_range", _native.ptr(h) - 8 * k0, _native.ptr(l) - 8 * k0,
                 _native.ptr(ko), p_lo, p_hi, _native.ptr(e), bcount, int(seed_cap),
                 int(bool(tie_desc)), _native.ptr(s) - 8 * p_lo * bcount,
                 _native.ptr(t) - 8 * p_lo * bcount, _native.ptr(st) - p_lo, _native.stream())
    seeds_out[p_lo * bcount:p_hi * bcount] = s.cpu().numpy().view(np.uint64)
    trials_out[p_lo * bcount:p_hi * bcount] = t.cpu().numpy()
    status_out[p_lo:p_hi] = st.cpu().numpy()


def query_many_kernel(his, los, n, nparts, deltas, entries, bcount, seed_mat, out) -> None:
    """_kernels.py:379-397."""
    nq = len(his)
    if nq == 0:
        return
    h, l = _dev(his), _dev(los)
    d = _dev(np.asarray(deltas, np.int64))
    e = _dev(np.asarray(entries, np.float64))
    m = _dev(np.asarray(seed_mat, np.uint64))
    o = torch.empty(nq, dtype=torch.int64, device=h.device)
    _native.call("phb_query_many", _native.ptr(h), _native.ptr(l), nq, int(n), int(nparts),
                 _native.ptr(d), _native.ptr(e), int(bcount), _native.ptr(m), _native.ptr(o),
                 _native.stream())
    out[:] = o.cpu().numpy()
