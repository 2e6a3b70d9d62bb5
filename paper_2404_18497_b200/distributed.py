"""Multi-GPU PHOBIC construction: one process per GPU, NCCL over NVLink.

SURVEY.md §8(e). The result is independent of the number of ranks G: every
quantity that defines the MPHF (n, nparts, partition index, bucket ids,
partition offsets, seeds) is global, and the bytes equal those of a
single-GPU build over the concatenated keys.

Per attempt (global_seed + attempt, the reference's retry, mphf.py:251-261):
  1. K1 on the local shard: per-partition counts over the GLOBAL nparts.
  2. all_gather of the count vectors -> C[s][j] (G x nparts int32). Every
     rank derives the global layout (key offsets, deltas, max |delta|).
  3. K3 on the local shard, grouped by partition with local offsets: since
     j = mulhi(hi, nparts) is monotone in hi and rank g owns the contiguous
     partition range [g*nparts/G, (g+1)*nparts/G), the local records are
     also grouped by destination rank.
  4. all_to_all_single of the (lo, bucket-id) records: 10 B/key, no
     re-hashing at the destination (string keys never move).
  5. regroup: the G received chunks (each partition-sorted) are merged into
     one partition-grouped array (a segmented copy, phb_regroup).
  6. K4 search on the owned partitions; all_reduce of the failure flag
     (collective retry) and of the trial count.
  7. sharded K5: the column statistics are all_reduced, every rank plans the
     same global geometry and writes its own rows' fields at their global bit
     addresses, and a uint8 SUM all_reduce ORs the bodies (each bit has one
     writer), so every rank holds the identical body and a queryable Mphf
     (encode="gather": all_gather of the seed rows + replicated K5).

The kernels are reached through an ``ops`` object. ``DeviceOps`` (default)
calls the C-ABI; the CPU tests inject an oracle-backed implementation to
check this orchestration with the gloo backend (tests/test_distributed.py).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .builder import BuildConfig, InvalidConfig, SeedExhausted, device_table
from .keygen import DeviceKeys, to_device
from .partitioning import num_partitions_for

MAX_ATTEMPTS = 4


def owner_bounds(nparts: int, world: int) -> list[int]:
    """Partition range of rank g is [b[g], b[g+1]) (contiguous, balanced)."""
    return [g * nparts // world for g in range(world + 1)]


class DeviceOps:
    """The C-ABI kernels (paper_2404_18497_b200/csrc), one CUDA stream."""

    aux_dtype = torch.int16  # bucket ids travel with the low words

    def __init__(self, config: BuildConfig):
        from .assignment import tabulate

        self.config = config
        self.dev = _native.require_device()
        self.spec = config.resolved_assignment()
        self.table = tabulate(self.spec)
        self.entries = device_table(self.table, self.dev)
        self.B = config.bucket_count
        self.peer: PeerBuffers | None = None  # p2p receive buffers, kept across builds

    def close(self) -> None:
        """Collective: unmap the peers' receive buffers and free our own."""
        if self.peer is not None:
            self.peer.close()
            self.peer = None

    def stage(self, keys) -> DeviceKeys:
        return to_device(keys, self.dev)

    def hash_count(self, dk: DeviceKeys, seed: int, nparts: int) -> torch.Tensor:
        counts = torch.zeros(nparts, dtype=torch.int32, device=self.dev)
        P = _native.ptr
        _native.call("phb_hash_count", None if dk.is_u64 else P(dk.buf),
                     None if dk.is_u64 else P(dk.offsets), P(dk.keys64) if dk.is_u64 else None,
                     dk.n, seed, nparts, P(counts), _native.stream())
        return counts

    def layout(self, counts: torch.Tensor, n: int, nparts: int):
        key_off = torch.empty(nparts + 1, dtype=torch.int64, device=self.dev)
        deltas = torch.empty(nparts + 1, dtype=torch.int64, device=self.dev)
        stats = torch.empty(2, dtype=torch.int64, device=self.dev)
        P = _native.ptr
        _native.call("phb_layout", P(counts), nparts, 0, 0, n, nparts, P(key_off), P(deltas),
                     P(stats), _native.stream())
        return key_off, deltas, stats

    def scatter(self, dk: DeviceKeys, seed: int, nparts: int, key_off: torch.Tensor):
        cursor = torch.zeros(nparts, dtype=torch.int32, device=self.dev)
        lo = torch.empty(dk.n, dtype=torch.int64, device=self.dev)
        aux = torch.empty(dk.n, dtype=torch.int16, device=self.dev)
        P = _native.ptr
        _native.call("phb_scatter", None if dk.is_u64 else P(dk.buf),
                     None if dk.is_u64 else P(dk.offsets), P(dk.keys64) if dk.is_u64 else None,
                     dk.n, seed, nparts, P(self.entries), self.B, P(key_off), P(cursor), P(lo),
                     P(aux), _native.stream())
        return lo, aux

    def regroup(self, lo_recv, aux_recv, C_owned: torch.Tensor, recv_splits):
        """Merge G partition-sorted chunks into one partition-grouped array."""
        G, np_g = C_owned.shape
        n = lo_recv.numel()
        lo = torch.empty(n, dtype=torch.int64, device=self.dev)
        aux = torch.empty(n, dtype=torch.int16, device=self.dev)
        key_off = torch.empty(np_g + 1, dtype=torch.int64, device=self.dev)
        C = C_owned.to(self.dev, torch.int32).contiguous()
        P = _native.ptr
        _native.call("phb_regroup", P(lo_recv), P(aux_recv), P(C), G, np_g, P(lo), P(aux),
                     P(key_off), _native.stream())
        return lo, aux, key_off

    def search(self, lo, aux, key_off, np_g: int, m_max: int):
        B = self.B
        seeds = torch.zeros(B * np_g, dtype=torch.int64, device=self.dev)
        part_trials = torch.empty(np_g, dtype=torch.int64, device=self.dev)
        status = torch.empty(np_g, dtype=torch.uint8, device=self.dev)
        glo = torch.empty(max(lo.numel(), 1), dtype=torch.int64, device=self.dev)
        queue = torch.empty(1, dtype=torch.int32, device=self.dev)
        P = _native.ptr
        cfg = self.config
        _native.call("phb_search", P(lo), P(aux), P(key_off), 0, np_g, 0, B, cfg.seed_cap,
                     cfg.tie_desc, m_max, P(seeds), 1, np_g, None, P(part_trials), P(status),
                     P(glo), P(queue), _native.stream())
        return seeds.view(B, np_g), part_trials, status

    def encode(self, seeds_cm: torch.Tensor, deltas, stats, nparts: int):
        """K5 over the global column-major seed matrix -> (blob, summary)."""
        mono, prefix = self.config.compact_prefix()
        B = self.B
        L = _native.lib()
        P = _native.ptr
        ws = torch.empty(int(L.phb_encode_workspace_bytes(nparts, B, mono)), dtype=torch.uint8,
                         device=self.dev)
        summ = np.zeros(8, np.int64)
        seeds_cm = seeds_cm.contiguous()
        _native.call("phb_encode_plan", P(seeds_cm), nparts, B, mono, prefix, P(deltas), nparts,
                     P(stats), None, None, P(ws), summ.ctypes.data_as(ctypes.c_void_p),
                     _native.stream())
        total = int(summ[0])
        blob = torch.empty((total + 16 + 3) // 4 * 4, dtype=torch.uint8, device=self.dev)
        _native.call("phb_encode_write", P(seeds_cm), nparts, B, mono, prefix, P(deltas),
                     nparts, P(stats), P(ws), P(blob), blob.numel(), _native.stream())
        return blob, summ


    def encode_sharded(self, seeds_own: torch.Tensor, p_lo: int, np_g: int, nparts: int,
                       deltas, stats, group, rank: int, world: int):
        """K5 over the ranks' own seed rows (phb_encode_shard_*): reduce the
        column statistics, plan the global geometry on every rank, write the
        own fields at their global bit addresses, OR the bodies together (a
        uint8 SUM, every bit has exactly one writer)."""
        mono, prefix = self.config.compact_prefix()
        B = self.B
        ncols = 1 if mono else B
        L = _native.lib()
        P = _native.ptr
        st = _native.stream()
        seeds_own = seeds_own.contiguous()
        colstat = torch.empty(ncols * 65, dtype=torch.int64, device=self.dev)
        _native.call("phb_encode_shard_stats", P(seeds_own), np_g, B, mono, P(colstat), st)
        cs = colstat.view(ncols, 65)
        mx = cs[:, 0].contiguous()   # seeds < 2^63: the int64 view orders like u64
        pops = cs[:, 1:].contiguous()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(pops, op=dist.ReduceOp.SUM, group=group)
        cs_g = torch.cat([mx[:, None], pops], 1).contiguous()
        ws = torch.empty(int(L.phb_encode_workspace_bytes(max(np_g, 1), B, mono)),
                         dtype=torch.uint8, device=self.dev)
        totals = torch.empty(ncols, dtype=torch.int64, device=self.dev)
        summ = np.zeros(8, np.int64)
        _native.call("phb_encode_shard_plan", P(seeds_own), np_g, p_lo, nparts, B, mono, prefix,
                     P(stats), P(cs_g), P(ws), P(totals), summ.ctypes.data_as(ctypes.c_void_p), st)
        allt = [torch.empty_like(totals) for _ in range(world)]
        dist.all_gather(allt, totals, group=group)
        base = torch.zeros_like(totals)
        for g in range(rank):
            base += allt[g]
        total = int(summ[0])
        blob = torch.empty((total + 16 + 3) // 4 * 4, dtype=torch.uint8, device=self.dev)
        _native.call("phb_encode_shard_write", P(seeds_own), np_g, p_lo, nparts, B, mono, prefix,
                     P(deltas), P(stats), P(base), int(rank == 0), P(ws), P(blob), blob.numel(),
                     st)
        dist.all_reduce(blob, op=dist.ReduceOp.SUM, group=group)
        return blob, summ


def _as_bytes(t: torch.Tensor) -> torch.Tensor:
    return t.contiguous().view(torch.uint8)


def build_distributed(local_keys, config: BuildConfig | None = None, group=None, ops=None,
                      to_host: bool = True, transport: str = "nccl", encode: str = "sharded"):
    """Collective build: every rank passes its shard; every rank returns the
    same Mphf (global n, identical bytes for any world size). With
    to_host=False the device-resident DeviceBuild is returned instead.

    transport: "nccl" = K3 + all_to_all_single + phb_regroup; "p2p" = the
    fused route, K3 writing every record straight into its owner's buffer
    over CUDA-IPC peer memory (phb_scatter_p2p; one process per GPU on one
    node).

    encode: "sharded" (device ops) = every rank encodes its own seed rows at
    their global bit addresses and the bodies are OR-ed (a uint8 all_reduce
    of ~bits/key * n / 8 bytes); "gather" = all_gather of the seed rows and a
    replicated encode (8 B per partition and bucket moved)."""
    from .mphf import BuildStats, DeviceBuild, DuplicateKeys, Mphf

    config = config or BuildConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ops = ops or DeviceOps(config)
    t0 = time.perf_counter()
    dk = ops.stage(local_keys)
    comm_dev = getattr(ops, "comm_device", None) or (ops.dev if hasattr(ops, "dev") else "cpu")
    n_t = torch.tensor([dk.n], dtype=torch.int64, device=comm_dev)
    dist.all_reduce(n_t, group=group)
    n = int(n_t.item())
    if n < 1:
        raise InvalidConfig("need at least one key")
    nparts = num_partitions_for(n, config.partition_size)
    bounds = owner_bounds(nparts, world)
    p_lo, p_hi = bounds[rank], bounds[rank + 1]
    np_g = p_hi - p_lo
    last = None
    for attempt in range(MAX_ATTEMPTS):
        seed = (config.global_seed + attempt) & 0xFFFFFFFFFFFFFFFF
        # 1-2. local counts, all_gather -> C[s][j]
        counts = ops.hash_count(dk, seed, nparts)
        gathered = [torch.empty_like(counts) for _ in range(world)]
        dist.all_gather(gathered, counts, group=group)
        C = torch.stack(gathered).to(torch.int64)            # [G, nparts]
        total_counts = C.sum(0).to(torch.int32)
        key_off_g, deltas, stats = ops.layout(total_counts.clone(), n, nparts)  # clobbers counts
        C_owned = C[:, p_lo:p_hi]
        # one small host read: every rank's receive count and the owned max size
        bt = torch.tensor(bounds, device=C.device)
        csum = torch.zeros(nparts + 1, dtype=torch.int64, device=C.device)
        torch.cumsum(total_counts.to(torch.int64), 0, out=csum[1:])
        own_max = (total_counts[p_lo:p_hi].max().to(torch.int64).reshape(1) if np_g
                   else torch.zeros(1, dtype=torch.int64, device=C.device))
        small = torch.cat([csum[bt[1:]] - csum[bt[:-1]], own_max]).cpu().tolist()
        recv_all, m_max = small[:world], int(small[world])
        routed = None
        if transport == "p2p":
            # 3-5 fused: records land partition-grouped in the owner's buffer
            routed = _route_p2p(ops, dk, seed, nparts, C, bounds, rank, world, group, recv_all)
            if routed is None:  # peer mapping unavailable on some rank: collective fallback
                transport = "nccl"
        if routed is not None:
            lo_g, aux_g, key_off_own, route = routed
        else:
            # 3. group own keys by partition (hence by destination rank)
            key_off_l = torch.zeros(nparts + 1, dtype=torch.int64, device=C.device)
            torch.cumsum(C[rank], 0, out=key_off_l[1:])
            lo, aux = ops.scatter(dk, seed, nparts, key_off_l)
            kb = key_off_l[torch.tensor(bounds, device=C.device)].cpu().tolist()
            send = [kb[g + 1] - kb[g] for g in range(world)]
            recv = C_owned.sum(1).cpu().tolist()
            # 4. all-to-all of the records (byte views: gloo/NCCL-safe dtypes)
            esz = aux.element_size()
            lo_r = torch.empty(sum(recv), dtype=lo.dtype, device=lo.device)
            aux_r = torch.empty(sum(recv) * esz, dtype=torch.uint8, device=lo.device)
            dist.all_to_all_single(lo_r, lo, recv, send, group=group)
            dist.all_to_all_single(aux_r, _as_bytes(aux), [r * esz for r in recv],
                                   [s * esz for s in send], group=group)
            aux_r = aux_r.view(aux.dtype)
            # 5. merge the G partition-sorted chunks
            lo_g, aux_g, key_off_own = ops.regroup(lo_r, aux_r, C_owned, recv)
            route = None
        # 6. search + collective failure / trials
        if np_g:
            seeds_own, part_trials, status = ops.search(lo_g, aux_g, key_off_own, np_g, m_max)
            st = status.to(torch.int64)
            bad_local = (torch.nonzero(st).flatten()[:1] + p_lo)
            bad = int(bad_local.item()) if bad_local.numel() else nparts
            code = int(st[bad - p_lo].item()) if bad < nparts else 0
            trials = int(part_trials.sum().item())
        else:
            seeds_own = torch.zeros((config.bucket_count, 0), dtype=torch.int64, device=C.device)
            bad, code, trials = nparts, 0, 0
        flag = torch.tensor([bad, trials], dtype=torch.int64, device=C.device)
        red = flag.clone()
        dist.all_reduce(red[0:1], op=dist.ReduceOp.MIN, group=group)
        dist.all_reduce(red[1:2], op=dist.ReduceOp.SUM, group=group)
        gbad = int(red[0].item())
        if gbad < nparts:
            code_t = torch.tensor([code if bad == gbad else 0], dtype=torch.int64, device=C.device)
            dist.all_reduce(code_t, op=dist.ReduceOp.MAX, group=group)
            reason = "unseparable duplicate hashes" if int(code_t.item()) == 1 else "seed cap hit"
            last = f"partition {gbad}: {reason}"
            continue
        trials_total = int(red[1].item())
        B = config.bucket_count
        if isinstance(ops, DeviceOps) and encode == "sharded":
            # 7. sharded encode: no rank assembles the seed matrix
            blob, summ = ops.encode_sharded(seeds_own, p_lo, np_g, nparts, deltas, stats, group,
                                            rank, world)
            stats_obj = BuildStats(attempt + 1, trials_total, trials_total / n,
                                   time.perf_counter() - t0)
            db = DeviceBuild(n, nparts, B, seed, key_off_g, deltas, None, blob, int(summ[0]),
                             int(summ[1]), trials_total)
            if not to_host:
                return db
            return Mphf._from_device(db, config, _EngineView(ops), stats_obj)
        # 7. all_gather the owned seed columns (padded to the widest range)
        width = max(bounds[g + 1] - bounds[g] for g in range(world))
        pad = torch.zeros((B, width), dtype=torch.int64, device=seeds_own.device)
        pad[:, :np_g] = seeds_own
        blocks = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(blocks, pad, group=group)
        seeds_cm = torch.cat([blocks[g][:, : bounds[g + 1] - bounds[g]] for g in range(world)], 1)
        blob, summ = ops.encode(seeds_cm, deltas, stats, nparts)
        stats_obj = BuildStats(attempt + 1, trials_total, trials_total / n,
                               time.perf_counter() - t0)
        if not isinstance(ops, DeviceOps):
            return ops.finish(blob, summ, seed, n, nparts, deltas, seeds_cm, stats_obj)
        db = DeviceBuild(n, nparts, B, seed, key_off_g, deltas, seeds_cm.reshape(-1), blob,
                         int(summ[0]), int(summ[1]), trials_total)
        if not to_host:
            return db
        eng = _EngineView(ops)
        return Mphf._from_device(db, config, eng, stats_obj)
    raise DuplicateKeys(
        f"construction failed after {MAX_ATTEMPTS} seeds ({SeedExhausted(last)}); "
        "input most likely contains duplicate keys")


class PeerBuffers:
    """CUDA-IPC receive buffers of the fused p2p route: one buffer of 16-byte
    {lo, bucket id} records per rank (one peer store per key), allocated
    once per DeviceOps and kept mapped in every peer across builds; they
    grow (collectively) only when some rank must receive more records than
    its buffer holds. Every rank derives every rank's receive count from the
    all-gathered per-partition counts, so the grow decision needs no extra
    collective."""

    REC = 16  # bytes per record

    def __init__(self, group, rank: int, world: int):
        self.group, self.rank, self.world = group, rank, world
        self.caps = [0] * world          # records per rank (identical on every rank)
        self.rec_p = ctypes.c_void_p()   # own receive buffer
        self.rec_ptrs = (ctypes.c_void_p * world)()
        self.opened: list[int] = []      # mapped peer buffers (not ours)
        self.maps = 0                    # how many times the buffers were (re)mapped

    def _unmap(self) -> None:
        L = _native.lib()
        _native.check(L.phb_sync(_native.stream()), "phb_sync")
        for ptr in self.opened:
            L.phb_ipc_close(ptr)
        self.opened = []
        dist.barrier(group=self.group)  # every peer unmapped our buffer
        if self.rec_p.value:
            L.phb_ipc_free(self.rec_p)
        self.rec_p = ctypes.c_void_p()

    def close(self) -> None:
        self._unmap()
        self.caps = [0] * self.world

    def ensure(self, recv: list[int], comm_dev) -> bool:
        """Make every rank's buffer hold recv[g] records (collective when
        any rank grows). False if some rank cannot map a peer buffer."""
        if all(r <= c for r, c in zip(recv, self.caps)) and self.rec_p.value:
            return True
        L = _native.lib()
        self._unmap()
        # 2% headroom so that the next builds (retries, other seeds) fit
        self.caps = [max(c, int(r * 1.02) + 4096) for r, c in zip(recv, self.caps)]
        _native.check(L.phb_ipc_alloc(self.caps[self.rank] * self.REC, ctypes.byref(self.rec_p)),
                      "phb_ipc_alloc")
        hbuf = np.zeros(64, np.uint8)
        _native.check(L.phb_ipc_handle(self.rec_p, hbuf.ctypes.data_as(ctypes.c_void_p)),
                      "phb_ipc_handle")
        mine = torch.from_numpy(hbuf).to(comm_dev)
        allh = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allh, mine, group=self.group)
        ok = True
        for g in range(self.world):
            if g == self.rank:
                self.rec_ptrs[g] = self.rec_p.value
                continue
            h = np.ascontiguousarray(allh[g].cpu().numpy())
            a = ctypes.c_void_p()
            if L.phb_ipc_open(h.ctypes.data_as(ctypes.c_void_p), ctypes.byref(a)) != 0:
                ok = False
                break
            self.opened.append(a.value)
            self.rec_ptrs[g] = a.value
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64, device=comm_dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
        self.maps += 1
        if int(flag.item()) == 0:
            self.close()
            return False
        return True


def _fence(group, dev) -> None:
    """Order every rank's peer stores before the owners' reads. NCCL: a
    1-element all_reduce enqueued on the stream (device-side ordering, no
    host sync); other backends: stream sync + barrier."""
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(torch.zeros(1, dtype=torch.int32, device=dev), group=group)
    else:
        _native.check(_native.lib().phb_sync(_native.stream()), "phb_sync")
        dist.barrier(group=group)


class _PtrTensor:
    """Minimal tensor-like view of a raw device pointer for _native.ptr()."""

    def __init__(self, ptr: int, n: int):
        self._p, self._n = ptr, n

    def data_ptr(self) -> int:
        return self._p

    def numel(self) -> int:
        return self._n


def _route_p2p(ops: DeviceOps, dk: DeviceKeys, seed: int, nparts: int, C: torch.Tensor,
               bounds: list[int], rank: int, world: int, group, recv_all: list[int]):
    """Fused K3 + all-to-all over peer memory (phb_scatter_p2p) into the
    persistent receive buffers. The next build's first collective (the
    count all_gather, stream-ordered after this rank's search) orders the
    owners' reads before the sources' next stores."""
    L = _native.lib()
    dev = ops.dev
    if ops.peer is None:
        ops.peer = PeerBuffers(group, rank, world)
    if not ops.peer.ensure(recv_all, C.device):
        ops.peer = None
        return None
    pb = ops.peer
    total = C.sum(0)                                       # [nparts] global counts
    ex = torch.zeros(nparts + 1, dtype=torch.int64, device=dev)
    torch.cumsum(total.to(dev), 0, out=ex[1:])
    owner = torch.empty(nparts, dtype=torch.uint8, device=dev)
    start = torch.empty(nparts, dtype=torch.int64, device=dev)
    for g in range(world):
        owner[bounds[g]:bounds[g + 1]] = g
        start[bounds[g]:bounds[g + 1]] = ex[bounds[g]]
    before = (C[:rank].sum(0) if rank else torch.zeros_like(total)).to(dev)
    part_base = (ex[:-1] - start + before).contiguous()   # my first slot per partition
    p_lo, p_hi = bounds[rank], bounds[rank + 1]
    recv_n = recv_all[rank]
    cursor = torch.empty(nparts, dtype=torch.int32, device=dev)
    P = _native.ptr
    _native.check(L.phb_scatter_p2p(
        None if dk.is_u64 else P(dk.buf), None if dk.is_u64 else P(dk.offsets),
        P(dk.keys64) if dk.is_u64 else None, dk.n, seed, nparts, P(ops.entries), ops.B,
        P(part_base), P(owner), pb.rec_ptrs, None, world, P(cursor), _native.stream()),
        "phb_scatter_p2p")
    _fence(group, dev)  # every source finished writing into every owner
    key_off_own = (ex[p_lo:p_hi + 1] - ex[p_lo]).contiguous()
    # 16-byte records: the search reads them with bid = NULL
    return (_PtrTensor(pb.rec_p.value, 2 * recv_n), None, key_off_own, None)


class _EngineView:
    """The attributes of BuildEngine that Mphf._from_device reads."""

    def __init__(self, ops: DeviceOps):
        self.spec = ops.spec
        self.table = ops.table
        self.entries = ops.entries
