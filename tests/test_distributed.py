"""Multi-process (gloo, CPU) tests of the sharded build's orchestration
(paper_2404_18497_b200/distributed.py): ownership ranges, the counts
all_gather, the record all-to-all, the regroup, the collective retry and
the seed gather. The per-rank kernels are replaced by the oracle (test
infrastructure) so the logic runs without a GPU; the serialized bytes must
equal the single-process oracle build for every world size."""

import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class OracleOps:
    """CPU stand-in for DeviceOps built from the oracle (tests only).
    aux carries the high word (the oracle derives bucket ids from it)."""

    comm_device = "cpu"

    def __init__(self, config):
        from oracle import oracle

        self.o = oracle
        self.config = config
        self.kind = "beta_eps"
        self.eps = oracle.default_epsilon(config.lambda_, config.partition_size)
        self.table = oracle.tabulate(self.kind, self.eps)
        self.B = config.bucket_count

    class Keys:
        def __init__(self, keys):
            self.keys = np.ascontiguousarray(keys, np.uint64)
            self.n = len(self.keys)

    def stage(self, keys):
        return self.Keys(keys)

    def _hash(self, dk, seed):
        return self.o.murmur3_u64(dk.keys, seed)

    def hash_count(self, dk, seed, nparts):
        hi, _ = self._hash(dk, seed)
        j = ((hi.astype(object) * nparts) >> 64).astype(np.int64)
        return torch.from_numpy(np.bincount(j, minlength=nparts).astype(np.int32))

    def layout(self, counts, n, nparts):
        c = counts.numpy().astype(np.int64)
        key_off = np.zeros(nparts + 1, np.int64)
        np.cumsum(c, out=key_off[1:])
        exp = np.array([(2 * j * n + nparts) // (2 * nparts) for j in range(nparts + 1)], np.int64)
        deltas = key_off - exp
        return torch.from_numpy(key_off), torch.from_numpy(deltas), None

    def scatter(self, dk, seed, nparts, key_off):
        hi, lo = self._hash(dk, seed)
        j = ((hi.astype(object) * nparts) >> 64).astype(np.int64)
        order = np.argsort(j, kind="stable")
        return (torch.from_numpy(lo[order].view(np.int64)),
                torch.from_numpy(hi[order].view(np.int64)))

    def regroup(self, lo_r, aux_r, C_owned, recv):
        C = C_owned.numpy()
        G, np_g = C.shape
        lo, aux = lo_r.numpy(), aux_r.numpy()
        starts = np.concatenate([[0], np.cumsum(recv)])
        lo_out, aux_out = [], []
        for j in range(np_g):
            for s in range(G):
                a = starts[s] + C[s, :j].sum()
                lo_out.append(lo[a:a + C[s, j]])
                aux_out.append(aux[a:a + C[s, j]])
        key_off = np.zeros(np_g + 1, np.int64)
        np.cumsum(C.sum(0), out=key_off[1:])
        cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)
        return torch.from_numpy(cat(lo_out)), torch.from_numpy(cat(aux_out)), key_off

    def search(self, lo, aux, key_off, np_g, m_max):
        cfg = self.config
        seeds, trials, status = self.o.build_partition_range(
            aux.numpy().view(np.uint64), lo.numpy().view(np.uint64), key_off, 0, np_g,
            self.table, self.B, cfg.seed_cap, cfg.tie_desc)
        return (torch.from_numpy(seeds.T.copy().view(np.int64)),
                torch.from_numpy(trials.sum(1)), torch.from_numpy(status))

    def encode(self, seeds_cm, deltas, stats, nparts):
        mat = seeds_cm.numpy().view(np.uint64).T.copy()
        return self.o.encode_body(mat, deltas.numpy(), self.config.encoder), None

    def finish(self, body, summ, seed, n, nparts, deltas, seeds_cm, stats):
        from oracle.oracle import OracleMphf

        f = OracleMphf(n, nparts, self.B, self.config.lambda_, self.config.partition_size,
                       self.kind, self.eps, seed, stats.attempts, deltas.numpy(),
                       seeds_cm.numpy().view(np.uint64).T.copy(), None, self.table,
                       self.config.encoder)
        return f, stats


def _worker(rank, world, path, keys, cfg_kw, out_path):
    from paper_2404_18497_b200 import BuildConfig
    from paper_2404_18497_b200.distributed import build_distributed

    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    try:
        shards = np.array_split(keys, world)
        cfg = BuildConfig(**cfg_kw)
        f, stats = build_distributed(shards[rank], cfg, ops=OracleOps(cfg))
        if rank == 0:
            np.save(out_path, np.frombuffer(f.serialize(), np.uint8))
            np.save(out_path + ".stats.npy", np.array([stats.attempts, stats.trials_total]))
    finally:
        dist.destroy_process_group()


def _run(world, keys, cfg_kw):
    d = tempfile.mkdtemp()
    out = os.path.join(d, "blob.npy")
    mp.spawn(_worker, args=(world, os.path.join(d, "rdv"), keys, cfg_kw, out), nprocs=world)
    return np.load(out).tobytes(), np.load(out + ".stats.npy")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg_kw", [dict(lambda_=5.0, partition_size=500.0, encoder="ic-c"),
                                    dict(lambda_=7.0, partition_size=300.0, encoder="ic-r",
                                         tie_break="desc-expected", global_seed=9)])
def test_sharded_build_bytes_equal_single_process(world, cfg_kw):
    from oracle import oracle

    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(6000, 77)
    blob, stats = _run(world, keys, cfg_kw)
    ref = oracle.build(keys, lambda_=cfg_kw["lambda_"], P=cfg_kw["partition_size"],
                       encoder=cfg_kw["encoder"], tie_break=cfg_kw.get("tie_break", "asc-expected"),
                       global_seed=cfg_kw.get("global_seed", 0), threads=2)
    assert blob == ref.serialize()
    assert stats[1] == int(ref.trials.sum())


def test_sharded_build_collective_retry_on_duplicates():
    """A duplicate key on one rank fails that rank's partition; every rank
    must retry with seed + 1 together and finally raise DuplicateKeys."""
    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(3000, 5)
    keys = np.concatenate([keys, keys[:1]])  # the duplicate lands on the last shard
    d = tempfile.mkdtemp()
    with pytest.raises(Exception, match="DuplicateKeys|duplicate"):
        mp.spawn(_worker, args=(2, os.path.join(d, "rdv"), keys,
                                dict(lambda_=4.0, partition_size=250.0), os.path.join(d, "b.npy")),
                 nprocs=2)


def test_owner_bounds_cover_all_partitions():
    from paper_2404_18497_b200.distributed import owner_bounds

    for nparts in (1, 7, 400, 40_000):
        for world in (1, 2, 3, 8):
            b = owner_bounds(nparts, world)
            assert b[0] == 0 and b[-1] == nparts and all(x <= y for x, y in zip(b, b[1:]))
            assert max(y - x for x, y in zip(b, b[1:])) - min(y - x for x, y in zip(b, b[1:])) <= 1
