"""Full-size parity in the driver-run GPU suite.

* C2 — the bench workload itself: 100M keys mix64(i), lambda = 9, P = 2500,
  IC-C. Built on the device exactly as bench.py times it (BuildEngine.run on
  resident keys) and through the public API; serialized bytes, the trial
  total and a 2M-key query sample equal the oracle's (all host cores), and
  the structure is a bijection (pilothash mphf.py:236-290, builder.py:224-277).
* C5 — 100M random strings of 10-100 B, lambda = 8, IC-R: bytes, trials and
  a query sample equal the oracle's.
* C3 — 1B keys on one GPU: bijection of every key, plus ~2,000 randomly
  chosen partitions rebuilt by the oracle from keys the oracle hashed and
  partitioned itself: per-bucket seeds and trials equal, row by row.

Each test is `slow` (the oracle needs 1-2 minutes per case on the host).
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def phb():
    import paper_2404_18497_b200 as m

    torch.cuda.set_device(0)
    return m


def _query_sample_equal(f, ref, orc, keys, idx, corpus=None):
    if corpus is None:
        sample = keys[idx]
        hi, lo = orc.murmur3_u64(sample, f.global_seed)
        got = f.query_many(sample)
    else:
        buf, off = corpus
        lens = off[idx + 1] - off[idx]
        soff = np.zeros(len(idx) + 1, np.int64)
        np.cumsum(lens, out=soff[1:])
        sbuf = np.concatenate([buf[off[i]:off[i + 1]] for i in idx])
        hi, lo = orc.murmur3_many(sbuf, soff, f.global_seed)
        import paper_2404_18497_b200 as m

        got = f.query_many(m.KeyCorpus(sbuf, soff))
    return np.array_equal(got, ref.query_hashes(hi, lo))


def test_c2_bench_workload_full_size_vs_oracle(phb, orc):
    from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64, synth_u64_device
    from paper_2404_18497_b200.mphf import HEADER_FIXED, BuildEngine

    n = 100_000_000
    cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
    # the timed path of bench.py: device-resident keys, BuildEngine.run
    dkeys = synth_u64_device(n, 0)
    db = BuildEngine(cfg).run(DeviceKeys(n, keys64=dkeys), 0)
    dev_body = db.blob[HEADER_FIXED:db.total_bytes].cpu().numpy()
    dev_trials = db.trials_total
    del db, dkeys
    torch.cuda.empty_cache()
    keys = synth_u64(n, 0)
    f = phb.build(keys, cfg)  # public API, host keys (the e2e path)
    ref = orc.build(keys, lambda_=9.0, P=2500.0, encoder="ic-c", threads=THREADS)
    blob, rblob = f.serialize(), ref.serialize()
    assert len(blob) == len(rblob) and blob == rblob
    assert np.array_equal(np.frombuffer(rblob, np.uint8)[HEADER_FIXED:len(rblob) - 8], dev_body)
    assert f.stats.trials_total == int(ref.trials.sum()) == dev_trials
    idx = np.random.default_rng(2).choice(n, 2_000_000, replace=False)
    assert _query_sample_equal(f, ref, orc, keys, idx)
    assert f.is_bijection_on(keys)


def test_c5_strings_full_size_vs_oracle(phb, orc):
    n = 100_000_000
    rng = np.random.default_rng(5)
    lens = rng.integers(10, 101, size=n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    del lens
    buf = rng.integers(33, 127, size=int(off[-1]), dtype=np.uint8)
    cfg = phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r")
    corpus = phb.KeyCorpus(buf, off)
    f = phb.build(corpus, cfg)
    ref = orc.build((buf, off), lambda_=8.0, P=2500.0, encoder="ic-r", threads=THREADS)
    assert f.serialize() == ref.serialize()
    assert f.stats.trials_total == int(ref.trials.sum())
    idx = np.random.default_rng(3).choice(n, 200_000, replace=False)
    assert _query_sample_equal(f, ref, orc, None, idx, corpus=(buf, off))
    assert f.is_bijection_on(corpus)
    # the batched device query of all 100M keys (hash pass + shared-table
    # query, in 32M-key chunks) agrees with the oracle on the sample
    full = f.query_many(corpus)
    lens = off[idx + 1] - off[idx]
    soff = np.zeros(len(idx) + 1, np.int64)
    np.cumsum(lens, out=soff[1:])
    sbuf = np.concatenate([buf[off[i]:off[i + 1]] for i in idx])
    hi, lo = orc.murmur3_many(sbuf, soff, f.global_seed)
    assert np.array_equal(full[idx], ref.query_hashes(hi, lo))


def test_c3_billion_keys_sampled_partitions_vs_oracle(phb, orc):
    from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64, synth_u64_device
    from paper_2404_18497_b200.mphf import BuildEngine

    n = 1_000_000_000
    lam, P = 9.0, 2500.0
    cfg = phb.BuildConfig(lambda_=lam, partition_size=P, encoder="ic-c")
    keys = synth_u64_device(n, 0)
    dk = DeviceKeys(n, keys64=keys)
    eng = BuildEngine(cfg)
    db = eng.run(dk, 0, instrument=True)
    assert not isinstance(db, tuple)
    nparts, B = db.nparts, db.bcount
    f = phb.Mphf._from_device(db, cfg, eng, None)
    assert f.verify_device(f.query_device(dk)), "1B keys: not a bijection"
    # the encoded-section query at n >= 2^29 (16-byte column descriptors) equals the matrix query
    sub = DeviceKeys(16_000_000, keys64=keys[:16_000_000])
    assert torch.equal(f.query_encoded_device(sub), f.query_device(sub))
    del sub
    key_off = db.key_off.cpu().numpy()
    rng = np.random.default_rng(33)
    sel = np.sort(rng.choice(nparts, 2000, replace=False))
    seeds_dev = db.seeds.view(B, nparts)[:, torch.from_numpy(sel).cuda()].t().cpu().numpy()
    trials_dev = db.trials.view(B, nparts)[:, torch.from_numpy(sel).cuda()].t().cpu().numpy()
    del f, db, keys, dk
    torch.cuda.empty_cache()

    # the oracle hashes and partitions the same 1B keys itself (chunked, all cores)
    want = np.zeros(nparts, bool)
    want[sel] = True
    chunk = 25_000_000

    def part(c):
        k = synth_u64(min(chunk, n - c), c)
        hi, lo = orc.murmur3_u64(k, 0)
        # mulhi(hi, nparts) (partitioning.py) without 128-bit numpy: split hi
        h1, h0 = hi >> np.uint64(32), hi & np.uint64(0xFFFFFFFF)
        npv = np.uint64(nparts)
        j = (h1 * npv + ((h0 * npv) >> np.uint64(32))) >> np.uint64(32)
        m = want[j.astype(np.int64)]
        return j[m].astype(np.int64), hi[m], lo[m]

    with ThreadPoolExecutor(max_workers=THREADS) as pool:
        got = list(pool.map(part, range(0, n, chunk)))
    js = np.concatenate([g[0] for g in got])
    his = np.concatenate([g[1] for g in got])
    los = np.concatenate([g[2] for g in got])
    order = np.lexsort((los, his, js))
    js, his, los = js[order], his[order], los[order]
    # partition sizes the oracle found equal the device layout
    cnt = np.bincount(js, minlength=nparts)[sel]
    assert np.array_equal(cnt, (key_off[sel + 1] - key_off[sel]))
    off = np.zeros(len(sel) + 1, np.int64)
    np.cumsum(cnt, out=off[1:])
    table = orc.tabulate("beta_eps", orc.default_epsilon(lam, P))
    assert B == orc.bucket_count(P, lam)
    seeds, trials, status = orc.build_partition_range(his, los, off, 0, len(sel), table, B,
                                                      cfg.seed_cap, cfg.tie_desc, THREADS)
    assert not status.any()
    assert np.array_equal(seeds, seeds_dev.view(np.uint64))
    assert np.array_equal(trials, trials_dev)


@pytest.mark.parametrize("lam", [4.0, 5.0])
def test_c4_low_lambda_full_size_vs_oracle(phb, orc, lam):
    """C4's low-lambda end at full size (100M u64 keys, IC-R): the low-lambda
    search kernel (speculative seed-0 steps over four buckets, batched
    singletons) gives the oracle's bytes and trial total."""
    from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64, synth_u64_device
    from paper_2404_18497_b200.mphf import HEADER_FIXED, BuildEngine

    n = 100_000_000
    cfg = phb.BuildConfig(lambda_=lam, partition_size=2500.0, encoder="ic-r")
    dkeys = synth_u64_device(n, 7)
    db = BuildEngine(cfg).run(DeviceKeys(n, keys64=dkeys), 0)
    body = db.blob[HEADER_FIXED:db.total_bytes].cpu().numpy()
    trials = db.trials_total
    del db, dkeys
    torch.cuda.empty_cache()
    ref = orc.build(synth_u64(n, 7), lambda_=lam, P=2500.0, encoder="ic-r", threads=THREADS)
    rblob = np.frombuffer(ref.serialize(), np.uint8)
    assert np.array_equal(rblob[HEADER_FIXED:len(rblob) - 8], body)
    assert trials == int(ref.trials.sum())
