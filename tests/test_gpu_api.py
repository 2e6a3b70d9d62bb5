"""API-level parity of the drop-in (build / query / serialize) against the
reference's own bytes and queries, plus the reference's API tests
(pkg/tests/test_mphf.py) restated against this package."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def phb():
    import paper_2404_18497_b200 as m
    from paper_2404_18497_b200 import _native

    _native.require_device()
    return m


def _e2e_cases(meta):
    return [(k[4:], enc) for k, v in meta.items() if k.startswith("e2e_") for enc in v["bytes"]]


def test_golden_bytes_every_preset(golden, meta, phb):
    from paper_2404_18497_b200 import KeyCorpus

    for name, enc in _e2e_cases(meta):
        m = meta[f"e2e_{name}"]
        corpus = KeyCorpus(golden[f"e2e_{name}_buf"], golden[f"e2e_{name}_off"])
        cfg = phb.BuildConfig(lambda_=m["lambda"], partition_size=m["P"], global_seed=m["gseed"],
                              encoder=enc, tie_break=m["tie"])
        f = phb.build(corpus, cfg)
        blob = f.serialize()
        want = golden[f"e2e_{name}_{enc}"].tobytes()
        assert blob == want, (name, enc, len(blob), len(want))
        assert f.stats.trials_total == m["bytes"][enc]["trials_total"], (name, enc)
        assert f.stats.attempts == m["bytes"][enc]["attempts"]
        assert f.bits_per_key() == m["bytes"][enc]["bits_per_key"]
        if f"e2e_{name}_query" in golden.files and enc == list(m["bytes"])[0]:
            assert np.array_equal(f.query_many(corpus), golden[f"e2e_{name}_query"])


def test_u64_keys_equal_byte_corpus(phb):
    """The u64 fast path == the reference's 8-byte-LE KeyCorpus path."""
    from paper_2404_18497_b200 import KeyCorpus

    rng = np.random.default_rng(5)
    keys = np.unique(rng.integers(0, 2**64, size=30_000, dtype=np.uint64))
    cfg = phb.BuildConfig(lambda_=6.0, partition_size=1000.0, encoder="ic-r")
    a = phb.build(keys, cfg).serialize()
    b = phb.build(KeyCorpus.from_u64(keys), cfg).serialize()
    c = phb.build(torch.from_numpy(keys.view(np.int64)).cuda(), cfg).serialize()
    assert a == b == c


def test_deserialize_roundtrip_every_preset(golden, meta, phb):
    from paper_2404_18497_b200 import KeyCorpus, Mphf

    m = meta["e2e_small"]
    corpus = KeyCorpus(golden["e2e_small_buf"], golden["e2e_small_off"])
    want_q = golden["e2e_small_query"]
    mats = []
    for enc in m["bytes"]:
        data = golden[f"e2e_small_{enc}"].tobytes()
        g = Mphf.deserialize(data)
        assert g.serialize() == data
        assert g.encoder_name == enc
        q = g.query_many(corpus)
        assert np.array_equal(q, want_q)  # same seeds -> same outputs for every preset
        mats.append(g.seeds.decode_matrix())
    for x in mats[1:]:
        assert np.array_equal(x, mats[0])


def test_scalar_accessors_match_decode(golden, phb):
    from paper_2404_18497_b200 import Mphf

    for enc in ("ic-r", "mono-r", "ic-c"):
        g = Mphf.deserialize(golden[f"e2e_small_{enc}"].tobytes())
        mat = g.seeds.decode_matrix()
        rng = np.random.default_rng(0)
        for _ in range(200):
            j = int(rng.integers(0, mat.shape[0]))
            i = int(rng.integers(1, mat.shape[1] + 1))
            assert g.seeds.seed_at(j, i) == mat[j, i - 1]


# ---- the reference's API tests (pkg/tests/test_mphf.py), restated ----

SMALL = dict(lambda_=4.0, partition_size=500.0, global_seed=3)


@pytest.fixture(scope="module")
def corpus_small(phb):
    return phb.gen_keys(20_000, 1)


def test_single_key(phb):
    f = phb.build([b"only"], phb.BuildConfig())
    assert f.n == 1 and f.query(b"only") == 0


def test_bijection_various_sizes(phb):
    for n in (1, 2, 17, 1000):
        corpus = phb.gen_keys(n, n)
        f = phb.build(corpus, phb.BuildConfig(lambda_=4.0, partition_size=250.0))
        assert np.array_equal(np.sort(f.query_many(corpus)), np.arange(n)), n
        assert f.is_bijection_on(corpus)


def test_query_nonmember_in_range(phb, corpus_small):
    f = phb.build(corpus_small, phb.BuildConfig(**SMALL))
    for s in (b"not-in-corpus", b"", b"x" * 500):
        assert 0 <= f.query(s) < f.n


def test_input_order_does_not_change_bytes(phb, corpus_small):
    keys = list(corpus_small)
    rev = phb.KeyCorpus.from_keys(keys[::-1])
    cfg = phb.BuildConfig(**SMALL)
    assert phb.build(corpus_small, cfg).serialize() == phb.build(rev, cfg).serialize()


def test_truncation_and_corruption_rejected(phb, corpus_small):
    data = phb.build(corpus_small, phb.BuildConfig(**SMALL)).serialize()
    for cut in (0, 3, 15, 16, 40, len(data) // 2, len(data) - 1):
        with pytest.raises(phb.FormatError):
            phb.Mphf.deserialize(data[:cut])
    for at in (0, 5, 20, len(data) // 2, len(data) - 3):
        bad = bytearray(data)
        bad[at] ^= 0x40
        with pytest.raises(phb.FormatError):
            phb.Mphf.deserialize(bytes(bad))


def test_save_load(tmp_path, phb, corpus_small):
    f = phb.build(corpus_small, phb.BuildConfig(**SMALL))
    path = tmp_path / "f.phob"
    f.save(path)
    g = phb.Mphf.load(path)
    assert np.array_equal(g.query_many(corpus_small), f.query_many(corpus_small))


def test_duplicate_keys_detected(phb):
    keys = [b"k%d" % i for i in range(500)] + [b"k7"]
    with pytest.raises(phb.DuplicateKeys):
        phb.build(keys, phb.BuildConfig(lambda_=4.0, partition_size=250.0))


def test_invalid_configs(phb):
    with pytest.raises(phb.InvalidConfig):
        phb.build([b"a"], phb.BuildConfig(lambda_=-1.0))
    with pytest.raises(phb.InvalidConfig):
        phb.build([], phb.BuildConfig())


def test_str_keys_accepted(phb):
    f = phb.build(["alpha", "beta", "gamma"], phb.BuildConfig(lambda_=2.0, partition_size=3.0))
    assert sorted(f.query(k.encode()) for k in ("alpha", "beta", "gamma")) == [0, 1, 2]


@pytest.mark.parametrize("lam,enc", [(5.0, "ic-c"), (9.0, "ic-c"), (8.0, "ic-r"),
                                     (6.0, "mono-r"), (4.0, "mixed:40")])
def test_million_u64_vs_oracle(phb, orc, lam, enc):
    rng = np.random.default_rng(int(lam * 10))
    keys = np.unique(rng.integers(0, 2**64, size=1_000_000, dtype=np.uint64))
    keys = keys[rng.permutation(len(keys))]
    cfg = phb.BuildConfig(lambda_=lam, partition_size=2500.0, encoder=enc)
    f = phb.build(keys, cfg)
    ref = orc.build(keys, lambda_=lam, P=2500.0, encoder=enc)
    assert f.serialize() == ref.serialize()
    assert f.stats.trials_total == int(ref.trials.sum())
    hi, lo = orc.murmur3_u64(keys[:100_000], f.global_seed)
    assert np.array_equal(f.query_many(keys[:100_000]), ref.query_hashes(hi, lo))
    assert f.is_bijection_on(keys)


def test_strings_vs_oracle(phb, orc):
    rng = np.random.default_rng(9)
    n = 300_000
    lens = rng.integers(10, 101, size=n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    buf = rng.integers(33, 127, size=int(off[-1]), dtype=np.uint8)
    corpus = phb.KeyCorpus(buf, off)
    f = phb.build(corpus, phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r"))
    ref = orc.build((buf, off), lambda_=8.0, P=2500.0, encoder="ic-r")
    assert f.serialize() == ref.serialize()
    assert f.is_bijection_on(corpus)


@pytest.mark.parametrize("lam,P,n,enc", [
    (10.0, 6000.0, 60_000, "ic-r"),    # m ~ 6000 > 3072: generic search path, multi-pass windows
    (11.0, 12000.0, 48_000, "ic-c"),   # very large partitions, buckets > 256 keys
    (1.0, 300.0, 60_000, "mono-c"),    # B = P: many empty / singleton buckets
    (3.0, 40.0, 50_000, "mixed:3"),    # tiny partitions
])
def test_unusual_configs_vs_oracle(phb, orc, lam, P, n, enc):
    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(n, int(lam * 1000 + P))
    cfg = phb.BuildConfig(lambda_=lam, partition_size=P, encoder=enc)
    f = phb.build(keys, cfg)
    ref = orc.build(keys, lambda_=lam, P=P, encoder=enc)
    assert f.serialize() == ref.serialize()
    assert f.stats.trials_total == int(ref.trials.sum())
    assert f.is_bijection_on(keys)


def test_strings_million_vs_oracle(phb, orc):
    rng = np.random.default_rng(12)
    n = 1_000_000
    lens = rng.integers(10, 101, size=n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    buf = rng.integers(33, 127, size=int(off[-1]), dtype=np.uint8)
    corpus = phb.KeyCorpus(buf, off)
    for enc in ("ic-r", "mono-r"):
        f = phb.build(corpus, phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder=enc))
        ref = orc.build((buf, off), lambda_=8.0, P=2500.0, encoder=enc)
        assert f.serialize() == ref.serialize()
    q = f.query_many(corpus)
    hi, lo = orc.murmur3_many(buf, off, f.global_seed)
    assert np.array_equal(q, ref.query_hashes(hi, lo))


@pytest.mark.slow
def test_hundred_million_properties(phb):
    """Full C2 size: bijection, determinism and input-order independence."""
    from paper_2404_18497_b200.keygen import synth_u64_device

    n = 100_000_000
    keys = synth_u64_device(n, 0)
    cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
    f = phb.build(keys, cfg)
    assert f.is_bijection_on(keys)
    assert 2.10 < f.bits_per_key() < 2.20
    perm = torch.randperm(n, device=keys.device)
    g = phb.build(keys[perm], cfg)
    assert f._body.tobytes() == g._body.tobytes()
    h = phb.Mphf.deserialize(f.serialize())
    sample = keys[:5_000_000]
    assert torch.equal(h.query_device(sample), f.query_device(sample))


def test_staged_ingestion_equals_device_keys(phb):
    """Pageable host keys (numpy, strided numpy, CPU tensor; 80 MB = two
    staging chunks) reach the device byte-identical to CUDA-resident keys."""
    from paper_2404_18497_b200.keygen import staged_h2d, synth_u64_device

    n = 10_000_001  # odd, > one 64 MB staging chunk
    dev_keys = synth_u64_device(n, 77)
    host = dev_keys.cpu().numpy()
    for src in (host, host.view(np.uint64), np.repeat(host, 2)[::2], torch.from_numpy(host)):
        got = staged_h2d(np.asarray(src), dev_keys.device).view(torch.int64)
        assert torch.equal(got, dev_keys)
    cfg = phb.BuildConfig(lambda_=6.0, partition_size=2500.0, encoder="ic-r")
    a = phb.build(dev_keys, cfg).serialize()
    b = phb.build(host.view(np.uint64), cfg).serialize()
    assert a == b
    padded = staged_h2d(np.arange(5, dtype=np.uint8), dev_keys.device, pad=11)
    assert padded.numel() == 16 and padded[5:].sum().item() == 0


def test_bench_workload_slice_vs_oracle(phb, orc):
    """The bench workload's own keys (mix64(i), C2 parameters lambda = 9,
    P = 2500, IC-C) on an 8M-key slice: bytes, trial total and queries equal
    the oracle's; the oracle runs on all host cores."""
    import os

    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(8_000_000, 0)
    cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
    f = phb.build(keys, cfg)
    ref = orc.build(keys, lambda_=9.0, P=2500.0, encoder="ic-c", threads=os.cpu_count() or 1)
    assert f.serialize() == ref.serialize()
    assert f.stats.trials_total == int(ref.trials.sum())
    hi, lo = orc.murmur3_u64(keys[:200_000], f.global_seed)
    assert np.array_equal(f.query_many(keys[:200_000]), ref.query_hashes(hi, lo))
    assert f.is_bijection_on(keys)


@pytest.mark.parametrize("case", range(30))
def test_random_configs_vs_oracle(phb, orc, case):
    """Randomised configurations (lambda, partition size, encoder preset, tie
    order, global seed, key count) against the oracle: bytes, trials and the
    bijection."""
    rng = np.random.default_rng(1000 + case)
    lam = float(rng.choice([2.5, 3.9, 4.5, 5.0, 6.5, 7.0, 8.0, 9.0, 10.0]))
    P = float(rng.choice([100.0, 500.0, 1000.0, 2500.0, 3000.0]))
    enc = str(rng.choice(["ic-c", "ic-r", "mono-c", "mono-r", "mixed:7", "mixed:50"]))
    tie = str(rng.choice(["asc-expected", "desc-expected"]))
    gseed = int(rng.integers(0, 2**63))
    n = int(rng.integers(20_000, 200_000))
    keys = np.unique(rng.integers(0, 2**64, size=n, dtype=np.uint64))
    cfg = phb.BuildConfig(lambda_=lam, partition_size=P, encoder=enc, tie_break=tie,
                          global_seed=gseed)
    f = phb.build(keys, cfg)
    ref = orc.build(keys, lambda_=lam, P=P, encoder=enc, tie_break=tie, global_seed=gseed)
    assert f.serialize() == ref.serialize(), (lam, P, enc, tie, gseed, n)
    assert f.stats.trials_total == int(ref.trials.sum())
    assert f.is_bijection_on(keys)


@pytest.mark.parametrize("case", range(6))
def test_random_string_configs_vs_oracle(phb, orc, case):
    """Randomised configurations over variable-length byte keys (0-120 B,
    full byte range, duplicates removed) against the oracle."""
    rng = np.random.default_rng(2000 + case)
    n = int(rng.integers(5_000, 60_000))
    lens = rng.integers(0, 121, size=n)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    buf = rng.integers(0, 256, size=int(off[-1]), dtype=np.uint8)
    uniq = {bytes(buf[off[i]:off[i + 1]]) for i in range(n)}
    keys = sorted(uniq)
    corpus = phb.KeyCorpus.from_keys(keys)
    lam = float(rng.choice([3.0, 5.0, 8.0]))
    P = float(rng.choice([200.0, 1000.0, 2500.0]))
    enc = str(rng.choice(["ic-c", "ic-r", "mono-r", "mixed:9"]))
    f = phb.build(corpus, phb.BuildConfig(lambda_=lam, partition_size=P, encoder=enc))
    ref = orc.build((corpus.buf, corpus.offsets), lambda_=lam, P=P, encoder=enc)
    assert f.serialize() == ref.serialize(), (lam, P, enc, n)
    assert f.is_bijection_on(corpus)


def test_pinned_chunked_build_equals_device_build(phb):
    """Pinned host keys (> one 8M-key chunk) take the overlapped path: chunked
    copies on a side stream, fixed-capacity grouping per landed chunk, strided
    search. Bytes equal the counted path's (keys already in HBM), also when a
    forced overflow sends the build back to the counted layout."""
    from paper_2404_18497_b200.keygen import synth_u64_device, to_device_chunked
    from paper_2404_18497_b200.mphf import BuildEngine

    n = 20_000_001
    dev_keys = synth_u64_device(n, 5)
    host = torch.empty(n, dtype=torch.int64, pin_memory=True)
    host.copy_(dev_keys)
    cfg = phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r")
    want = phb.build(dev_keys, cfg).serialize()
    assert phb.build(host, cfg).serialize() == want
    # forced overflow: 100 slots per partition cannot hold ~2500 keys
    eng = BuildEngine(cfg)
    eng.padded_capacity = lambda n: 100
    dk, chunks = to_device_chunked(host, dev_keys.device)
    assert chunks and len(chunks) == 3
    res = eng.run(dk, 0, chunks=chunks)
    torch.cuda.synchronize()
    ref = BuildEngine(cfg).run(phb.keygen.to_device(dev_keys, dev_keys.device), 0)
    assert torch.equal(res.blob[57:res.total_bytes], ref.blob[57:ref.total_bytes])


def test_long_and_mixed_length_keys_vs_oracle(phb, orc):
    """Byte keys from 0 B to 6 KB (many murmur3 blocks, every alignment in
    the flat buffer) against the oracle: bytes, trials and queries, through
    both the per-thread and the batched (two-pass, >= 606k keys) query."""
    rng = np.random.default_rng(4242)
    n = 700_000
    lens = rng.integers(0, 64, size=n)
    long_idx = rng.choice(n, 300, replace=False)
    lens[long_idx] = rng.integers(64, 6001, size=300)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    buf = rng.integers(0, 256, size=int(off[-1]), dtype=np.uint8)
    uniq = sorted({bytes(buf[off[i]:off[i + 1]]) for i in range(n)})
    corpus = phb.KeyCorpus.from_keys(uniq)
    cfg = phb.BuildConfig(lambda_=7.0, partition_size=2500.0, encoder="ic-r")
    f = phb.build(corpus, cfg)
    ref = orc.build((corpus.buf, corpus.offsets), lambda_=7.0, P=2500.0, encoder="ic-r")
    assert f.serialize() == ref.serialize()
    assert f.stats.trials_total == int(ref.trials.sum())
    hi, lo = orc.murmur3_many(corpus.buf, corpus.offsets, f.global_seed)
    want = ref.query_hashes(hi, lo)
    assert np.array_equal(f.query_many(corpus), want)            # batched (two-pass) path
    sub = phb.KeyCorpus.from_keys(uniq[:5000])
    assert np.array_equal(f.query_many(sub), want[:5000])        # per-thread path
