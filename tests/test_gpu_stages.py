"""Stage-by-stage parity of the CUDA path (through the C-ABI) against the
reference's golden vectors and the pinned oracle. Bit-exact throughout:
this path is integer / byte work plus a separately-rounded FP64 bucket
function, so there is no tolerance anywhere."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def nat():
    from paper_2404_18497_b200 import _native

    _native.require_device()
    return _native


def u64t(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).to(DEV)


def host_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def test_murmur3_bytes(golden, nat):
    buf = torch.from_numpy(golden["kat_buf"]).to(DEV)
    off = torch.from_numpy(golden["kat_off"]).to(DEV)
    n = len(golden["kat_off"]) - 1
    for s in golden["kat_seeds"]:
        hi = torch.empty(n, dtype=torch.int64, device=DEV)
        lo = torch.empty_like(hi)
        nat.call("phb_murmur3_many", nat.ptr(buf), nat.ptr(off), n, int(s), nat.ptr(hi),
                 nat.ptr(lo), nat.stream())
        assert np.array_equal(host_u64(hi), golden[f"kat_hi_{int(s)}"])
        assert np.array_equal(host_u64(lo), golden[f"kat_lo_{int(s)}"])


def test_murmur3_u64(golden, nat):
    keys = u64t(golden["kat64_keys"])
    n = keys.numel()
    for s in (0, 1, 2**64 - 1):
        hi = torch.empty(n, dtype=torch.int64, device=DEV)
        lo = torch.empty_like(hi)
        nat.call("phb_murmur3_u64", nat.ptr(keys), n, s, nat.ptr(hi), nat.ptr(lo), nat.stream())
        assert np.array_equal(host_u64(hi), golden[f"kat64_hi_{s}"])
        assert np.array_equal(host_u64(lo), golden[f"kat64_lo_{s}"])


def test_murmur3_random_lengths_vs_oracle(nat, orc):
    rng = np.random.default_rng(3)
    lens = rng.integers(0, 130, size=50_000)
    off = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=off[1:])
    buf = rng.integers(0, 256, size=int(off[-1]), dtype=np.uint8)
    want_hi, want_lo = orc.murmur3_many(buf, off, 99)
    dbuf = torch.from_numpy(buf).to(DEV)
    # unaligned start: the kernel must not assume any alignment of buf
    dbuf1 = torch.cat([torch.zeros(3, dtype=torch.uint8, device=DEV), dbuf])[3:]
    doff = torch.from_numpy(off).to(DEV)
    for b in (dbuf, dbuf1):
        hi = torch.empty(len(lens), dtype=torch.int64, device=DEV)
        lo = torch.empty_like(hi)
        nat.call("phb_murmur3_many", nat.ptr(b), nat.ptr(doff), len(lens), 99, nat.ptr(hi),
                 nat.ptr(lo), nat.stream())
        assert np.array_equal(host_u64(hi), want_hi)
        assert np.array_equal(host_u64(lo), want_lo)


def test_bucket_ids(golden, meta, nat, orc):
    his = u64t(golden["bkt_his"])
    n = his.numel()
    for name, (kind, eps, B) in meta["bucket_specs"].items():
        tab = torch.from_numpy(golden[f"tab_{name}"]).to(DEV)
        out = torch.empty(n, dtype=torch.int16, device=DEV)
        nat.call("phb_bucket_ids", nat.ptr(his), n, nat.ptr(tab), B, nat.ptr(out), nat.stream())
        got = out.cpu().numpy().view(np.uint16)
        assert np.array_equal(got, golden[f"bkt_{name}"]), name


def test_bucket_ids_dense_random_vs_oracle(nat, orc):
    """2^24 random words per table: FMA contraction would show up here."""
    rng = np.random.default_rng(17)
    his = rng.integers(0, 2**64, size=1 << 24, dtype=np.uint64)
    d = u64t(his)
    for lam in (4.0, 5.0, 9.0):
        table = orc.tabulate("beta_eps", orc.default_epsilon(lam, 2500.0))
        B = orc.bucket_count(2500.0, lam)
        tab = torch.from_numpy(table).to(DEV)
        out = torch.empty(his.size, dtype=torch.int16, device=DEV)
        nat.call("phb_bucket_ids", nat.ptr(d), his.size, nat.ptr(tab), B, nat.ptr(out),
                 nat.stream())
        got = out.cpu().numpy().view(np.uint16).astype(np.int64)
        assert np.array_equal(got, orc.bucket_ids(his, table, B)), lam


@pytest.mark.parametrize("n", [40_000, 5000, 1, 6250])
def test_layout(golden, meta, nat, n):
    from paper_2404_18497_b200.partitioning import num_partitions_for

    keys = u64t(golden[f"part_{n}_keys"])
    P = meta[f"part_{n}"]["P"]
    nparts = num_partitions_for(n, P)
    counts = torch.zeros(nparts, dtype=torch.int32, device=DEV)
    nat.call("phb_hash_count", None, None, nat.ptr(keys), n, 0, nparts, nat.ptr(counts),
             nat.stream())
    key_off = torch.empty(nparts + 1, dtype=torch.int64, device=DEV)
    deltas = torch.empty_like(key_off)
    stats = torch.empty(2, dtype=torch.int64, device=DEV)
    nat.call("phb_layout", nat.ptr(counts), nparts, 0, 0, n, nparts, nat.ptr(key_off),
             nat.ptr(deltas), nat.ptr(stats), nat.stream())
    want_off = golden[f"part_{n}_keyoff"]
    assert np.array_equal(key_off.cpu().numpy(), want_off)
    assert np.array_equal(deltas.cpu().numpy(), golden[f"part_{n}_deltas"])
    st = stats.cpu().numpy()
    assert st[0] == np.abs(golden[f"part_{n}_deltas"]).max()
    assert st[1] == np.diff(want_off).max()


def _search_inputs(golden, meta, orc, prefix, name):
    m = meta[f"{prefix}_{name}"]
    hi, lo = orc.murmur3_many(golden[f"{prefix}_{name}_buf"], golden[f"{prefix}_{name}_off"],
                              m.get("gseed", 0))
    hs, ls, key_off, _ = orc.partition(hi, lo, m["P"])
    return m, hs, ls, key_off


def _device_search(nat, orc, m, hs, ls, key_off, tie_desc, shuffle=False):
    if shuffle:  # in-partition order must not matter (SURVEY.md §0 finding 2)
        rng = np.random.default_rng(1)
        hs, ls = hs.copy(), ls.copy()
        for j in range(len(key_off) - 1):
            a, b = key_off[j], key_off[j + 1]
            p = rng.permutation(b - a) + a
            hs[a:b], ls[a:b] = hs[p], ls[p]
    table = orc.tabulate("beta_eps", orc.default_epsilon(m["lambda"], m["P"]))
    B = orc.bucket_count(m["P"], m["lambda"])
    nparts = len(key_off) - 1
    seeds = torch.zeros(nparts * B, dtype=torch.int64, device=DEV)
    trials = torch.zeros(nparts * B, dtype=torch.int64, device=DEV)
    status = torch.zeros(nparts, dtype=torch.uint8, device=DEV)
    tab = torch.from_numpy(table).to(DEV)
    koff = torch.from_numpy(key_off).to(DEV)
    dhs, dls = u64t(hs), u64t(ls)  # keep alive across the call (caching allocator)
    nat.call("phb_build_partition_range", nat.ptr(dhs), nat.ptr(dls), nat.ptr(koff), 0,
             nparts, nat.ptr(tab), B, m.get("seed_cap", 1 << 40), int(tie_desc), nat.ptr(seeds),
             nat.ptr(trials), nat.ptr(status), nat.stream())
    return (host_u64(seeds).reshape(nparts, B), trials.cpu().numpy().reshape(nparts, B),
            status.cpu().numpy())


@pytest.mark.parametrize("shuffle", [False, True])
def test_search_seeds_and_trials(golden, meta, nat, orc, shuffle):
    for name in meta["search_cases"]:
        m, hs, ls, key_off = _search_inputs(golden, meta, orc, "srch", name)
        seeds, trials, status = _device_search(nat, orc, m, hs, ls, key_off,
                                               m["tie"] == "asc-expected", shuffle)
        assert not status.any(), name
        assert np.array_equal(seeds, golden[f"srch_{name}_seeds"]), name
        assert np.array_equal(trials, golden[f"srch_{name}_trials"]), name


@pytest.mark.parametrize("name", ["dup", "cap", "capneg"])
def test_search_failure_statuses(golden, meta, nat, orc, name):
    m, hs, ls, key_off = _search_inputs(golden, meta, orc, "stat", name)
    seeds, trials, status = _device_search(nat, orc, m, hs, ls, key_off, True)
    assert np.array_equal(status, golden[f"stat_{name}_status"])
    # failed partitions stop at the same bucket as the reference, so even
    # their partially written seeds / trials agree
    assert np.array_equal(seeds.reshape(-1), golden[f"stat_{name}_seeds"])
    assert np.array_equal(trials.reshape(-1), golden[f"stat_{name}_trials"])


@pytest.mark.parametrize("lam,P,n", [(4.0, 2500.0, 300_000), (7.0, 2500.0, 200_000),
                                     (9.0, 2500.0, 200_000), (3.0, 600.0, 100_000),
                                     (14.0, 2500.0, 40_000), (1.5, 64.0, 30_000)])
def test_search_vs_oracle_random(nat, orc, lam, P, n):
    rng = np.random.default_rng(int(lam * 100) + n)
    keys = rng.integers(0, 2**64, size=n, dtype=np.uint64)
    hi, lo = orc.murmur3_u64(np.unique(keys), 0)
    hs, ls, key_off, _ = orc.partition(hi, lo, P)
    table = orc.tabulate("beta_eps", orc.default_epsilon(lam, P))
    B = orc.bucket_count(P, lam)
    for tie in (1, 0):
        ws, wt, wst = orc.build_partition_range(hs, ls, key_off, 0, len(key_off) - 1, table, B,
                                                1 << 40, tie, threads=8)
        m = {"lambda": lam, "P": P}
        seeds, trials, status = _device_search(nat, orc, m, hs, ls, key_off, tie, shuffle=True)
        assert np.array_equal(status, wst)
        assert np.array_equal(seeds, ws)
        assert np.array_equal(trials, wt)


@pytest.mark.parametrize("nparts", [1, 2, 3, 4095, 4096, 4097, 8192, 123_457, 600_000])
def test_layout_multi_tile(nat, nparts):
    """K2's multi-CTA scan (tiles of 4096 partitions, decoupled look-back)
    against numpy, at tile boundaries and at 147 tiles, with a shard offset
    (key_base / part_base as the multi-GPU owner ranges pass them)."""
    rng = np.random.default_rng(nparts)
    counts_np = rng.integers(0, 5000, size=nparts).astype(np.int64)
    part_base = nparts // 3
    gnparts = nparts + part_base + 7
    key_base = int(rng.integers(0, 1_000_000))
    gn = int(counts_np.sum()) + key_base + 12345
    counts = torch.from_numpy(counts_np.astype(np.int32)).to(DEV)
    key_off = torch.empty(nparts + 1, dtype=torch.int64, device=DEV)
    deltas = torch.empty_like(key_off)
    stats = torch.empty(2, dtype=torch.int64, device=DEV)
    nat.call("phb_layout", nat.ptr(counts), nparts, key_base, part_base, gn, gnparts,
             nat.ptr(key_off), nat.ptr(deltas), nat.ptr(stats), nat.stream())
    want_off = np.zeros(nparts + 1, np.int64)
    np.cumsum(counts_np, out=want_off[1:])
    j = np.arange(nparts + 1, dtype=object) + part_base
    expected = np.array((2 * j * gn + gnparts) // (2 * gnparts), dtype=np.int64)
    want_d = key_base + want_off - expected
    assert np.array_equal(key_off.cpu().numpy(), want_off)
    assert np.array_equal(deltas.cpu().numpy(), want_d)
    st = stats.cpu().numpy()
    assert st[0] == np.abs(want_d).max() and st[1] == counts_np.max()
