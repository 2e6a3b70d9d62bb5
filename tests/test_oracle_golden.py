"""The oracle (oracle/phobic_oracle.c) against the reference's own outputs.

Pins the CPU restatement before it is trusted as the GPU parity checker:
every stage is compared with golden vectors produced by running pilothash
itself (tests/golden/make_golden.py).
"""

import hashlib

import numpy as np
import pytest


def test_master_hash_bytes(golden, orc):
    buf, off = golden["kat_buf"], golden["kat_off"]
    for s in golden["kat_seeds"]:
        hi, lo = orc.murmur3_many(buf, off, int(s))
        assert np.array_equal(hi, golden[f"kat_hi_{int(s)}"])
        assert np.array_equal(lo, golden[f"kat_lo_{int(s)}"])


def test_master_hash_public_vector(orc):
    # canonical MurmurHash3_x64_128("hello", 0)
    hi, lo = orc.murmur3_many(np.frombuffer(b"hello", np.uint8), np.array([0, 5]), 0)
    assert (int(hi[0]), int(lo[0])) == (0xCBD8A7B341BD9B02, 0x5B1E906A48AE1D19)


def test_master_hash_u64(golden, orc):
    keys = golden["kat64_keys"]
    for s in (0, 1, 2**64 - 1):
        hi, lo = orc.murmur3_u64(keys, s)
        assert np.array_equal(hi, golden[f"kat64_hi_{s}"])
        assert np.array_equal(lo, golden[f"kat64_lo_{s}"])


def test_tables_and_buckets(golden, meta, orc):
    his = golden["bkt_his"]
    for name, (kind, eps, B) in meta["bucket_specs"].items():
        table = orc.tabulate(kind, eps)
        assert np.array_equal(table, golden[f"tab_{name}"]), name
        assert np.array_equal(orc.bucket_ids(his, table, B), golden[f"bkt_{name}"]), name


@pytest.mark.parametrize("n", [40_000, 5000, 1, 6250])
def test_partition_layout(golden, meta, orc, n):
    keys = golden[f"part_{n}_keys"]
    hi, lo = orc.murmur3_u64(keys, 0)
    hs, ls, key_off, deltas = orc.partition(hi, lo, meta[f"part_{n}"]["P"])
    assert np.array_equal(key_off, golden[f"part_{n}_keyoff"])
    assert np.array_equal(deltas, golden[f"part_{n}_deltas"])
    assert hashlib.sha256(hs.tobytes() + ls.tobytes()).hexdigest() == meta[f"part_{n}"]["sorted_sha"]


def _search(golden, meta, orc, name, threads=1):
    m = meta[f"srch_{name}"]
    hi, lo = orc.murmur3_many(golden[f"srch_{name}_buf"], golden[f"srch_{name}_off"], m["gseed"])
    hs, ls, key_off, _ = orc.partition(hi, lo, m["P"])
    table = orc.tabulate("beta_eps", orc.default_epsilon(m["lambda"], m["P"]))
    B = orc.bucket_count(m["P"], m["lambda"])
    return orc.build_partition_range(hs, ls, key_off, 0, len(key_off) - 1, table, B,
                                     m["seed_cap"], m["tie"] == "asc-expected", threads)


def test_search_seeds_and_trials(golden, meta, orc):
    for name in meta["search_cases"]:
        seeds, trials, status = _search(golden, meta, orc, name)
        assert not status.any(), name
        assert np.array_equal(seeds, golden[f"srch_{name}_seeds"]), name
        assert np.array_equal(trials, golden[f"srch_{name}_trials"]), name


def test_search_thread_invariance(golden, meta, orc):
    a = _search(golden, meta, orc, "u5", threads=1)
    b = _search(golden, meta, orc, "u5", threads=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["dup", "cap", "capneg"])
def test_failure_statuses(golden, meta, orc, name):
    m = meta[f"stat_{name}"]
    hi, lo = orc.murmur3_many(golden[f"stat_{name}_buf"], golden[f"stat_{name}_off"], 0)
    hs, ls, key_off, _ = orc.partition(hi, lo, m["P"])
    table = orc.tabulate("beta_eps", orc.default_epsilon(m["lambda"], m["P"]))
    B = orc.bucket_count(m["P"], m["lambda"])
    seeds, trials, status = orc.build_partition_range(hs, ls, key_off, 0, len(key_off) - 1,
                                                      table, B, m["seed_cap"], True)
    assert np.array_equal(status, golden[f"stat_{name}_status"])
    assert np.array_equal(seeds.reshape(-1), golden[f"stat_{name}_seeds"])
    assert np.array_equal(trials.reshape(-1), golden[f"stat_{name}_trials"])


def _e2e_cases(meta):
    out = []
    for k, v in meta.items():
        if k.startswith("e2e_"):
            for enc in v["bytes"]:
                out.append((k[4:], enc))
    return out


def test_end_to_end_bytes_and_queries(golden, meta, orc):
    for name, enc in _e2e_cases(meta):
        m = meta[f"e2e_{name}"]
        keys = (golden[f"e2e_{name}_buf"], golden[f"e2e_{name}_off"])
        f = orc.build(keys, lambda_=m["lambda"], P=m["P"], encoder=enc,
                      tie_break=m["tie"], global_seed=m["gseed"], threads=2)
        blob = f.serialize()
        want = golden[f"e2e_{name}_{enc}"].tobytes()
        assert len(blob) == len(want), (name, enc)
        assert blob == want, (name, enc)
        assert int(f.trials.sum()) == m["bytes"][enc]["trials_total"]
        if f"e2e_{name}_query" in golden.files and enc == list(m["bytes"])[0]:
            hi, lo = orc.hash_keys(keys, f.global_seed)
            assert np.array_equal(f.query_hashes(hi, lo), golden[f"e2e_{name}_query"])
