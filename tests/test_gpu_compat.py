"""The pilothash._kernels drop-in (compat_kernels) driven exactly the way the
reference's builder / mphf modules call it, against the reference goldens."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_compat_murmur3_many(golden):
    from paper_2404_18497_b200 import compat_kernels as K

    buf, off = golden["kat_buf"], golden["kat_off"]
    n = len(off) - 1
    for s in golden["kat_seeds"]:
        hi = np.empty(n, np.uint64)
        lo = np.empty(n, np.uint64)
        K.murmur3_many(buf, off, np.uint64(s), hi, lo)
        assert np.array_equal(hi, golden[f"kat_hi_{int(s)}"])
        assert np.array_equal(lo, golden[f"kat_lo_{int(s)}"])


def test_compat_build_partition_range_and_query(golden, meta, orc):
    """builder.build_all_partitions (builder.py:224-277) + mphf.query_many
    (mphf.py:130-145) semantics through the shim."""
    from paper_2404_18497_b200 import compat_kernels as K

    for name in meta["search_cases"]:
        m = meta[f"srch_{name}"]
        hi, lo = orc.murmur3_many(golden[f"srch_{name}_buf"], golden[f"srch_{name}_off"],
                                  m["gseed"])
        hs, ls, key_off, deltas = orc.partition(hi, lo, m["P"])
        table = orc.tabulate("beta_eps", orc.default_epsilon(m["lambda"], m["P"]))
        B = orc.bucket_count(m["P"], m["lambda"])
        nparts = len(key_off) - 1
        seeds = np.zeros(nparts * B, np.uint64)
        trials = np.zeros(nparts * B, np.int64)
        status = np.zeros(nparts, np.uint8)
        K.build_partition_range(hs, ls, key_off, 0, nparts, table, B, m["seed_cap"],
                                m["tie"] == "asc-expected", seeds, trials, status)
        assert not status.any()
        assert np.array_equal(seeds.reshape(nparts, B), golden[f"srch_{name}_seeds"])
        assert np.array_equal(trials.reshape(nparts, B), golden[f"srch_{name}_trials"])
        out = np.empty(len(hi), np.int64)
        K.query_many_kernel(hi, lo, len(hi), nparts, deltas, table, B, seeds, out)
        want = orc.query_many(hi, lo, len(hi), nparts, deltas, table, B, seeds.reshape(nparts, B))
        assert np.array_equal(out, want)
        assert np.array_equal(np.sort(out), np.arange(len(hi)))


def test_compat_build_partition_range_threads(golden, meta, orc):
    """builder.build_all_partitions with config.threads = 3 (builder.py:260-271):
    concurrent calls over disjoint partition ranges of SHARED output arrays
    must leave every thread's rows intact."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2404_18497_b200 import compat_kernels as K

    for name in meta["search_cases"]:
        m = meta[f"srch_{name}"]
        hi, lo = orc.murmur3_many(golden[f"srch_{name}_buf"], golden[f"srch_{name}_off"],
                                  m["gseed"])
        hs, ls, key_off, _ = orc.partition(hi, lo, m["P"])
        table = orc.tabulate("beta_eps", orc.default_epsilon(m["lambda"], m["P"]))
        B = orc.bucket_count(m["P"], m["lambda"])
        nparts = len(key_off) - 1
        seeds = np.zeros(nparts * B, np.uint64)
        trials = np.zeros(nparts * B, np.int64)
        status = np.full(nparts, 7, np.uint8)  # every row must be written by its owner
        nchunks = min(3, nparts)
        bounds = np.linspace(0, nparts, nchunks + 1).astype(np.int64)
        with ThreadPoolExecutor(max_workers=nchunks) as pool:
            futs = [pool.submit(K.build_partition_range, hs, ls, key_off, int(bounds[c]),
                                int(bounds[c + 1]), table, B, m["seed_cap"],
                                m["tie"] == "asc-expected", seeds, trials, status)
                    for c in range(nchunks)]
            for f in futs:
                f.result()
        assert not status.any()
        assert np.array_equal(seeds.reshape(nparts, B), golden[f"srch_{name}_seeds"])
        assert np.array_equal(trials.reshape(nparts, B), golden[f"srch_{name}_trials"])
