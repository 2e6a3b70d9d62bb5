"""Generate golden vectors by running the REFERENCE itself (pilothash 0.1.0).

Runs only in the development container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ golden_meta.json). The fixtures are small
and committed; the GPU box never reads /root/reference. Every stage of the
construction path gets its own vectors so that a parity failure points at
one stage: master hash (murmur3_many), assignment tables and bucket ids,
partition layout, build_all_partitions seeds + per-bucket trials (both tie
orders, several lambda), status codes for the failure paths, serialized
bytes for every encoder preset, and query outputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import pilothash  # noqa: E402
from pilothash import BuildConfig, build, gen_keys  # noqa: E402
from pilothash import _kernels  # noqa: E402
from pilothash.assignment import AssignmentSpec, bucket_many, tabulate  # noqa: E402
from pilothash.builder import build_all_partitions  # noqa: E402
from pilothash.hashing import master_hash_many, normalized_hash_many  # noqa: E402
from pilothash.keygen import KeyCorpus  # noqa: E402
from pilothash.partitioning import partition_arrays  # noqa: E402

OUT = Path(__file__).resolve().parent
G: dict[str, np.ndarray] = {}
META: dict = {"reference": "pilothash " + pilothash.__version__}


def u64_corpus(keys: np.ndarray) -> KeyCorpus:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    return KeyCorpus(keys.view(np.uint8).copy(), np.arange(len(keys) + 1, dtype=np.int64) * 8)


def u64_keys(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    k = np.unique(rng.integers(0, 2**64, size=n + 64, dtype=np.uint64))[:n]
    return k[rng.permutation(len(k))]


def put(name, arr):
    G[name] = np.asarray(arr)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


# 1. master hash -----------------------------------------------------------
texts = [b"", b"a", b"hello", b"abcdefghi", b"0123456789abcdef", b"0123456789abcdefX",
         b"0123456789abcdef0123456789abcde", b"0123456789abcdef0123456789abcdef"]
rng = np.random.default_rng(7)
for L in list(range(0, 41)) + [63, 64, 65, 100, 127, 128, 255]:
    texts.append(bytes(rng.integers(0, 256, size=L, dtype=np.uint8)))
kc = KeyCorpus.from_keys(texts)
put("kat_buf", kc.buf)
put("kat_off", kc.offsets)
seeds = [0, 1, 7, 12345, 2**64 - 1]
put("kat_seeds", np.array(seeds, dtype=np.uint64))
for s in seeds:
    h, l = master_hash_many(kc.buf, kc.offsets, s)
    put(f"kat_hi_{s}", h)
    put(f"kat_lo_{s}", l)
k64 = np.concatenate([np.array([0, 1, 0x0123456789ABCDEF, 2**64 - 1], dtype=np.uint64),
                      u64_keys(2000, 11)])
put("kat64_keys", k64)
c64 = u64_corpus(k64)
for s in (0, 1, 2**64 - 1):
    h, l = master_hash_many(c64.buf, c64.offsets, s)
    put(f"kat64_hi_{s}", h)
    put(f"kat64_lo_{s}", l)

# 2. tables and bucket ids ---------------------------------------------------
specs = {
    "be5": (AssignmentSpec("beta_eps", 5.0 / (5.0 * 50.0)), 500),
    "be9": (AssignmentSpec("beta_eps", 9.0 / (5.0 * 50.0)), 278),
    "be4": (AssignmentSpec("beta_eps", 4.0 / (5.0 * 50.0)), 625),
    "uni": (AssignmentSpec("uniform"), 100),
    "skew": (AssignmentSpec("skew"), 37),
    "bstar": (AssignmentSpec("beta_star"), 312),
    "be32": (AssignmentSpec("beta_eps", 0.032), 312),
}
his = np.concatenate([np.array([0, 1, 2**63, 2**64 - 1], dtype=np.uint64),
                      np.random.default_rng(5).integers(0, 2**64, 60_000, dtype=np.uint64)])
put("bkt_his", his)
x = normalized_hash_many(his)
for name, (spec, B) in specs.items():
    t = tabulate(spec)
    put(f"tab_{name}", t.entries)
    put(f"bkt_{name}", bucket_many(t, x, B).astype(np.uint16))
META["bucket_specs"] = {k: [v[0].kind, v[0].epsilon, v[1]] for k, v in specs.items()}

# 3. partition layout --------------------------------------------------------
for n, P in [(40_000, 2500.0), (5000, 500.0), (1, 2500.0), (6250, 2500.0)]:
    keys = u64_keys(n, 300 + n)
    c = u64_corpus(keys)
    h, l = master_hash_many(c.buf, c.offsets, 0)
    ks, lay = partition_arrays(h, l, P)
    put(f"part_{n}_keys", keys)
    put(f"part_{n}_keyoff", ks.key_offsets)
    put(f"part_{n}_deltas", lay.deltas)
    META[f"part_{n}"] = {"P": P, "sorted_sha": sha(ks.his.tobytes() + ks.los.tobytes())}

# 4. build_all_partitions: seeds + per-bucket trials -------------------------
search_cases = []


def search_case(name, corpus, lam, P, tie, gseed, seed_cap=1 << 40):
    cfg = BuildConfig(lambda_=lam, partition_size=P, tie_break=tie, seed_cap=seed_cap)
    table = tabulate(cfg.resolved_assignment())
    h, l = master_hash_many(corpus.buf, corpus.offsets, gseed)
    ks, lay = partition_arrays(h, l, P)
    seeds, trials = build_all_partitions(ks.his, ks.los, ks.key_offsets, table, cfg)
    put(f"srch_{name}_buf", corpus.buf)
    put(f"srch_{name}_off", corpus.offsets)
    put(f"srch_{name}_seeds", seeds)
    put(f"srch_{name}_trials", trials)
    META[f"srch_{name}"] = {"lambda": lam, "P": P, "tie": tie, "gseed": gseed,
                            "seed_cap": seed_cap, "trials_total": int(trials.sum())}
    search_cases.append(name)


search_case("s4asc", gen_keys(3000, 100), 4.0, 300.0, "asc-expected", 5)
search_case("s4desc", gen_keys(3000, 100), 4.0, 300.0, "desc-expected", 5)
search_case("s8asc", gen_keys(4000, 101), 8.0, 500.0, "asc-expected", 5)
search_case("s8desc", gen_keys(4000, 101), 8.0, 500.0, "desc-expected", 5)
search_case("u5", u64_corpus(u64_keys(20_000, 21)), 5.0, 2500.0, "asc-expected", 0)
search_case("u9", u64_corpus(u64_keys(30_000, 22)), 9.0, 2500.0, "asc-expected", 0)
search_case("u6", u64_corpus(u64_keys(5000, 23)), 6.0, 400.0, "asc-expected", 0)
search_case("u12", u64_corpus(u64_keys(8000, 24)), 12.0, 1000.0, "asc-expected", 0)
META["search_cases"] = search_cases

# 4b. failure statuses straight from the reference kernel --------------------
def status_case(name, corpus, lam, P, seed_cap):
    cfg = BuildConfig(lambda_=lam, partition_size=P)
    table = tabulate(cfg.resolved_assignment())
    h, l = master_hash_many(corpus.buf, corpus.offsets, 0)
    ks, lay = partition_arrays(h, l, P)
    nparts = lay.num_partitions
    B = cfg.bucket_count
    seeds = np.zeros(nparts * B, np.uint64)
    trials = np.zeros(nparts * B, np.int64)
    status = np.zeros(nparts, np.uint8)
    _kernels.build_partition_range(ks.his, ks.los, ks.key_offsets, 0, nparts,
                                   np.ascontiguousarray(table.entries), B, seed_cap, True,
                                   seeds, trials, status)
    put(f"stat_{name}_buf", corpus.buf)
    put(f"stat_{name}_off", corpus.offsets)
    put(f"stat_{name}_seeds", seeds)
    put(f"stat_{name}_trials", trials)
    put(f"stat_{name}_status", status)
    META[f"stat_{name}"] = {"lambda": lam, "P": P, "seed_cap": seed_cap}


dup = [b"k%d" % i for i in range(2000)] + [b"k7", b"k1999"]
status_case("dup", KeyCorpus.from_keys(dup), 4.0, 250.0, 1 << 40)
status_case("cap", gen_keys(3000, 55), 6.0, 300.0, 300)
status_case("capneg", gen_keys(600, 56), 4.0, 300.0, -1)

# 5. end to end: serialized bytes + queries for every preset -----------------
def e2e_case(name, corpus, cfg, presets, store_queries=True):
    META[f"e2e_{name}"] = {"lambda": cfg.lambda_, "P": cfg.partition_size,
                           "gseed": cfg.global_seed, "tie": cfg.tie_break, "bytes": {}}
    put(f"e2e_{name}_buf", corpus.buf)
    put(f"e2e_{name}_off", corpus.offsets)
    for enc in presets:
        c2 = BuildConfig(lambda_=cfg.lambda_, partition_size=cfg.partition_size,
                         global_seed=cfg.global_seed, encoder=enc, tie_break=cfg.tie_break)
        f = build(corpus, c2)
        blob = f.serialize()
        put(f"e2e_{name}_{enc}", np.frombuffer(blob, dtype=np.uint8))
        META[f"e2e_{name}"]["bytes"][enc] = {"len": len(blob), "sha": sha(blob),
                                             "bits_per_key": f.bits_per_key(),
                                             "attempts": f.stats.attempts,
                                             "trials_total": f.stats.trials_total}
        if store_queries and enc == presets[0]:
            put(f"e2e_{name}_query", f.query_many(corpus).astype(np.int32))


small = gen_keys(20_000, 1)
e2e_case("small", small, BuildConfig(lambda_=4.0, partition_size=500.0, global_seed=3),
         ["ic-r", "ic-c", "mixed:7", "mono-r", "mono-c"])
tiny = u64_corpus(np.arange(1, 1001, dtype=np.uint64))
e2e_case("tiny", tiny, BuildConfig(lambda_=4.0, partition_size=250.0), ["ic-c", "ic-r"])
c1 = u64_corpus(u64_keys(60_000, 2024))
e2e_case("c1", c1, BuildConfig(lambda_=5.0, partition_size=2500.0), ["ic-c", "ic-r"])
c9 = u64_corpus(u64_keys(50_000, 2025))
e2e_case("c9", c9, BuildConfig(lambda_=9.0, partition_size=2500.0), ["ic-c"])
strs = gen_keys(3000, 77)
e2e_case("desc", strs, BuildConfig(lambda_=6.0, partition_size=700.0, global_seed=11,
                                   tie_break="desc-expected"), ["ic-r", "mixed:40"])
one = KeyCorpus.from_keys([b"only"])
e2e_case("one", one, BuildConfig(), ["ic-r", "ic-c"])
three = KeyCorpus.from_keys([b"alpha", b"beta", b"gamma"])
e2e_case("three", three, BuildConfig(lambda_=2.0, partition_size=3.0), ["ic-r"])

np.savez_compressed(OUT / "golden.npz", **G)
(OUT / "golden_meta.json").write_text(json.dumps(META, indent=1, sort_keys=True))
print("wrote", OUT / "golden.npz", sum(a.nbytes for a in G.values()) / 1e6, "MB raw")
