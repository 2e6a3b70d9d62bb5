"""Golden outputs of the REFERENCE's analysis.measure_work (pilothash 0.1.0,
analysis.py:185-249), for tests/test_gpu_analysis.py.

Runs only in the development container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_work.py

Writes tests/golden/measure_work.json.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from pilothash import BuildConfig, gen_keys  # noqa: E402
from pilothash.analysis import measure_work, work_csv  # noqa: E402
from pilothash.assignment import AssignmentSpec, default_epsilon  # noqa: E402
from pilothash.keygen import KeyCorpus  # noqa: E402

OUT = Path(__file__).resolve().parent
cases = []


def run(name, corpus, variants, cfg, corpus_desc):
    reps = measure_work(corpus, variants, cfg)
    cases.append({
        "name": name, "corpus": corpus_desc,
        "config": {"lambda_": cfg.lambda_, "partition_size": cfg.partition_size,
                   "global_seed": cfg.global_seed, "encoder": cfg.encoder},
        "variants": [[v.kind, v.epsilon] if isinstance(v, AssignmentSpec) else [v, 0.0]
                     for v in variants],
        "csv_prefix": [ln.rsplit(",", 1)[0] for ln in work_csv(reps).strip().split("\n")],
        "reports": [{
            "assignment": r.assignment, "n": r.n,
            "per_bucket_trials": [int(x) for x in r.per_bucket_trials],
            "per_partition_trials": [int(x) for x in r.per_partition_trials],
            "total_trials": int(r.total_trials),
            "size_histogram": {str(k): int(v) for k, v in sorted(r.size_histogram.items())},
            "bits_per_key": r.bits_per_key,
        } for r in reps],
    })


# the reference's own smoke case (test_analysis.py:169-184)
run("smoke", gen_keys(4000, 12), [AssignmentSpec("uniform"), "beta_eps"],
    BuildConfig(lambda_=4.0, partition_size=500.0, global_seed=12),
    {"gen_keys": [4000, 12]})

# u64 keys, the acceptance-style variants (test_acceptance.py:143-160)
rng = np.random.default_rng(2024)
keys = np.unique(rng.integers(0, 2**64, size=30_000, dtype=np.uint64))
keys = keys[rng.permutation(len(keys))]
corpus = KeyCorpus(keys.view(np.uint8).copy(), np.arange(len(keys) + 1, dtype=np.int64) * 8)
run("u64_l8", corpus,
    [AssignmentSpec("beta_eps", default_epsilon(8.0, 2500.0)), AssignmentSpec("skew"),
     AssignmentSpec("beta_star")],
    BuildConfig(lambda_=8.0, partition_size=2500.0, global_seed=1, encoder="ic-c"),
    {"u64_unique_rng2024": 30_000})

(OUT / "measure_work.json").write_text(json.dumps(cases))
print("wrote", OUT / "measure_work.json", sum(len(c["reports"]) for c in cases), "reports")
