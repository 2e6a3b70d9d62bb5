"""analysis.measure_work on the device == the reference's measure_work
(analysis.py:185-249) on the same keys: per-bucket and per-partition trials,
bucket-size histograms and bits/key (goldens from tests/golden/make_golden_work.py)."""

import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _corpus(desc):
    from paper_2404_18497_b200 import KeyCorpus, gen_keys

    if "gen_keys" in desc:
        return gen_keys(*desc["gen_keys"])
    rng = np.random.default_rng(2024)
    keys = np.unique(rng.integers(0, 2**64, size=desc["u64_unique_rng2024"], dtype=np.uint64))
    keys = keys[rng.permutation(len(keys))]
    return KeyCorpus(keys.view(np.uint8).copy(), np.arange(len(keys) + 1, dtype=np.int64) * 8)


def test_measure_work_equals_reference():
    from paper_2404_18497_b200 import AssignmentSpec, BuildConfig
    from paper_2404_18497_b200.analysis import CSV_HEADER, measure_work, work_csv

    cases = json.loads((GOLDEN / "measure_work.json").read_text())
    for case in cases:
        corpus = _corpus(case["corpus"])
        cfg = BuildConfig(**case["config"])
        variants = [AssignmentSpec(k, e) for k, e in case["variants"]]
        reps = measure_work(corpus, variants, cfg)
        assert len(reps) == len(case["reports"])
        for r, want in zip(reps, case["reports"]):
            assert r.assignment == want["assignment"] and r.n == want["n"]
            assert r.per_bucket_trials.tolist() == want["per_bucket_trials"], case["name"]
            assert r.per_partition_trials.tolist() == want["per_partition_trials"], case["name"]
            assert r.total_trials == want["total_trials"]
            assert r.trials_per_key == r.total_trials / r.n
            assert {str(k): v for k, v in r.size_histogram.items()} == want["size_histogram"]
            assert sum(s * c for s, c in r.size_histogram.items()) == r.n
            assert r.bits_per_key == want["bits_per_key"]
        lines = work_csv(reps).strip().split("\n")
        assert lines[0] == CSV_HEADER
        assert [ln.rsplit(",", 1)[0] for ln in lines] == case["csv_prefix"]


def test_measure_work_deterministic():
    """test_analysis.py:187-194."""
    from paper_2404_18497_b200 import BuildConfig, gen_keys
    from paper_2404_18497_b200.analysis import measure_work

    corpus = gen_keys(2000, 13)
    cfg = BuildConfig(lambda_=4.0, partition_size=500.0, global_seed=13)
    r1 = measure_work(corpus, ["beta_eps"], cfg)[0]
    r2 = measure_work(corpus, ["beta_eps"], cfg)[0]
    assert r1.total_trials == r2.total_trials
    assert r1.bits_per_key == r2.bits_per_key
    assert np.array_equal(r1.per_bucket_trials, r2.per_bucket_trials)
