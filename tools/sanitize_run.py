"""Small builds + queries for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2404_18497_b200 as phb

rng = np.random.default_rng(5)
keys = np.unique(rng.integers(0, 2**64, size=30_000, dtype=np.uint64))
for enc, lam, P in (("ic-c", 9.0, 2500.0), ("ic-r", 5.0, 300.0), ("mono-r", 7.0, 1000.0)):
    f = phb.build(keys, phb.BuildConfig(lambda_=lam, partition_size=P, encoder=enc))
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    assert f.verify_device(f.query_device(dk))
    assert torch.equal(f.query_encoded_device(dk), f.query_device(dk))
    g = phb.Mphf.deserialize(f.serialize())
    assert torch.equal(g.query_device(dk), f.query_device(dk))
# multi-tile layout (10k partitions), the low-lambda search kernel, and the
# shared-memory query path (>= 148 * 4096 u64 keys)
big = np.unique(rng.integers(0, 2**64, size=1_000_000, dtype=np.uint64))
f = phb.build(big, phb.BuildConfig(lambda_=4.0, partition_size=100.0, encoder="ic-c"))
db = torch.from_numpy(big.view(np.int64)).cuda()
assert f.verify_device(f.query_device(db))
# the encoded-section shared-table query (8-byte column descriptors, seed-hash table)
assert torch.equal(f.query_encoded_device(db), f.query_device(db))
# string keys: the batched query in two passes (hash pairs, shared-table query)
scorpus = phb.gen_keys(650_000, 11)
fs = phb.build(scorpus, phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r"))
assert fs.is_bijection_on(scorpus)
corpus = phb.gen_keys(5000, 3)
f = phb.build(corpus, phb.BuildConfig(lambda_=8.0, partition_size=500.0))
assert f.is_bijection_on(corpus)
torch.cuda.synchronize()
print("sanitize run ok")
