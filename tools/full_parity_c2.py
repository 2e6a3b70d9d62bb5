"""One-off full-size parity check: the bench workload (C2: 100M keys mix64(i),
lambda=9, P=2500, IC-C) built on the GPU and by the oracle (all host cores);
serialized bytes, trial totals and a query sample must agree."""
import hashlib, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2404_18497_b200 as phb
from oracle import oracle
from paper_2404_18497_b200.keygen import synth_u64

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
oracle.build_lib()
keys = synth_u64(n, 0)
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
t = time.perf_counter(); f = phb.build(keys, cfg); tg = time.perf_counter() - t
blob = f.serialize()
t = time.perf_counter()
ref = oracle.build(keys, lambda_=9.0, P=2500.0, encoder="ic-c", threads=os.cpu_count())
tc = time.perf_counter() - t
rblob = ref.serialize()
hi, lo = oracle.murmur3_u64(keys[:1_000_000], f.global_seed)
q_ok = bool(np.array_equal(f.query_many(keys[:1_000_000]), ref.query_hashes(hi, lo)))
print(f"n={n:,} gpu build (API, host keys) {tg:.2f} s, oracle {tc:.1f} s on {os.cpu_count()} cores")
print(f"bytes equal: {blob == rblob} ({len(blob):,} B, sha256 {hashlib.sha256(blob).hexdigest()[:16]}"
      f" vs {hashlib.sha256(rblob).hexdigest()[:16]})")
print(f"trials equal: {f.stats.trials_total == int(ref.trials.sum())} ({f.stats.trials_total:,})")
print(f"queries (first 1M keys) equal: {q_ok}; bijection: {f.is_bijection_on(keys)}")
