"""Work and per-phase cycle counters of the search kernel.

Needs a -DPHB_STATS build, selected with PHB_LIB:
  tools/build_variants.sh stats -DPHB_STATS
  PHB_LIB=_variants/stats.so python tools/search_stats.py [n] [lambda]
Cycle counters are summed clock64() deltas of lane 0 of every warp, so the
shares (not the absolute values) are what to read.
"""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import _native
from paper_2404_18497_b200.keygen import synth_u64_device, to_device
from paper_2404_18497_b200.mphf import BuildEngine
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
lam = float(sys.argv[2]) if len(sys.argv) > 2 else 9.0
keys = synth_u64_device(n, 0); dk = to_device(keys, keys.device)
eng = BuildEngine(phb.BuildConfig(lambda_=lam, partition_size=2500.0, encoder="ic-c"))
L = _native.lib(); st = np.zeros(32, np.uint64)
eng.run(dk, 0); torch.cuda.synchronize()
L.phb_search_stats(st.ctypes.data_as(ctypes.c_void_p), 1)
res = eng.run(dk, 0); torch.cuda.synchronize()
L.phb_search_stats(st.ctypes.data_as(ctypes.c_void_p), 1)
nparts = res.nparts
print(f"n={n} lambda={lam} nparts={nparts} trials/key={res.trials_total / n:.1f}")
names = ["G1 batches", "G2 batches", "G4 batches", "small key-steps", "generic s-iters",
         "generic key-rounds", "singletons", "buckets k>=2", "early exits", "generic d-searches"]
for i, nm in enumerate(names):
    print(f"{nm:20s} total {int(st[i]):14d}  per partition {st[i] / nparts:10.1f}")
cyc = {"queue+output": st[14], "prologue": st[10], "singletons": st[11], "small k<=32": st[12],
       "generic k>32": st[13]}
tot = sum(int(v) for v in cyc.values())
print("cycle shares (lane-0 clock64 sums):")
for k, v in cyc.items():
    print(f"  {k:14s} {int(v) / tot * 100:6.2f}%   {int(v) / nparts:12.0f} cyc/partition")
for c, nm in enumerate(["k 2..8", "k 9..16", "k 17..32"]):
    nb = int(st[19 + c]); cy = int(st[16 + c]); sd = int(st[22 + c])
    print(f"  {nm:10s} buckets/part {nb / nparts:7.1f}  cycles share {cy / tot * 100:6.2f}%  "
          f"seeds/bucket {sd / max(nb, 1):8.2f}  cyc/seed {cy / max(sd, 1):8.0f}")
