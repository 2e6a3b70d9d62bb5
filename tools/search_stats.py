"""Work counters of the search kernel (needs a -DPHB_STATS build via PHB_LIB)."""
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
L = _native.lib(); st = np.zeros(16, np.uint64)
L.phb_search_stats(st.ctypes.data_as(ctypes.c_void_p), 1)
res = eng.run(dk, 0); torch.cuda.synchronize()
L.phb_search_stats(st.ctypes.data_as(ctypes.c_void_p), 1)
nparts = res.nparts
names = ["G1 batches", "G2 batches", "G4 batches", "small key-steps", "generic s-iters",
         "generic key-rounds", "singletons", "buckets k>=2", "early exits"]
for i, nm in enumerate(names):
    print(f"{nm:20s} total {int(st[i]):14d}  per partition {st[i] / nparts:10.1f}")
