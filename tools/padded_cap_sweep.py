"""Time the fixed-capacity grouping pass (phb_scatter_padded) at C2 for several
per-partition capacities (its footprint grows with the capacity)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import _native
from paper_2404_18497_b200.keygen import synth_u64_device, DeviceKeys
from paper_2404_18497_b200.mphf import BuildEngine
n = 100_000_000
keys = synth_u64_device(n, 0)
dk = DeviceKeys(n, keys64=keys)
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
L = _native.lib()
for cap in (2900, 2901, 2917, 3000, 3001, 3072, 3073, 3200):
    eng = BuildEngine(cfg)
    eng.padded_capacity = lambda n, c=cap: c
    nparts = 40000
    P = _native.ptr; st = _native.stream()
    ts = []
    for r in range(4):
        cursor = torch.empty(nparts, dtype=torch.int32, device="cuda")
        lo = torch.empty(nparts * cap, dtype=torch.int64, device="cuda")
        bid = torch.empty(nparts * cap, dtype=torch.int16, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.phb_scatter_padded(P(keys), n, 0, nparts, P(eng.entries), eng.bcount, cap, 1, P(cursor), P(lo), P(bid), P(flag), st)
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(cap, [round(t, 3) for t in ts])
