"""Batched query rate for byte keys (C5: 100M strings of 10-100 B, lambda=8, IC-R)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import DeviceKeys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(2024)
lens = torch.randint(10, 101, (n,), generator=g, device=dev, dtype=torch.int64)
offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
torch.cumsum(lens, 0, out=offsets[1:])
total = int(offsets[-1].item())
buf = torch.randint(33, 127, (total,), generator=g, device=dev, dtype=torch.uint8)
dk = DeviceKeys(n, buf=buf, offsets=offsets)
f = phb.build(dk, phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r"))
out = f.query_device(dk)
torch.cuda.synchronize()
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = f.query_device(dk)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"strings query {ms:.3f} ms  {n / ms / 1e6:.2f} Gq/s  bijection {f.verify_device(out)}")
