"""Matrix vs encoded-section query rate at C2 (100M u64 keys, lambda=9)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
enc = sys.argv[2] if len(sys.argv) > 2 else "ic-c"
keys = synth_u64_device(n, 0)
dk = DeviceKeys(n, keys64=keys)
f = phb.build(dk, phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder=enc))
for name, fn in (("matrix", f.query_device), ("encoded", f.query_encoded_device)):
    out = fn(dk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out = fn(dk)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{enc} {name:8s} {ms:7.3f} ms  {n / ms / 1e6:8.2f} Gq/s  bijection {f.verify_device(out)}")
g = phb.Mphf.deserialize(f.serialize())
for name, fn in (("loaded matrix", g.query_device), ("loaded encoded", g.query_encoded_device)):
    out = fn(dk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out = fn(dk)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{enc} {name:15s} {ms:7.3f} ms  {n / ms / 1e6:8.2f} Gq/s")
