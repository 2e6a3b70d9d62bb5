"""Per-stage device timing for string keys (C5: 100M keys of 10-100 B, lambda=8 IC-R)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import _native
from paper_2404_18497_b200.keygen import DeviceKeys
from paper_2404_18497_b200.mphf import BuildEngine

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
eng = BuildEngine(phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r"))
L = _native.lib()
times = {}
for name in ["phb_hash_count", "phb_hash_count_store", "phb_layout", "phb_scatter", "phb_scatter_hashed", "phb_search", "phb_encode_plan",
             "phb_encode_write"]:
    fn = getattr(L, name)

    def make(fn, name):
        def wrapped(*a):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn(*a)
            e1.record()
            times.setdefault(name, []).append((e0, e1))
            return rc
        return wrapped

    setattr(L, name, make(fn, name))
for r in range(3):
    times.clear()
    res = eng.run(dk, 0)
    torch.cuda.synchronize()
    parts = {k: sum(a.elapsed_time(b) for a, b in v) for k, v in times.items()}
    print(f"rep {r}: " + "  ".join(f"{k[4:]}={v:.3f}ms" for k, v in parts.items()), flush=True)
bytes_per_pass = total + 8 * (n + 1)
print(f"key bytes {total / n:.1f} B/key; hash_count {bytes_per_pass / parts.get('phb_hash_count', parts.get('phb_hash_count_store')) / 1e6:.0f} GB/s,"
      f" scatter read {bytes_per_pass / parts.get('phb_scatter', parts.get('phb_scatter_hashed')) / 1e6:.0f} GB/s")
