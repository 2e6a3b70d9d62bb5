"""Time K3 (phb_scatter) alone at C2 size: keys -> counts -> layout -> scatter x reps."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import _native
from paper_2404_18497_b200.builder import device_table
from paper_2404_18497_b200.assignment import tabulate
from paper_2404_18497_b200.keygen import synth_u64_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
RECORDS = "--arrays" not in sys.argv  # default: the build's 16-byte record layout
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
dev = torch.device("cuda", 0)
keys = synth_u64_device(n, 0)
nparts = max(1, round(n / 2500.0))
B = cfg.bucket_count
L = _native.lib(); P = _native.ptr; st = _native.stream()
entries = device_table(tabulate(cfg.resolved_assignment()), dev)
counts = torch.zeros(nparts, dtype=torch.int32, device=dev)
_native.check(L.phb_hash_count(None, None, P(keys), n, 0, nparts, P(counts), st), "hc")
key_off = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
deltas = torch.empty(nparts + 1, dtype=torch.int64, device=dev)
stats = torch.empty(2, dtype=torch.int64, device=dev)
_native.check(L.phb_layout(P(counts), nparts, 0, 0, n, nparts, P(key_off), P(deltas), P(stats), st), "l")
cur = torch.empty(nparts * 32, dtype=torch.int32, device=dev)  # room for strided-cursor variants
lo = torch.empty(2 * n, dtype=torch.int64, device=dev)  # room for 16-byte record variants
bid = torch.empty(n, dtype=torch.int16, device=dev)
ts = []
for r in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.check(L.phb_scatter(None, None, P(keys), n, 0, nparts, P(entries), B, P(key_off),
                                P(cur), P(lo), None if RECORDS else P(bid), st), "sc")
    e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("scatter ms", [round(t, 3) for t in ts])
