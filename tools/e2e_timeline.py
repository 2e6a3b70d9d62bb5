"""Timeline of the end-to-end public-API build (pinned host keys -> Mphf):
CUDA events around every native call, relative to an event recorded before
phb.build(host); the H2D chunk copies run on a side stream in between."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import _native
from paper_2404_18497_b200.keygen import synth_u64_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
host = torch.empty(n, dtype=torch.int64, pin_memory=True)
host.copy_(synth_u64_device(n, 0))
torch.cuda.synchronize()
L = _native.lib()
marks = []
for name in [k for k in dir(L) if k.startswith("phb_")]:
    fn = getattr(L, name)
    if not callable(fn):
        continue

    def mk(fn, name):
        def w(*a):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn(*a)
            e1.record()
            marks.append((name, e0, e1, time.perf_counter()))
            return rc
        return w

    setattr(L, name, mk(fn, name))
for rep in range(3):
    marks.clear()
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s0.record()
    t0 = time.perf_counter()
    f = phb.build(host, cfg)
    s1 = torch.cuda.Event(enable_timing=True)
    s1.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    print(f"rep {rep}: wall {wall:.2f} ms, device {s0.elapsed_time(s1):.2f} ms")
    if rep == 2:
        agg = {}
        for name, e0, e1, th in marks:
            try:
                a, b = s0.elapsed_time(e0), s0.elapsed_time(e1)
            except RuntimeError:
                continue
            print(f"  {name:26s} start {a:8.3f}  end {b:8.3f}  dur {b - a:7.3f}  host {(th - t0) * 1e3:8.3f}")
