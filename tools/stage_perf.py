"""Per-stage device timing of one build pass (CUDA events on the current stream)."""
import argparse
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import _native
from paper_2404_18497_b200.keygen import synth_u64_device, to_device
from paper_2404_18497_b200.mphf import BuildEngine

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--lam", type=float, default=9.0)
ap.add_argument("--enc", default="ic-c")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

keys = synth_u64_device(a.n, 12345)
cfg = phb.BuildConfig(lambda_=a.lam, partition_size=2500.0, encoder=a.enc)
eng = BuildEngine(cfg)
dk = to_device(keys, keys.device)
# instrument by wrapping the native calls with events
L = _native.lib()
times = {}
orig = {}
for name in ["phb_hash_count", "phb_layout", "phb_scatter", "phb_search", "phb_encode_plan",
             "phb_encode_write"]:
    fn = getattr(L, name)
    orig[name] = fn

    def make(fn, name):
        def wrapped(*args):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = fn(*args)
            e1.record()
            times.setdefault(name, []).append((e0, e1))
            return rc
        return wrapped

    setattr(L, name, make(fn, name))
for r in range(a.reps):
    times.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = eng.run(dk, 0)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    parts = {k: sum(e0.elapsed_time(e1) for e0, e1 in v) for k, v in times.items()}
    print(f"rep {r}: wall {wall*1e3:.2f} ms  ({wall*1e9/a.n:.3f} ns/key)  " +
          "  ".join(f"{k[4:]}={v:.3f}ms" for k, v in parts.items()), flush=True)
print("bits/key", (res.total_bytes + 8 - 16) * 8 / a.n, "trials/key", res.trials_total / a.n)
