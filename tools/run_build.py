"""Run N device builds of synthetic u64 keys (for ncu captures)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import synth_u64_device, to_device
from paper_2404_18497_b200.mphf import BuildEngine
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--lam", type=float, default=9.0)
ap.add_argument("--enc", default="ic-c")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
keys = synth_u64_device(a.n, 12345)
eng = BuildEngine(phb.BuildConfig(lambda_=a.lam, partition_size=2500.0, encoder=a.enc))
dk = to_device(keys, keys.device)
for _ in range(a.reps):
    eng.run(dk, 0)
torch.cuda.synchronize()
print("ok")
