"""Secondary BASELINE configs (C1, C3 1B keys on one GPU, C4 lambda sweep, C5
strings): device build time, bits/key, query rate, bijection. Prints one JSON
line per config.

    python tools/sweep.py [--configs C1,C3,C4,C5] [--n3 1000000000] [--n4 100000000] [--n5 100000000]
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch

import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64_device
from paper_2404_18497_b200.mphf import BuildEngine


def timed_build(dk, cfg, reps=3):
    eng = BuildEngine(cfg)
    res = eng.run(dk, 0)  # warm-up
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        res = eng.run(dk, 0)
    e1.record()
    torch.cuda.synchronize()
    assert not isinstance(res, tuple), "build failed"
    return e0.elapsed_time(e1) / reps, res, eng


def query_rate(res, eng, cfg, dk):
    f = phb.Mphf._from_device(res, cfg, eng, None)
    out = f.query_device(dk)
    ok = f.verify_device(out)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        f.query_device(dk)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 3, ok


def report(name, n, cfg, ms, res, q_ms, ok, extra=None):
    line = {"config": name, "n": n, "lambda": cfg.lambda_, "encoder": cfg.encoder,
            "build_ms": round(ms, 3), "ns_per_key": ms * 1e6 / n,
            "keys_per_s": n / (ms * 1e-3), "bits_per_key": (res.total_bytes + 8 - 16) * 8 / n,
            "trials_per_key": res.trials_total / n,
            "query_ms": round(q_ms, 3), "query_Mq_s": n / (q_ms * 1e-3) / 1e6, "bijection": ok}
    if extra:
        line.update(extra)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C4,C5")
    ap.add_argument("--n3", type=int, default=1_000_000_000)
    ap.add_argument("--n4", type=int, default=100_000_000)
    ap.add_argument("--n5", type=int, default=100_000_000)
    a = ap.parse_args()
    cfgs = a.configs.split(",")
    dev = torch.device("cuda", 0)
    if "C1" in cfgs:
        n = 1_000_000
        keys = synth_u64_device(n, 0)
        dk = DeviceKeys(n, keys64=keys)
        cfg = phb.BuildConfig(lambda_=5.0, partition_size=2500.0, encoder="ic-c")
        ms, res, eng = timed_build(dk, cfg, reps=10)
        q, ok = query_rate(res, eng, cfg, dk)
        report("C1 1M u64 lambda=5 IC-C", n, cfg, ms, res, q, ok)
    if "C3" in cfgs:
        # BASELINE configs[2] is 1B keys over 2/4/8 GPUs; one B200 holds it whole
        # (keys 8 GB + build buffers ~20 GB), which is the G = 1 point of that sweep
        n = a.n3
        keys = synth_u64_device(n, 0)
        dk = DeviceKeys(n, keys64=keys)
        cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
        ms, res, eng = timed_build(dk, cfg, reps=2)
        q, ok = query_rate(res, eng, cfg, dk)
        report(f"C3 {n // 1_000_000}M u64 lambda=9 IC-C, 1 GPU", n, cfg, ms, res, q, ok)
        del keys, dk, res, eng
        torch.cuda.empty_cache()
    if "C4" in cfgs:
        n = a.n4
        keys = synth_u64_device(n, 0)
        dk = DeviceKeys(n, keys64=keys)
        for lam in (4.0, 5.0, 6.0, 7.0, 8.0, 9.0):
            cfg = phb.BuildConfig(lambda_=lam, partition_size=2500.0, encoder="ic-r")
            ms, res, eng = timed_build(dk, cfg)
            q, ok = query_rate(res, eng, cfg, dk)
            report(f"C4 {n // 1_000_000}M u64 lambda={lam:g} IC-R", n, cfg, ms, res, q, ok)
        del keys, dk
        torch.cuda.empty_cache()
    if "C5" in cfgs:
        n = a.n5
        g = torch.Generator(device=dev)
        g.manual_seed(2024)
        lens = torch.randint(10, 101, (n,), generator=g, device=dev, dtype=torch.int64)
        offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(lens, 0, out=offsets[1:])
        total = int(offsets[-1].item())
        buf = torch.randint(33, 127, (total,), generator=g, device=dev, dtype=torch.uint8)
        dk = DeviceKeys(n, buf=buf, offsets=offsets)
        cfg = phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r")
        ms, res, eng = timed_build(dk, cfg)
        q, ok = query_rate(res, eng, cfg, dk)
        report(f"C5 {n // 1_000_000}M strings 10-100 B, lambda=8 IC-R", n, cfg, ms, res, q, ok,
               {"mean_key_bytes": total / n, "key_bytes_total": total})


if __name__ == "__main__":
    main()
