"""Break down the end-to-end public-API build (pinned host keys -> Mphf)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200 import mphf as M
from paper_2404_18497_b200.keygen import synth_u64_device, to_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
host = torch.empty(n, dtype=torch.int64, pin_memory=True)
host.copy_(synth_u64_device(n, 0))
torch.cuda.synchronize()
for rep in range(3):
    T = {}
    t0 = time.perf_counter()
    dk = to_device(host, torch.device("cuda")); torch.cuda.synchronize(); T["h2d"] = time.perf_counter() - t0
    t1 = time.perf_counter(); eng = M.BuildEngine(cfg); T["engine"] = time.perf_counter() - t1
    t1 = time.perf_counter(); res = eng.run(dk, 0); torch.cuda.synchronize(); T["run"] = time.perf_counter() - t1
    t1 = time.perf_counter()
    blob = res.blob[: res.total_bytes].cpu(); T["d2h"] = time.perf_counter() - t1
    t1 = time.perf_counter(); f = M.Mphf._from_device(res, cfg, eng, None); T["from_device"] = time.perf_counter() - t1
    t1 = time.perf_counter(); f2 = phb.build(host, cfg); torch.cuda.synchronize(); T["build_api"] = time.perf_counter() - t1
    t1 = time.perf_counter(); data = f2.serialize(); T["serialize"] = time.perf_counter() - t1
    print(rep, {k: round(v * 1e3, 2) for k, v in T.items()}, len(data))
