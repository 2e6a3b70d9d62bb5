"""Host-side format costs at scale: serialize (body D2H already done by build,
blake2b, concatenation), deserialize (checksum, parse, validation), and the
first query of a loaded structure (device decode + query). C2 / C3 sizes."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64_device

for n in [int(x) for x in (sys.argv[1:] or ["100000000", "1000000000"])]:
    keys = synth_u64_device(n, 0)
    dk = DeviceKeys(n, keys64=keys)
    cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
    t = time.perf_counter(); f = phb.build(dk, cfg); torch.cuda.synchronize(); tb = time.perf_counter() - t
    t = time.perf_counter(); blob = f.serialize(); ts = time.perf_counter() - t
    t = time.perf_counter(); g = phb.Mphf.deserialize(blob); td = time.perf_counter() - t
    t = time.perf_counter(); out = g.query_device(dk); torch.cuda.synchronize(); tq = time.perf_counter() - t
    t = time.perf_counter(); oute = g.query_encoded_device(dk); torch.cuda.synchronize(); tqe = time.perf_counter() - t
    ok = g.verify_device(out) and torch.equal(out, oute)
    print(f"n={n:,} bytes={len(blob):,} build {tb*1e3:.1f} ms serialize {ts*1e3:.1f} ms "
          f"deserialize {td*1e3:.1f} ms first query (decode+query) {tq*1e3:.1f} ms "
          f"first encoded query {tqe*1e3:.1f} ms bijection {ok}", flush=True)
    del keys, dk, f, g, out, oute
    torch.cuda.empty_cache()
