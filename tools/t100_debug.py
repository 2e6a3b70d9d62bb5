import sys, time
sys.path.insert(0, "/root/repo")
import torch, paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import synth_u64_device
t=time.time()
def lap(msg):
    global t
    torch.cuda.synchronize(); print(f"{msg}: {time.time()-t:.2f}s", flush=True); t=time.time()
n = 100_000_000
keys = synth_u64_device(n, 0)
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
f = phb.build(keys, cfg); lap("build")
print(f.is_bijection_on(keys)); lap("bij")
perm = torch.randperm(n, device=keys.device); lap("perm")
g = phb.build(keys[perm], cfg); lap("build2")
print(f._body.tobytes() == g._body.tobytes()); lap("cmp")
data = f.serialize(); lap("serialize")
h = phb.Mphf.deserialize(data); lap("deserialize")
st = h._device_state(); lap("device_state")
sample = keys[:5_000_000]
print(torch.equal(h.query_device(sample), f.query_device(sample))); lap("query")
