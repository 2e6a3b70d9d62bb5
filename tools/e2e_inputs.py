import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import synth_u64_device
n = 100_000_000
cfg = phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c")
dev_keys = synth_u64_device(n, 0)
pinned = torch.empty(n, dtype=torch.int64, pin_memory=True); pinned.copy_(dev_keys)
npk = dev_keys.cpu().numpy().view(np.uint64)
pageable = torch.from_numpy(npk.view(np.int64))
torch.cuda.synchronize()
for name, k in (("pinned", pinned), ("numpy", npk), ("pageable_tensor", pageable)):
    ts = []
    for r in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        f = phb.build(k, cfg); torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    t = time.perf_counter(); d = torch.from_numpy(npk.view(np.int64)).to("cuda"); torch.cuda.synchronize(); h2d = time.perf_counter() - t
    print(name, [round(x*1e3,1) for x in ts], "pageable H2D alone", round(h2d*1e3,1))
