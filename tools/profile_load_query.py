import sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
import paper_2404_18497_b200 as phb
from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64_device
n = 1_000_000_000
keys = synth_u64_device(n, 0); dk = DeviceKeys(n, keys64=keys)
f = phb.build(dk, phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c"))
blob = f.serialize()
pr = cProfile.Profile(); pr.enable()
g = phb.Mphf.deserialize(blob)
out = g.query_device(dk); torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
