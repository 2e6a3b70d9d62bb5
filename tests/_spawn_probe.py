"""Launched by tests/test_bench_contract.py through bench.spawn_ranks: checks
the torchrun environment bench.py relies on (gloo, CPU)."""
import os
import sys

import torch.distributed as dist

assert sys.argv[1:] == ["--gpus", "2"], sys.argv
dist.init_process_group("gloo")
assert dist.get_world_size() == int(os.environ["WORLD_SIZE"]) == 2
dist.barrier()
print(f"probe ok world={dist.get_world_size()} rank={dist.get_rank()}", flush=True)
dist.destroy_process_group()
