"""Probe: 2 ranks on one GPU with gloo over CUDA tensors (collectives used by distributed.py)."""
import os, sys, tempfile
import torch, torch.distributed as dist, torch.multiprocessing as mp

def run(rank, ws, path):
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=ws)
    d = torch.device("cuda", 0)
    x = torch.arange(4, dtype=torch.int64, device=d) + 10 * rank
    out = torch.empty(3 if rank == 0 else 5, dtype=torch.int64, device=d)
    ok = []
    try:
        dist.all_to_all_single(out, x, [1, 2] if rank == 0 else [3, 2], [1, 3] if rank == 0 else [2, 2]); ok.append("a2a")
    except Exception as e: ok.append(f"a2a FAIL {e}")
    try:
        lst = [torch.empty(3, dtype=torch.int32, device=d) for _ in range(ws)]
        dist.all_gather(lst, torch.ones(3, dtype=torch.int32, device=d)); ok.append("allgather")
    except Exception as e: ok.append(f"ag FAIL {e}")
    try:
        t = torch.ones(2, dtype=torch.int64, device=d); dist.all_reduce(t, op=dist.ReduceOp.MIN); ok.append("allreduce")
    except Exception as e: ok.append(f"ar FAIL {e}")
    print(rank, ok, out.tolist(), flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    mp.spawn(run, args=(2, tempfile.mktemp()), nprocs=2)
