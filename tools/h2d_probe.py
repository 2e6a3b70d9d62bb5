"""H2D bandwidth of pinned host memory at the e2e size (800 MB): one stream
vs the copy split over 2 / 4 streams, chunked like to_device_chunked."""
import sys
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
host = torch.empty(n, dtype=torch.int64, pin_memory=True)
host.fill_(7)
dev = torch.empty(n, dtype=torch.int64, device="cuda")
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = 1 << 23
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        for i, a in enumerate(range(0, n, chunk)):
            b = min(a + chunk, n)
            with torch.cuda.stream(streams[i % nstreams]):
                dev[a:b].copy_(host[a:b], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"streams {nstreams} rep {rep}: {ms:.2f} ms  {n * 8 / ms / 1e6:.1f} GB/s")
