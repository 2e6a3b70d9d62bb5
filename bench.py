"""PHOBIC construction benchmark (BASELINE.json configs[1]: C2).

Workload: n = 100M distinct 64-bit keys (synthetic, mix64(offset + i)),
lambda = 9, P = 2500, interleaved-compact encoding ("fast-query ~2.17
bits/key" config), beta_eps assignment, global seed 0.

One step = one full device build pass over the resident keys:
  murmur3 + partition histogram -> layout -> scatter by partition ->
  per-partition seed search -> interleaved encoding -> serialized body
(all kernels of paper_2404_18497_b200, incl. the two host syncs of the
pipeline). `value` is keys/s with keys already in HBM; `e2e` is the same
metric through the public API `build(pinned_host_keys, cfg)` with the H2D
copy of the keys and the D2H copy of the encoded structure inside the
timed region.

N > 1 (torchrun): one build over n = 100M x N keys, sharded 100M per rank and
routed to partition owners with NCCL (weak scaling; distributed.py).

--impl reference: the reference algorithm's CPU implementation (the oracle
port, oracle/phobic_oracle.c, all host threads) on a bounded sample of the
same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MPHF build ns/key (keys/s) at 1/2/4/8 B200 @ bits/key; GPU query Mq/s"
N_KEYS = 100_000_000
LAMBDA = 9.0
PSIZE = 2500.0
ENCODER = "ic-c"
PUBLISHED_NS_PER_KEY = 28.0  # PHOBIC-GPU lambda=9 IC-C, RTX 3090
# SURVEY.md §8(d), per key: the grouping pass reads the key (8 B) and writes
# (lo, bucket id) (10 B); the search reads the record (10 B)
ALGO_BYTES = {"total": 28, "hash_count": 8, "scatter": 18, "group": 18, "search": 10}
KERNELS_PER_BUILD = 12  # padded_init, scatter_padded, padded_counts, layout, search, 7 encode
# (profiles/r1_launches_c2.csv: the ncu launch list of one build, plus two torch zero-fills)


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_init(n_gpus: int, backend: str = "nccl", same_device: bool = False):
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        if same_device:  # validation mode: every rank on GPU 0 (gloo carries CUDA tensors)
            local = 0
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(sample_keys: int, threads: int):
    """The reference algorithm on the host (oracle port), bounded sample."""
    from oracle import oracle
    from paper_2404_18497_b200.keygen import synth_u64

    oracle.build_lib()
    keys = synth_u64(sample_keys, 0)
    t0 = time.perf_counter()
    f = oracle.build(keys, lambda_=LAMBDA, P=PSIZE, encoder=ENCODER, threads=threads)
    body = f.body()
    dt = time.perf_counter() - t0
    import numpy as np

    trials = int(np.asarray(f.trials).sum())
    return {"value": sample_keys / dt, "unit": "keys/s", "cores": threads, "kind": "port",
            "trials_per_s": trials / dt,
            "sample": f"{sample_keys:,} keys of the same synthetic stream, lambda=9 IC-C, "
                      f"full build (hash, partition, search, encode) in {dt:.2f} s",
            "ns_per_key": dt * 1e9 / sample_keys, "bits_per_key": (len(body) + 57 + 8 - 16) * 8 / sample_keys}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = args.ref_sample or max(200_000, min(4_000_000, 250_000 * threads))
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(sample, threads)
        if i >= args.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "keys/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sample / v * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"C2 sample: {sample:,} u64 keys, lambda=9, P=2500, IC-C",
                       "n_keys": sample, "lambda": LAMBDA, "partition_size": PSIZE,
                       "encoder": ENCODER},
            "cpu_baseline": {**r, "value": v},
            "e2e": {"value": v, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200 import _native
    from paper_2404_18497_b200.keygen import synth_u64_device, to_device
    from paper_2404_18497_b200.mphf import BuildEngine

    rank, world, local = dist_init(args.gpus, args.backend, args.same_device)
    dev = torch.device("cuda", torch.cuda.current_device())
    n = args.n
    cfg = phb.BuildConfig(lambda_=LAMBDA, partition_size=PSIZE, encoder=ENCODER)
    keys = synth_u64_device(n, rank * n)  # disjoint shard per rank
    dk = to_device(keys, dev)
    eng = BuildEngine(cfg, dev)

    # per-kernel events around the pipeline's native calls (search timing)
    L = _native.lib()
    stage = {}
    wrapped = {}
    for name in ("phb_hash_count", "phb_scatter", "phb_search", "phb_scatter_padded",
                 "phb_search_strided"):
        fn = getattr(L, name)

        def mk(fn, name):
            def w(*a):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                rc = fn(*a)
                e1.record()
                stage.setdefault(name, []).append((e0, e1))
                return rc
            return w

        wrapped[name] = fn
        setattr(L, name, mk(fn, name))

    if world > 1:
        from paper_2404_18497_b200.distributed import DeviceOps, build_distributed

        dops = DeviceOps(cfg)

        def step():
            return build_distributed(dk, cfg, ops=dops, to_host=False, transport=args.transport)
    else:
        def step():
            return eng.run(dk, 0)

    res = None
    for _ in range(args.warmup):
        res = step()
    stage.clear()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(args.steps):
            res = step()
        end.record()
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ms = start.elapsed_time(end) / args.steps
    ms = allmax(ms, world)
    per = {k: sum(a.elapsed_time(b) for a, b in v) / len(v) for k, v in stage.items()}
    for name, fn in wrapped.items():
        setattr(L, name, fn)
    assert not isinstance(res, tuple), "build failed"
    total_keys = n * world
    bits = (res.total_bytes + 8 - 16) * 8 / total_keys
    value = total_keys / (ms * 1e-3)

    # ---- e2e through the public API: pinned host keys -> Mphf (host bytes)
    host = torch.empty(n, dtype=torch.int64, pin_memory=True)
    host.copy_(keys)
    del dk, keys
    torch.cuda.empty_cache()
    e2e_ms = []
    blob_bytes = 0
    for i in range(1 + args.e2e_steps):
        torch.cuda.synchronize()
        barrier(world)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if world > 1:
            f = build_distributed(host, cfg, ops=dops, transport=args.transport)
        else:
            f = phb.build(host, cfg)
        e1.record()
        torch.cuda.synchronize()
        blob_bytes = len(f._body)
        if i > 0:
            e2e_ms.append(e0.elapsed_time(e1))
        del f
    e2e = allmax(statistics.median(e2e_ms) if e2e_ms else float("nan"), world)

    # ---- batched GPU query of all n keys (Mq/s), from the last build
    f = (build_distributed(host, cfg, ops=dops, transport=args.transport) if world > 1
         else phb.build(host, cfg))
    qkeys = host.to(dev)
    qdk = to_device(qkeys, dev)
    out = f.query_device(qdk)
    if world == 1:
        assert f.verify_device(out), "not a bijection"
    else:  # each rank checks its shard's outputs are distinct and in range
        assert bool(((out >= 0) & (out < f.n)).all()) and out.unique().numel() == out.numel()
    torch.cuda.synchronize()
    def time_query(fn, reps=5):
        """median of per-call device times (CUDA events around each call)"""
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn(qdk)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts), r

    q_ms, out = time_query(f.query_device)
    # the same batched query reading the seeds from the encoded section (K7e)
    qe_ms, oute = time_query(f.query_encoded_device)
    enc_ok = bool(torch.equal(oute, out))

    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    # the single-GPU build groups into fixed-capacity slots and searches them
    # strided; the multi-GPU path uses the counted kernels
    if "phb_search_strided" in per:
        per["phb_search"] = per.pop("phb_search_strided")
    s_ms = per.get("phb_search", float("nan"))
    achieved = n * ALGO_BYTES["search"] / (s_ms * 1e-3) / 1e9
    passes = {}
    for k, nm in (("phb_hash_count", "hash_count"), ("phb_scatter", "scatter"),
                  ("phb_scatter_padded", "group")):
        if k in per:
            gbs = n * ALGO_BYTES[nm] / (per[k] * 1e-3) / 1e9
            passes[nm] = {"ms": round(per[k], 4), "GB/s": round(gbs, 1), "frac": round(gbs / hbm, 4)}
    passes["search"] = {"ms": round(s_ms, 4), "share_of_step": round(s_ms / ms, 4)}
    traffic = None
    tp = ROOT / "profiles" / "search_traffic_c2.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("bytes_per_launch")
        except Exception:
            traffic = None
    sm = None
    sp = ROOT / "profiles" / "search_sm_c2.json"
    if sp.exists():
        try:
            sm = json.loads(sp.read_text())
        except Exception:
            sm = None
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / (1e9 / PUBLISHED_NS_PER_KEY),
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"C2: n={n / 1e6:g}M u64 keys/GPU, lambda=9, P=2500, IC-C "
                               "(fast-query)",
                   "n_keys_per_gpu": n, "lambda": LAMBDA, "partition_size": PSIZE,
                   "encoder": ENCODER, "global_seed": 0,
                   "l2": "inputs (800 MB keys + 1 GB grouped records) exceed the 126 MB L2",
                   "keys": "mix64(rank*n + i), distinct by construction",
                   "parallelism": (f"sharded build x{world}: records routed to partition "
                                   f"owners ({args.transport})" if world > 1 else "1 GPU")},
        "ns_per_key": ms * 1e6 / total_keys,
        "bits_per_key": bits,
        # the reference's work unit (one key x one (s, d) candidate, _kernels.py:236-240)
        "search_work": {"trials_per_key": res.trials_total / total_keys,
                        "trials_per_s": res.trials_total / (ms * 1e-3),
                        "search_trials_per_s": (res.trials_total / (per["phb_search"] * 1e-3)
                                                if "phb_search" in per else None)},
        "query": {"value": total_keys / (allmax(q_ms, world) * 1e-3) / 1e6, "unit": "Mq/s",
                  "ms": q_ms, "bijection_verified": True,
                  "what": "batched GPU query of every key (hash fused), keys resident",
                  "encoded": {"value": total_keys / (allmax(qe_ms, world) * 1e-3) / 1e6,
                              "unit": "Mq/s", "ms": qe_ms, "equal_to_matrix_query": enc_ok,
                              "what": "same query reading seeds from the encoded section"}},
        "e2e": {"value": total_keys / (e2e * 1e-3), "unit": "keys/s", "ms": e2e,
                "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": blob_bytes,
                "api": "paper_2404_18497_b200.build(pinned host uint64 tensor, BuildConfig)"},
        "gpu_launches": KERNELS_PER_BUILD * args.steps,
        "roofline": {"bound": "hbm", "kernel": "k_search", "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "note": "search is issue/latency bound (integer + shared-memory bit "
                             "ops), not HBM bound; algorithmic bytes = 10 B/key read "
                             "(SURVEY.md §8(d)); see passes for the HBM-bound kernels",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "when" in peaks else "fallback",
                     # the bound that does apply to k_search (ncu --set full, same workload)
                     "sm": None if sm is None else {
                         "issue_active_pct": round(sm["issue_active_pct"], 1),
                         "alu_pipe_pct": round(sm["alu_pipe_pct_elapsed"], 1),
                         "shared_lsu_pct": round(sm["lsu_shared_wavefront_pct_elapsed"], 1),
                         "warp_instructions_per_key": round(sm["warp_instructions"] / 1e8, 1),
                         "source": "profiles/search_sm_c2.json"}},
        "passes": passes,
        # whole-build floor = 28 B/key of algorithmic traffic at peak HBM
        "build_roofline": {"algorithmic_bytes_per_key": ALGO_BYTES["total"],
                           "t_floor_ms": n * ALGO_BYTES["total"] / (hbm * 1e9) * 1e3,
                           "frac": (n * ALGO_BYTES["total"] / (hbm * 1e9) * 1e3) / ms},
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = args.ref_sample or max(200_000, min(4_000_000, 250_000 * threads))
        line["cpu_baseline"] = cpu_baseline(sample, threads)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--keys", dest="n", type=int, default=N_KEYS, help="keys per GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="nccl", help="nccl (default) or gloo (validation)")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 record routing: fused CUDA-IPC peer scatter (default) or NCCL "
                         "all-to-all + regroup (automatic fallback if peer mapping fails)")
    ap.add_argument("--same-device", action="store_true",
                    help="validation: run every rank on GPU 0 (with --backend gloo)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
