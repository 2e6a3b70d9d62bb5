"""A/B timing of library variants (each a .so built by tools/build_variants.sh).

  python tools/variant_bench.py base=_variants/base.so new=paper_2404_18497_b200/libphobic_b200.so \
      [--n 100000000] [--lams 9,5] [--reps 5]

Each variant runs in its own process (PHB_LIB selects the library). Per
lambda it reports the median search-kernel time (CUDA events around
phb_search), the median build-pass time, and a digest of the encoded body +
trials, which must agree across variants (a variant that changes a seed is
wrong, whatever its speed).
"""
import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def child(n, lams, reps):
    sys.path.insert(0, str(ROOT))
    import torch

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200 import _native
    from paper_2404_18497_b200.keygen import synth_u64_device, to_device
    from paper_2404_18497_b200.mphf import BuildEngine

    keys = synth_u64_device(n, 0)
    dk = to_device(keys, keys.device)
    L = _native.lib()
    fn = L.phb_search
    ev = []

    def wrapped(*a):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = fn(*a)
        e1.record()
        ev.append((e0, e1))
        return rc

    L.phb_search = wrapped
    out = {}
    for lam in lams:
        enc = "ic-c"
        eng = BuildEngine(phb.BuildConfig(lambda_=lam, partition_size=2500.0, encoder=enc))
        res = eng.run(dk, 0)
        torch.cuda.synchronize()
        s_ms, b_ms = [], []
        for _ in range(reps):
            ev.clear()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            res = eng.run(dk, 0)
            t1.record()
            torch.cuda.synchronize()
            b_ms.append(t0.elapsed_time(t1))
            s_ms.append(sum(a.elapsed_time(b) for a, b in ev))
        h = hashlib.sha256(res.blob[: res.total_bytes].cpu().numpy().tobytes())
        h.update(str(res.trials_total).encode())
        out[str(lam)] = {"search_ms": statistics.median(s_ms), "build_ms": statistics.median(b_ms),
                         "digest": h.hexdigest()[:16], "trials_per_key": res.trials_total / n}
    print("RESULT " + json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("variants", nargs="*")
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--lams", default="9,5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    lams = [float(x) for x in a.lams.split(",")]
    if a.child:
        child(a.n, lams, a.reps)
        return
    results = {}
    for v in a.variants:
        name, path = v.split("=", 1)
        env = dict(os.environ, PHB_LIB=str(Path(path).resolve()))
        r = subprocess.run([sys.executable, __file__, "--child", "--n", str(a.n), "--lams", a.lams,
                            "--reps", str(a.reps)], env=env, capture_output=True, text=True)
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")]
        if r.returncode != 0 or not line:
            print(f"{name}: FAILED rc={r.returncode}\n{r.stderr[-2000:]}", flush=True)
            continue
        results[name] = json.loads(line[0][7:])
        for lam, d in results[name].items():
            print(f"{name:14s} lambda={lam:4s} search {d['search_ms']:8.3f} ms  build {d['build_ms']:8.3f} ms"
                  f"  digest {d['digest']}  trials/key {d['trials_per_key']:.1f}", flush=True)
    digests = {lam: {r[lam]["digest"] for r in results.values()} for lam in map(str, lams)}
    for lam, ds in digests.items():
        print(f"lambda={lam}: {'all variants agree' if len(ds) == 1 else 'DIGEST MISMATCH ' + str(ds)}")


if __name__ == "__main__":
    main()
