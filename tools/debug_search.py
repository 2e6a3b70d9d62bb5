import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np, torch
from oracle import oracle as orc
from test_gpu_stages import _search_inputs, _device_search
from paper_2404_18497_b200 import _native as nat
g = np.load("tests/golden/golden.npz"); meta = json.load(open("tests/golden/golden_meta.json"))
for name in meta["search_cases"]:
    m, hs, ls, key_off = _search_inputs(g, meta, orc, "srch", name)
    seeds, trials, status = _device_search(nat, orc, m, hs, ls, key_off, m["tie"] == "asc-expected")
    ws, wt = g[f"srch_{name}_seeds"], g[f"srch_{name}_trials"]
    bad = np.flatnonzero((seeds != ws).any(1) | (trials != wt).any(1))
    print(name, "nparts", len(key_off)-1, "bad partitions", bad[:10], "status", status.sum())
    if len(bad):
        j = bad[0]
        a, b = key_off[j], key_off[j+1]
        mm = b - a
        table = orc.tabulate("beta_eps", orc.default_epsilon(m["lambda"], m["P"]))
        B = orc.bucket_count(m["P"], m["lambda"])
        bid = orc.bucket_ids(hs[a:b], table, B)
        sizes = np.bincount(bid, minlength=B+1)
        tie = np.arange(B+1) if m["tie"] == "asc-expected" else B - np.arange(B+1)
        key = sizes * (B+1) + tie
        order = [bb for bb in np.argsort(-key) if sizes[bb] > 0]
        print(" m", mm, "B", B)
        for oi, bb in enumerate(order[:400]):
            if seeds[j, bb-1] != ws[j, bb-1] or trials[j, bb-1] != wt[j, bb-1]:
                print("  first diff at order", oi, "bucket", bb, "k", sizes[bb], "dev", seeds[j, bb-1], trials[j, bb-1], "ref", ws[j, bb-1], wt[j, bb-1])
                for oj in range(max(0, oi-3), min(len(order), oi+3)):
                    b2 = order[oj]
                    print("    ", oj, b2, sizes[b2], seeds[j, b2-1], trials[j, b2-1], ws[j, b2-1], wt[j, b2-1])
                break
