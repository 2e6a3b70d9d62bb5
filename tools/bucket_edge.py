"""Bucket ids at the edges of the FP64 bucket function (xb near powers of two,
round-half-even ties of the u64 -> f64 conversion, t = 2048): device
(phb_bucket_ids) vs the oracle, on high words chosen through the inverse of
mix64 so that mix64(hi ^ BUCKET_SALT) hits each edge value exactly."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

M64 = (1 << 64) - 1
SALT = 0xC2B2AE3D27D4EB4F


def unxorshift(z, s):
    x = z
    for _ in range(64 // s + 1):
        x = z ^ (x >> s)
    return x & M64


def unmix64(z):
    z = unxorshift(z, 31)
    z = (z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M64
    z = unxorshift(z, 27)
    z = (z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M64
    return unxorshift(z, 30)


def mix64(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def edge_words():
    xs = set()
    for e in range(0, 64):
        for d in (-3, -2, -1, 0, 1, 2, 3):
            xs.add(((1 << e) + d) & M64)
    for e in range(53, 64):  # ties of the rounding to 53 bits: half an ulp above multiples
        ulp = 1 << (e - 52)
        for base in ((1 << e), (1 << e) + ulp, (1 << e) + 5 * ulp, M64 - 3 * ulp):
            for off in (ulp // 2 - 1, ulp // 2, ulp // 2 + 1, ulp - 1):
                xs.add((base + off) & M64)
    for k in range(0, 2049, 7):  # t = 2048 x near every table knot
        base = k << 53
        for d in (-2, -1, 0, 1, 2, 1 << 52, (1 << 52) - 1):
            xs.add((base + d) & M64)
    xs.add(M64)
    return sorted(xs)


def main():
    import torch

    from oracle import oracle
    from paper_2404_18497_b200 import _native

    his = np.array([unmix64(x) ^ SALT for x in edge_words()], np.uint64)
    assert all(mix64(int(h) ^ SALT) == x for h, x in zip(his[:50], edge_words()[:50]))
    bad = 0
    for lam, P in ((4.0, 2500.0), (9.0, 2500.0), (1.0, 300.0), (14.0, 3000.0)):
        table = oracle.tabulate("beta_eps", oracle.default_epsilon(lam, P))
        B = oracle.bucket_count(P, lam)
        want = oracle.bucket_ids(his, table, B)
        h = torch.from_numpy(his.view(np.int64)).cuda()
        e = torch.from_numpy(np.ascontiguousarray(table)).cuda()
        out = torch.empty(len(his), dtype=torch.int16, device="cuda")
        _native.call("phb_bucket_ids", _native.ptr(h), len(his), _native.ptr(e), B,
                     _native.ptr(out), _native.stream())
        got = out.cpu().numpy().view(np.uint16).astype(np.int64)
        bad += int((got != want).sum())
    print(f"{len(his)} edge words x 4 tables: {bad} mismatches")
    return bad


if __name__ == "__main__":
    sys.exit(1 if main() else 0)
