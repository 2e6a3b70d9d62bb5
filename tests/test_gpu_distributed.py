"""GPU side of the sharded build: the regroup kernel against a numpy
restatement, and the full NCCL orchestration at world size 1 (the only
size one GPU allows) against the single-GPU build."""

import os
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_regroup_kernel_matches_numpy():
    from paper_2404_18497_b200 import _native

    rng = np.random.default_rng(4)
    for G, np_g in [(1, 5), (3, 17), (8, 400), (2, 0), (5, 1)]:
        C = rng.integers(0, 40, size=(G, np_g)).astype(np.int32)
        recv = C.sum(1)
        total = int(recv.sum())
        lo = rng.integers(0, 2**63, size=total, dtype=np.int64)
        aux = rng.integers(0, 2**15, size=total).astype(np.int16)
        starts = np.concatenate([[0], np.cumsum(recv)])
        want_lo, want_aux = [], []
        for j in range(np_g):
            for s in range(G):
                a = starts[s] + C[s, :j].sum()
                want_lo.append(lo[a:a + C[s, j]])
                want_aux.append(aux[a:a + C[s, j]])
        d_lo = torch.from_numpy(lo).cuda()
        d_aux = torch.from_numpy(aux).cuda()
        d_C = torch.from_numpy(C).cuda()
        o_lo = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
        o_aux = torch.empty(max(total, 1), dtype=torch.int16, device="cuda")
        koff = torch.empty(np_g + 1, dtype=torch.int64, device="cuda")
        _native.call("phb_regroup", _native.ptr(d_lo), _native.ptr(d_aux), _native.ptr(d_C), G,
                     np_g, _native.ptr(o_lo), _native.ptr(o_aux), _native.ptr(koff),
                     _native.stream())
        if total:
            assert np.array_equal(o_lo.cpu().numpy()[:total], np.concatenate(want_lo))
            assert np.array_equal(o_aux.cpu().numpy()[:total], np.concatenate(want_aux))
        want_off = np.zeros(np_g + 1, np.int64)
        np.cumsum(C.sum(0), out=want_off[1:])
        assert np.array_equal(koff.cpu().numpy(), want_off)


def test_nccl_world1_equals_single_gpu_build():
    import torch.distributed as dist

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200.distributed import build_distributed
    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(250_000, 3)
    cfg = phb.BuildConfig(lambda_=8.0, partition_size=2500.0, encoder="ic-r")
    path = os.path.join(tempfile.mkdtemp(), "rdv")
    dist.init_process_group("nccl", init_method=f"file://{path}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        f = build_distributed(keys, cfg)
    finally:
        dist.destroy_process_group()
    g = phb.build(keys, cfg)
    assert f.serialize() == g.serialize()
    assert f.stats.trials_total == g.stats.trials_total
    assert f.is_bijection_on(keys)
