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


def _dev_worker(rank, world, path, keys, cfg_kw, out_path, transport="nccl", encode="sharded"):
    import torch.distributed as dist

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200.distributed import build_distributed

    torch.cuda.set_device(0)  # every rank shares the one GPU; gloo carries CUDA tensors
    dist.init_process_group("gloo", init_method=f"file://{path}", rank=rank, world_size=world)
    try:
        shards = np.array_split(keys, world)
        f = build_distributed(shards[rank], phb.BuildConfig(**cfg_kw), transport=transport,
                              encode=encode)
        out = f.query_device(shards[rank])
        ok = bool(((out >= 0) & (out < f.n)).all()) and out.unique().numel() == out.numel()
        outs = [torch.empty(len(s), dtype=torch.int64, device="cuda") for s in shards]
        dist.all_gather(outs, out)
        allout = torch.cat(outs)
        ok = ok and allout.unique().numel() == f.n
        np.save(out_path + f".{rank}.npy", np.frombuffer(f.serialize(), np.uint8))
        np.save(out_path + f".{rank}.ok.npy", np.array([ok, f.stats.trials_total]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 3])
def test_device_sharded_build_gloo_on_one_gpu(world, transport):
    """The DeviceOps path (K1/K3 per shard, all-to-all + phb_regroup or the
    fused CUDA-IPC peer scatter, K4 on owned partitions, sharded K5)
    with `world` ranks sharing one GPU over gloo: every rank's bytes equal
    the single-GPU build."""
    import torch.multiprocessing as mp

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(300_000, 11)
    cfg_kw = dict(lambda_=7.0, partition_size=2500.0, encoder="ic-r")
    d = tempfile.mkdtemp()
    out = os.path.join(d, "blob")
    mp.spawn(_dev_worker, args=(world, os.path.join(d, "rdv"), keys, cfg_kw, out, transport),
             nprocs=world)
    want = phb.build(keys, phb.BuildConfig(**cfg_kw))
    for r in range(world):
        assert np.load(out + f".{r}.npy").tobytes() == want.serialize()
        ok, trials = np.load(out + f".{r}.ok.npy")
        assert ok and trials == want.stats.trials_total


@pytest.mark.parametrize("encoder,encode", [("mono-r", "sharded"), ("ic-c", "sharded"),
                                            ("mixed:100", "sharded"), ("ic-r", "gather")])
def test_sharded_encode_every_preset(encoder, encode):
    """Sharded K5 (column stats all_reduce, per-rank fields at global bit
    addresses, OR of the bodies) for every preset at world 3: mono-r's one
    column spans all ranks, so Rice select samples and unary runs cross
    shard boundaries; "gather" is the all_gather + replicated encode."""
    import torch.multiprocessing as mp

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(300_000, 13)
    cfg_kw = dict(lambda_=7.0, partition_size=2500.0, encoder=encoder)
    d = tempfile.mkdtemp()
    out = os.path.join(d, "blob")
    world = 3
    mp.spawn(_dev_worker, args=(world, os.path.join(d, "rdv"), keys, cfg_kw, out, "nccl", encode),
             nprocs=world)
    want = phb.build(keys, phb.BuildConfig(**cfg_kw))
    for r in range(world):
        assert np.load(out + f".{r}.npy").tobytes() == want.serialize(), (encoder, r)


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_sharded_build_rank_without_partitions(transport):
    """2 partitions over 3 ranks: the last rank owns no partition (empty
    search, empty encode shard) and still returns the identical structure."""
    import torch.multiprocessing as mp

    import paper_2404_18497_b200 as phb
    from paper_2404_18497_b200.keygen import synth_u64

    keys = synth_u64(999, 21)  # equal shards (the harness all_gathers query outputs)
    cfg_kw = dict(lambda_=4.0, partition_size=500.0, encoder="ic-r")
    d = tempfile.mkdtemp()
    out = os.path.join(d, "blob")
    mp.spawn(_dev_worker, args=(3, os.path.join(d, "rdv"), keys, cfg_kw, out, transport),
             nprocs=3)
    want = phb.build(keys, phb.BuildConfig(**cfg_kw))
    for r in range(3):
        assert np.load(out + f".{r}.npy").tobytes() == want.serialize(), r
