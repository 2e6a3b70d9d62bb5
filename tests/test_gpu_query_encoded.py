"""K7e: queries answered straight from the encoded seed section (no decoded
matrix) equal the reference's queries (golden) and the matrix-based kernel,
for every preset, including Rice columns whose select spans many samples."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def phb():
    import paper_2404_18497_b200 as m
    from paper_2404_18497_b200 import _native

    _native.require_device()
    return m


def test_encoded_query_matches_reference_goldens(golden, meta, phb):
    """Structures deserialized from the reference's own bytes, queried from
    the encoded section, give the reference's query outputs."""
    from paper_2404_18497_b200 import KeyCorpus, Mphf

    checked = 0
    for key, m in meta.items():
        if not key.startswith("e2e_"):
            continue
        name = key[4:]
        if f"e2e_{name}_query" not in golden.files:
            continue
        corpus = KeyCorpus(golden[f"e2e_{name}_buf"], golden[f"e2e_{name}_off"])
        want = golden[f"e2e_{name}_query"]
        for enc in m["bytes"]:
            f = Mphf.deserialize(golden[f"e2e_{name}_{enc}"].tobytes())
            got = f.query_encoded_device(corpus).cpu().numpy()
            assert np.array_equal(got[: len(want)], want), (name, enc)
            checked += 1
    assert checked > 0


@pytest.mark.parametrize("enc", ["ic-c", "ic-r", "mixed:40", "mono-r", "mono-c"])
def test_encoded_query_equals_matrix_query(phb, enc):
    """P = 100 gives 3000 partitions, so every interleaved Rice column has
    more than one select sample (one per 1024 ones)."""
    rng = np.random.default_rng(11)
    keys = np.unique(rng.integers(0, 2**64, size=300_000, dtype=np.uint64))
    cfg = phb.BuildConfig(lambda_=5.0, partition_size=100.0, encoder=enc)
    f = phb.build(keys, cfg)
    assert f.num_partitions > 2048
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    a = f.query_device(dk)
    b = f.query_encoded_device(dk)
    assert torch.equal(a, b), enc
    assert f.verify_device(b)
    # the same through a deserialized copy (section uploaded from host bytes)
    g = phb.Mphf.deserialize(f.serialize())
    assert torch.equal(g.query_encoded_device(dk), a), enc


def test_encoded_query_string_keys(phb):
    from paper_2404_18497_b200 import gen_keys

    corpus = gen_keys(50_000, 3)
    f = phb.build(corpus, phb.BuildConfig(lambda_=8.0, partition_size=500.0, encoder="ic-r"))
    out = f.query_encoded_device(corpus)
    assert np.array_equal(out.cpu().numpy(), f.query_many(corpus))
    assert f.verify_device(out)


def test_encoded_query_c2_scale(phb):
    """100M keys of the bench workload (C2, IC-C): encoded-section queries are
    a bijection and agree with the matrix kernel on a sample."""
    from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64_device

    n = 100_000_000
    keys = synth_u64_device(n, 0)
    f = phb.build(DeviceKeys(n, keys64=keys),
                  phb.BuildConfig(lambda_=9.0, partition_size=2500.0, encoder="ic-c"))
    out = f.query_encoded_device(DeviceKeys(n, keys64=keys))
    assert f.verify_device(out)
    sample = keys[::997].contiguous()
    assert torch.equal(out[::997], f.query_device(DeviceKeys(sample.numel(), keys64=sample)))


def test_encoded_query_without_select_directory(phb):
    """phb_query_encoded with select_dir = NULL scans from the serialized
    every-1024th samples; same outputs as with the dense directory."""
    from paper_2404_18497_b200 import _native

    rng = np.random.default_rng(17)
    keys = np.unique(rng.integers(0, 2**64, size=200_000, dtype=np.uint64))
    f = phb.build(keys, phb.BuildConfig(lambda_=5.0, partition_size=300.0, encoder="mono-r"))
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    with_dir = f.query_encoded_device(dk)
    key_off, entries, _ = f._device_state(matrix=False)
    blob, info, num_enc, mono, dsel, _ = f.seeds.device_encoded()
    assert dsel is not None
    out = torch.empty_like(with_dir)
    P = _native.ptr
    _native.call("phb_query_encoded", None, None, P(dk), dk.numel(),
                 f.global_seed & 0xFFFFFFFFFFFFFFFF, f.n, f.num_partitions, P(key_off),
                 P(entries), f.bcount, P(blob), P(info), num_enc, mono, None, 1, P(out),
                 _native.stream())
    assert torch.equal(out, with_dir)
    assert torch.equal(with_dir, f.query_device(dk))


@pytest.mark.parametrize("enc", ["ic-c", "ic-r", "mixed:40"])
def test_large_batch_encoded_query_shared_tables(phb, enc):
    """Batches of >= 148 * 4096 u64 keys take the shared-memory matrix query
    (K7s) and, for all-Compact sections, the shared-memory encoded query
    (K7es: offsets, bucket pairs and column descriptors in shared memory);
    every path equals the global-table kernels on a sample and is a
    bijection."""
    from paper_2404_18497_b200.keygen import DeviceKeys, synth_u64_device

    n = 2_000_003  # odd: exercises the 4-key tail
    keys = synth_u64_device(n, 99)
    f = phb.build(DeviceKeys(n, keys64=keys),
                  phb.BuildConfig(lambda_=7.0, partition_size=2500.0, encoder=enc))
    big = f.query_encoded_device(DeviceKeys(n, keys64=keys))
    assert f.verify_device(big)
    assert torch.equal(big, f.query_device(DeviceKeys(n, keys64=keys)))
    sample = keys[::101].contiguous()  # small batch: the global-table kernels
    assert torch.equal(big[::101], f.query_encoded_device(DeviceKeys(sample.numel(), keys64=sample)))
