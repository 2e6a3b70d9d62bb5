"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the host-side config / format logic matches the reference, and the product
path refuses to run without a GPU (no CPU fallback)."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "phobic.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(phb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2404_18497_b200 import _native

    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert lib.phb_version().startswith(b"phobic-b200")
    assert lib.phb_error_string(1003) == b"invalid arguments"


def test_ctypes_signatures_cover_the_header():
    from paper_2404_18497_b200 import _native

    bound = set(_native.SIGNATURES) | set(_native.OTHER)
    assert set(declared_symbols()) <= bound


def test_shared_library_is_sm100a():
    import subprocess

    from paper_2404_18497_b200 import _native

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2404_18497_b200 as phb

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        phb.build([b"a", b"b"], phb.BuildConfig())


# ---- host config logic vs the reference's frozen values (pkg/tests) ----

def test_empty_input_rejected_before_the_device():
    """build([]) raises InvalidConfig like the reference (mphf.py:243-245,
    test_mphf.py:139-144), from host logic alone."""
    import paper_2404_18497_b200 as phb

    for empty in ([], np.zeros(0, np.uint64), phb.KeyCorpus.from_keys([])):
        with pytest.raises(phb.InvalidConfig):
            phb.build(empty, phb.BuildConfig())


def test_build_config_validation():
    from paper_2404_18497_b200 import BuildConfig, InvalidConfig
    from paper_2404_18497_b200.builder import parse_encoder

    with pytest.raises(InvalidConfig):
        BuildConfig(lambda_=0.0)
    with pytest.raises(InvalidConfig):
        BuildConfig(partition_size=0.5)
    with pytest.raises(InvalidConfig):
        BuildConfig(seed_cap=100, partition_size=2500.0)
    with pytest.raises(InvalidConfig):
        BuildConfig(encoder="zip")
    with pytest.raises(InvalidConfig):
        BuildConfig(tie_break="sideways")
    assert parse_encoder("mixed:12") == ("mixed", 12)
    assert parse_encoder("ic-r") == ("ic-r", None)
    assert BuildConfig().tie_desc == 1 and BuildConfig(tie_break="desc-expected").tie_desc == 0
    assert BuildConfig(lambda_=8.0).bucket_count == 312
    assert BuildConfig(lambda_=9.0, encoder="ic-c").compact_prefix() == (0, 278)
    assert BuildConfig(encoder="mixed:400").compact_prefix() == (0, 312)
    assert BuildConfig(encoder="mono-c").compact_prefix() == (1, 1)


def test_assignment_known_answers():
    from paper_2404_18497_b200.assignment import (AssignmentSpec, beta_eps, beta_star,
                                                  bucket_count, bucket_for_hash, default_epsilon,
                                                  eval_table, tabulate)

    assert beta_star(0.5) == pytest.approx(0.15342640972002735, abs=1e-15)
    assert beta_eps(0.5, 0.032) == pytest.approx(0.16451676460898647, abs=1e-15)
    assert default_epsilon(8.0, 2500.0) == pytest.approx(0.032, abs=1e-15)
    assert default_epsilon(1e9, 1.0) == 0.99
    assert bucket_count(2500.0, 8.0) == 312 and bucket_count(2500.0, 4.0) == 625
    t = tabulate(AssignmentSpec("beta_eps", 0.032))
    assert eval_table(t, 3 / 4096) == pytest.approx(2.3726071037234354e-05, rel=1e-12)
    assert bucket_for_hash(t, 0.5, 312) == 52
    with pytest.raises(ValueError):
        AssignmentSpec("nope")
    assert AssignmentSpec("beta-eps", 0.01).kind == "beta_eps"


def test_tables_bit_identical_to_reference(golden, meta):
    from paper_2404_18497_b200.assignment import AssignmentSpec, tabulate

    for name, (kind, eps, _B) in meta["bucket_specs"].items():
        assert np.array_equal(tabulate(AssignmentSpec(kind, eps)).entries, golden[f"tab_{name}"])


def test_partition_counts_and_offsets():
    from paper_2404_18497_b200.partitioning import (PartitionLayout, expected_offset,
                                                    num_partitions_for, offset)

    assert num_partitions_for(10_000, 2500.0) == 4
    assert num_partitions_for(3750, 2500.0) == 2  # half-even
    assert num_partitions_for(10**8, 2500.0) == 40_000
    assert expected_offset(1, 5, 2) == 3
    lay = PartitionLayout(10000, 4, np.array([0, 10, -10, -5, 0], np.int64))
    assert [offset(lay, j) for j in range(5)] == [0, 2510, 4990, 7495, 10000]
    with pytest.raises(IndexError):
        offset(lay, 5)


def test_pack_unpack_deltas_roundtrip_and_reference_bytes(golden, meta):
    from paper_2404_18497_b200.partitioning import pack_deltas, unpack_deltas

    rng = np.random.default_rng(9)
    for _ in range(50):
        d = rng.integers(-200, 201, size=rng.integers(1, 40)).astype(np.int64)
        w, data = pack_deltas(d)
        assert np.array_equal(unpack_deltas(w, data, len(d)), d)
    w, data = pack_deltas(np.zeros(5, np.int64))
    assert w == 1
    # the delta section inside a reference-produced blob
    blob = golden["e2e_c1_ic-c"].tobytes()
    nparts = int.from_bytes(blob[16:24], "little")
    w = blob[57]
    nbytes = ((nparts + 1) * w + 7) // 8
    deltas = unpack_deltas(w, blob[58:58 + nbytes], nparts + 1)
    assert deltas[0] == 0 and deltas[-1] == 0
    assert pack_deltas(deltas) == (w, blob[58:58 + nbytes])


def test_deserialize_rejects_bad_input_without_touching_the_gpu(golden):
    from paper_2404_18497_b200 import FormatError, Mphf

    data = golden["e2e_small_ic-r"].tobytes()
    for cut in (0, 3, 15, 16, 40, len(data) // 2, len(data) - 1):
        with pytest.raises(FormatError):
            Mphf.deserialize(data[:cut])
    for at in (0, 5, 20, len(data) // 2, len(data) - 3):
        bad = bytearray(data)
        bad[at] ^= 0x40
        with pytest.raises(FormatError):
            Mphf.deserialize(bytes(bad))


def test_deserialize_parses_reference_bytes(golden, meta):
    """Host-side parse of every preset's reference bytes: header fields,
    encoder kinds, and re-serialisation of the parsed store."""
    from paper_2404_18497_b200 import Mphf
    from paper_2404_18497_b200.encoders import CompactVector, RiceVector

    m = meta["e2e_small"]
    for enc in m["bytes"]:
        data = golden[f"e2e_small_{enc}"].tobytes()
        g = Mphf.deserialize(data)
        assert g.n == 20_000 and g.global_seed == 3 and g.bcount == 125
        assert g.encoder_name == enc
        assert g.serialize() == data
        assert g.bits_per_key() == m["bytes"][enc]["bits_per_key"]
        encs = g.seeds.encoders
        assert all(isinstance(e, (CompactVector, RiceVector)) for e in encs)
        assert g.seeds.section() == data[data.index(g.seeds.section()):][:len(g.seeds.section())]


def test_scalar_rice_and_compact_access_matches_reference_layout(golden):
    """Host scalar accessors (select over the sampled index) agree with each
    other across presets that store the same seeds."""
    from paper_2404_18497_b200 import Mphf

    stores = {e: Mphf.deserialize(golden[f"e2e_small_{e}"].tobytes()).seeds
              for e in ("ic-r", "ic-c", "mono-r", "mono-c", "mixed:7")}
    rng = np.random.default_rng(1)
    for _ in range(300):
        j = int(rng.integers(0, 40))
        i = int(rng.integers(1, 126))
        vals = {e: s.seed_at(j, i) for e, s in stores.items()}
        assert len(set(vals.values())) == 1, vals
