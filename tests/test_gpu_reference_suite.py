"""The reference's OWN test suite (pilothash 0.1.0, pkg/tests) run with
compat_kernels installed as ``pilothash._kernels`` (tests/ref_shim), i.e.
every murmur3_many / build_partition_range / query_many_kernel call the
reference's builder, mphf and analysis modules make goes to
libphobic_b200.so on the B200.

Needs the offline install of the reference (tools/install_reference.sh ->
baseline/_ref, git-ignored; it travels to the GPU box with the snapshot).
Skipped when that install is absent. test_cli / test_service exercise the
click / FastAPI transports (out of scope) and are not run.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "reference_tests"
FILES = ["test_hashing.py", "test_builder.py", "test_mphf.py", "test_acceptance.py",
         "test_analysis.py", "test_partitioning.py", "test_assignment.py", "test_keygen.py",
         "test_encoders.py"]
# fail with the reference's own numba kernels too (encoder-size properties
# of the reference; the un-shimmed suite here: 2 failed, 138 passed)
KNOWN_REFERENCE_FAILURES = [
    "test_encoders.py::test_mixed_sweep_total_bits_non_decreasing",
    "test_mphf.py::test_space_ordering_compact_vs_rice",
]


@pytest.mark.skipif(not (REF / "pilothash").is_dir() or not SUITE.is_dir(),
                    reason="reference not installed (tools/install_reference.sh)")
def test_reference_suite_through_compat_kernels(tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests" / "ref_shim"), str(REF), str(ROOT)])
    env["NUMBA_CACHE_DIR"] = str(tmp_path / "numba")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "phb_ref_shim", "-p", "no:cacheprovider",
           "-rA", "--rootdir", str(SUITE), *FILES]
    for t in KNOWN_REFERENCE_FAILURES:
        cmd += ["--deselect", t]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=3000)
    out = r.stdout + r.stderr
    log = ROOT / "gpurun_out" / "reference_suite_shim.log"
    try:
        log.parent.mkdir(exist_ok=True)
        log.write_text(out)
    except OSError:
        pass
    assert "phb_ref_shim: pilothash._kernels -> " in out, out[-3000:]
    assert r.returncode == 0, out[-6000:]
    # every reference entry point was served by the shim (and so by the B200 library)
    calls = dict(kv.split("=") for kv in out.split("phb_ref_shim calls: ")[1].split()[:4])
    for k in ("murmur3_many", "build_partition_range", "query_many_kernel", "launches"):
        assert int(calls[k]) > 0, calls
