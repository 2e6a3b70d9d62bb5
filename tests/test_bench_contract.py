"""bench.py's reference arm runs on the host (pilothash itself from
baseline/_ref when installed, else the oracle port): its JSON line follows
the driver's contract (CPU-only; the GPU arm is exercised on the B200).
bench.py --gpus N without torchrun re-executes itself under torchrun."""

import json
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps",
                        "1", "--warmup", "0", "--ref-sample", "20000"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["unit"] == "keys/s" and line["value"] > 0 and line["higher_is_better"]
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


import pytest  # noqa: E402


def test_self_spawn_under_torchrun(monkeypatch):
    """--gpus N > 1 with WORLD_SIZE unset: bench.py re-executes itself under
    torchrun with N ranks on 127.0.0.1 and exits with the ranks' status."""
    sys.path.insert(0, str(ROOT))
    import bench

    seen = {}

    class R:
        returncode = 0

    def fake_run(cmd, env=None, **kw):
        seen["cmd"], seen["env"] = cmd, env
        return R()

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_world_size_must_match_gpus(monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit):
        bench.dist_init(4)


def test_self_spawned_ranks_run_end_to_end_gloo():
    """The spawned torchrun ranks come up, rendezvous on 127.0.0.1 and run
    (gloo, CPU): a tiny script launched the same way bench.py launches itself."""
    script = ROOT / "tests" / "_spawn_probe.py"
    r = subprocess.run([sys.executable, "-c",
                        "import sys; sys.path.insert(0, %r); import bench; "
                        "sys.argv=['bench.py', '--gpus', '2']; sys.exit(bench.spawn_ranks(2, %r))"
                        % (str(ROOT), str(script))],
                       capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**__import__("os").environ, "PYTHONPATH": str(ROOT)})
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert r.stdout.count("probe ok world=2") == 2, r.stdout[-2000:]


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """bench.py's GPU arm on a small key count: every field of the driver's
    contract plus the roofline / cpu_baseline / e2e objects."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                        "--keys", "4000000", "--e2e-steps", "1", "--ref-sample", "200000",
                        "--no-configs", "--no-c3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks", "cpu_baseline", "query", "bits_per_key"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["value"] > 0
    assert line["gpu_launches"] > 0 and line["timed_build_equals_e2e_build"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in line["roofline"], k
    assert line["e2e"]["h2d_bytes_per_step"] == 4_000_000 * 8
    assert line["query"]["bijection_verified"] and line["query"]["encoded"]["equal_to_matrix_query"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in line["cpu_baseline"], k
