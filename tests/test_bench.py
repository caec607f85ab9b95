"""bench.py's driver contract on the CPU: the reference arm prints one JSON line with the
contract's keys and the reference's own result (equal to the golden), and an N-GPU request on a
box without N GPUs fails cleanly instead of measuring something else."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")
KEYS = {"metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "result", "parity"}


def _run(*args, env=None, timeout=300):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, timeout=timeout, env=e,
                          cwd=ROOT)


def test_reference_arm_json_line():
    from oracle.refbind import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    r = _run("--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["parity"]["equal"] is True  # the reference's result equals its golden
    assert d["config"]["workload"].startswith("cfg1")


def test_gpus_request_without_gpus_fails_cleanly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("GPUs present")
    r = _run("--gpus", "2", "--steps", "1", env={"RHG_BENCH_ONE_GPU": ""})
    assert r.returncode == 2
    assert "needs 2 visible GPUs" in r.stderr
