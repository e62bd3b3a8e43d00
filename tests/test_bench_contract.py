"""bench.py's reference arm on CPU: one JSON line with the driver's contract keys,
on the same metric as the CUDA arm, timing the reference package itself
(baseline/_ref, kind "reference") on the host threads -- or the C oracle port
(kind "port") where it is not installed -- with the config of what actually
ran; under torchrun only rank 0 prints (the others exit 0 without work)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "impl", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e")


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--cpu-n", "16", "--steps", "2", "--warmup", "1", *args],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert all(k in d for k in KEYS)
    assert d["impl"] == "reference" and d["unit"] == "pt*step/s" and d["value"] > 0
    assert d["metric"] == "grid-point RK4-step updates/sec (fp64, 512^3)"
    assert d["config"]["grid"] == 16 and d["config"]["scheme"] == "rk4"
    assert "16^3" in d["config"]["sample"] and "CPU" in d["config"]["parallelism"]
    cb = d["cpu_baseline"]
    installed = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "hitdns"))
    assert cb["kind"] == ("reference" if installed else "port")
    assert cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "pt*step/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_non_zero_ranks_are_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}) == []
