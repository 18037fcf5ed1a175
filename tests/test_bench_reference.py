"""CPU: the reference arm of bench.py (the oracle on the host, tier framing) prints one JSON line on
the same metric / unit / workload naming as the GPU arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_arm_line_config1():
    line = _run("--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1")
    assert line["impl"] == "reference" and line["unit"] == "elements/s" and line["higher_is_better"] is True
    assert line["config"]["workload"].startswith("config 1: ")
    assert line["config"]["elements"] == 2048 and line["config"]["nodes"] == 1089
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["gpu_launches"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""
