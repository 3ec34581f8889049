"""CPU checks of bench.py's host-side contract: the reference arm (the oracle
timed on host cores) prints one JSON line with the keys the driver reads, and
ranks other than 0 exit 0 without work. No GPU, no CUDA extension."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--config", "c3_posets", "--steps", "1", "--warmup", "0",
                           "--cpu-seconds", "0.6", *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)


def test_reference_arm_json_line():
    p = _run()
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "valuations/s" and d["unit"] == "valuations/s"
    assert d["higher_is_better"] is True and d["steps"] == 1 and d["warmup"] == 0
    assert d["value"] > 0 and d["ms_per_step"] > 0
    # ms_per_step is the time for the whole 2^n workload at the measured rate
    assert abs(d["ms_per_step"] - (1 << 25) / d["value"] * 1e3) < 1e-6 * d["ms_per_step"]
    assert d["config"]["n"] == 25 and d["config"]["workload"].startswith("c3_posets")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "sub-cube" in cb["sample"] and "of 2^" in cb["sample"] and cb["cpu_model"]
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_nonzero_rank_is_silent():
    p = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip() == ""


def test_reference_arm_small_n():
    """n = 9 (C1) is smaller than the oracle-rate probe's first sub-cube:
    the probe must clamp to the whole cube instead of asking for a bad range."""
    env = dict(os.environ)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "c1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["config"]["n"] == 9 and "2^9 valuations [0, 512)" in d["cpu_baseline"]["sample"]
