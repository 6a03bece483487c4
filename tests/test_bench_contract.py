"""bench.py contract on CPU: the reference arm (oracle port on host cores)
prints one JSON line with the driver's keys; non-zero ranks exit silently."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1",
                           "--tokens", "8"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def test_reference_arm_json_line():
    p = _run({})
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "µs" and d["higher_is_better"] is False
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "µs", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["tokens_per_rank"] == 8


def test_reference_arm_nonzero_rank_is_silent():
    p = _run({"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0
    assert p.stdout.strip() == ""
