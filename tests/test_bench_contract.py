"""bench.py's reference arm on CPU: the driver's JSON-line contract (one line,
impl "reference", cpu_baseline + e2e keys) and rank > 0 doing nothing under
torchrun."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, timeout=600, env=e, cwd=ROOT)


def test_reference_arm_json_line():
    r = run_bench("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("sign-allreduce Gelem/s")
    assert d["unit"] == "Gelem/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["config"]["workload"].startswith("c1")
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_nonzero_rank_is_silent():
    r = run_bench("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "1",
                  env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_gpus_must_match_world_size():
    """--gpus N under a launcher with another WORLD_SIZE fails loudly (it used to
    be silently rewritten)."""
    r = run_bench("--gpus", "2", env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "does not match WORLD_SIZE" in r.stderr
