"""Randomised determinism stress (tools/stress_determinism.py): random ring /
torus configurations, ragged sizes, merge kernels, tilings, coin budgets,
fused rounds and emulated P2P ranks on concurrent streams, three carried
rounds each, every compensation vector bit-identical to the oracle.  A
missing ordering in the merge barriers, the cluster barriers or the P2P flag
protocol would show up as a mismatch (profiles/r02_checked_build.txt runs the
same against the checked build that injects random sleeps at every barrier)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_random_configs_bit_exact_vs_oracle():
    env = dict(os.environ, STRESS_CONFIGS="16", STRESS_SEED="11")
    env.pop("MARSIT_SO", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_determinism.py")],
                       env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["rounds"] == 48 and d["mismatches"] == 0
