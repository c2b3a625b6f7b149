"""bench.py's N > 1 path end to end: torchrun with 2 ranks (P2P transport,
CUDA IPC over torch.distributed), both ranks on cuda:0 through
MARSIT_BENCH_DEVICE (gloo for the bench's own barriers).  The ranks only
wait on each other through stream-ordered flag waits, never inside a kernel.
Checks that the run terminates (the warm-up length is decided by rank 0 for
every rank), prints one JSON line with n_gpus = 2, and that the G-rank round
equals one context holding all M workers (`parity_vs_g1`)."""
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


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_bench_two_ranks_p2p_parity(config):
    env = dict(os.environ, MARSIT_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29541" if config == "c3" else "29542",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--transport", "p2p", "--config", config,
           "--steps", "3", "--warmup", "3", "--min-busy-s", "0.5", "--e2e-steps", "2"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3
    assert d["parity_vs_g1"] == "bit-exact"
    assert len(d["per_rank_phases_ms"]) == 2
    assert d["nvlink"]["bytes_in_per_rank_per_step"] > 0
    assert d["value"] > 0 and d["e2e"]["value"] > 0
