"""The P2P transport's multi-process setup (CUDA IPC handle exchange over
torch.distributed) end to end: torchrun with 2 ranks (one process each),
compared bit for bit with the single-context round (tools/p2p_ipc_check.py)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_p2p_transport_across_processes():
    env = dict(os.environ, P2P_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.join(ROOT, "tools", "p2p_ipc_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "P2P IPC CHECK OK" in r.stdout, r.stdout[-2000:]
