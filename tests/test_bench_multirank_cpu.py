"""bench.py's N > 1 warm-up on CPU (gloo, world size 2): the ranks' own clocks
differ (rank 1 steps 3x slower), yet rank 0's decision is broadcast so both
run the same number of rounds — a rank that ran ahead would wait forever on
P2P flags / NCCL collectives its peers never issue (transport.hpp:27-35)."""
import os
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    import time

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)

    comm = bench.Comm.__new__(bench.Comm)  # bench.Comm over gloo with CPU tensors
    comm.dist, comm.world, comm.rank = dist, world, rank
    import torch
    comm.tdev = torch.device("cpu")
    delay = 0.002 if rank == 0 else 0.006
    n = bench.warm_up(comm, lambda t: time.sleep(delay), lambda: None, 5, 0.3)
    q.put((rank, n))
    dist.destroy_process_group()


def test_warm_up_round_count_agreed_across_ranks():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res[0] == res[1] and res[0] >= 5
