#!/usr/bin/env python3
"""Multi-process check of the P2P transport setup: every rank (one process)
creates its context, exchanges CUDA IPC handles of its buffers over
torch.distributed (gloo) and runs sign + dense rounds; rank 0 compares every
rank's compensation with a single-context run.  Launched by
tests/test_gpu_p2p_ipc.py with torchrun (all ranks may share one GPU: ranks
never run kernels that wait on each other, only stream-ordered flag waits)."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_06787_b200 as mb  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("P2P_DEVICE", rank % max(torch.cuda.device_count(), 1)))
    torch.cuda.set_device(dev)
    D, W, seed, eta, period = 200_003, 8, 11, 2.0 ** -10, 3
    sched = mb.build_ring_schedule(W)
    ml = W // G
    ctx = mb.Context(D, sched, torch.float32, dev, nranks=G, rank=rank, transport="p2p")
    opened = mb.exchange_p2p_buffers(ctx)
    comp = [torch.zeros(D, device=f"cuda:{dev}") for _ in range(ml)]
    for t in range(0, 4):  # t = 0, 3 dense
        grads = [torch.empty(D, device=f"cuda:{dev}") for _ in range(ml)]
        for i in range(ml):
            mb.fill_recipe(grads[i], 0, seed, rank * ml + i, t)
        if t % period == 0:
            mean = torch.empty(D, device=f"cuda:{dev}")
            ctx.dense_round(t, grads, comp, mean)
        else:
            ctx.sign_round(t, eta, seed, grads, comp)
    torch.cuda.synchronize()
    ctx.check()
    got = [c.cpu() for c in comp]
    allc = [None] * G
    dist.all_gather_object(allc, got)
    ok = True
    if rank == 0:
        single = mb.Context(D, sched, torch.float32, dev)
        comp1 = [torch.zeros(D, device=f"cuda:{dev}") for _ in range(W)]
        for t in range(0, 4):
            grads = [torch.empty(D, device=f"cuda:{dev}") for _ in range(W)]
            for w in range(W):
                mb.fill_recipe(grads[w], 0, seed, w, t)
            if t % period == 0:
                single.dense_round(t, grads, comp1, torch.empty(D, device=f"cuda:{dev}"))
            else:
                single.sign_round(t, eta, seed, grads, comp1)
        torch.cuda.synchronize()
        for w in range(W):
            ok &= torch.equal(allc[w // ml][w % ml], comp1[w].cpu())
        print("P2P IPC CHECK", "OK" if ok else "MISMATCH", f"(G={G})", flush=True)
    dist.barrier()
    del ctx
    for p in opened:
        mb._native.lib().marsit_ipc_close(p)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
