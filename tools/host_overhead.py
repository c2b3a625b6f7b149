"""Host enqueue time of one sign round through the Python API at C1 size vs
the wall time per round once the queue drains (is the small config host-bound?)."""
import sys, os, time, torch
sys.path.insert(0, os.getcwd())
import paper_2204_06787_b200 as mb
D=1_000_000; s=mb.build_ring_schedule(4)
ctx=mb.Context(D,s,torch.float32,0)
g=[torch.empty(D,device='cuda') for _ in range(4)]
for w in range(4): mb.fill_recipe(g[w],0,2026,w,1)
c=[torch.zeros(D,device='cuda') for _ in range(4)]
for t in range(1,20): ctx.sign_round(t,2**-10,2026,g,c)
torch.cuda.synchronize()
N=2000
t0=time.perf_counter()
for t in range(20,20+N): ctx.sign_round(t,2**-10,2026,g,c)
t1=time.perf_counter()
torch.cuda.synchronize()
t2=time.perf_counter()
print(f"host enqueue {((t1-t0)/N)*1e6:.1f} us/round; wall incl. drain {((t2-t0)/N)*1e6:.1f} us/round")
