"""C5 (355M, 8 workers) driver step with and without the fused replica update
for three bucket sizes, and one bucket-sized context's per-phase times."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2204_06787_b200 as mb
def timed(fn, it=3):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/it
D,M=355_000_000,8
s=mb.build_ring_schedule(M)
g=[torch.empty(D,device='cuda') for _ in range(M)]
for w in range(M): mb.fill_recipe(g[w],0,5,w,1)
x=[torch.zeros(D,device='cuda') for _ in range(M)]
for bucket in (100_000_000, 50_000_000, 200_000_000):
    drv=mb.Driver(D,s,eta_s=2**-10,global_seed=5,bucket_elems=bucket,first_round=1)
    print(bucket, "with params %.2f ms"%timed(lambda: drv.step(g,params=x)), "no params %.2f ms"%timed(lambda: drv.step(g)), flush=True)
    del drv; torch.cuda.empty_cache()
ctx=mb.Context(88_750_000,s,torch.float32,0)
gg=[t[:88_750_000] for t in g]; cc=[torch.zeros(88_750_000,device='cuda') for _ in range(M)]
st={'t':1}
def r():
    ctx.sign_round(st['t'],2**-10,5,gg,cc); st['t']+=1
print("ctx 88.75M sign round %.3f ms"%timed(r,5))
ctx.set_timing(True); ctx.timing(reset=True)
for _ in range(5): r()
torch.cuda.synchronize(); print({k:(v[0]/5) for k,v in ctx.timing(reset=True).items() if v[1]})
