"""Step time with and without the per-phase CUDA-event instrumentation
(marsit_ctx_set_timing) at C3."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2204_06787_b200 as mb
D=25_600_000; s=mb.build_ring_schedule(8)
ctx=mb.Context(D,s,torch.float32,0)
g=[torch.empty(D,device='cuda') for _ in range(8)]
for w in range(8): mb.fill_recipe(g[w],0,2026,w,1)
c=[torch.zeros(D,device='cuda') for _ in range(8)]
st={'t':1}
def r():
    ctx.sign_round(st['t'],2**-10,2026,g,c); st['t']+=1
def timed(n=50):
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): r()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/n*1e3
for _ in range(300): r()
for i in range(3):
    ctx.set_timing(False); off=timed()
    ctx.set_timing(True); ctx.timing(reset=True); on=timed(); ctx.set_timing(False)
    print(f"timing off {off:.1f} us/round, on {on:.1f} us/round")
