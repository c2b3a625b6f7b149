"""Disagreement rate per round under error feedback with a fixed Gaussian
gradient (C3 size): the drift above 1/2 that the adaptive coin budget follows."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2204_06787_b200 as mb
D=25_600_000; s=mb.build_ring_schedule(8)
ctx=mb.Context(D,s,torch.float32,0)
gen=torch.Generator(device='cuda').manual_seed(1)
g=[(torch.randn(D,device='cuda',generator=gen,dtype=torch.float64)*1e-3).float() for _ in range(8)]
c=[torch.zeros(D,device='cuda') for _ in range(8)]
ctx.set_metrics(True)
for t in range(1,9):
    ctx.sign_round(t,2**-10,5,g,c)
    m=ctx.metrics()
    print(t, round(m.disagreement_rate,4), m.disagreements, m.compared_bits, round(m.matching_rate,4), flush=True)
for x,name in ((0.53,'budget'),):
    print(name, x)
