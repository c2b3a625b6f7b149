#!/usr/bin/env python3
"""CPU check of the merge kernel's byte-parallel deposit (expand_masks /
expand_apply in kernels.cu) against a bit-serial pdep."""
import random
M32=0xFFFFFFFF
def pdep(x,m):
    r=0; k=0
    for i in range(32):
        if m>>i&1:
            if x>>k&1: r|=1<<i
            k+=1
    return r
def masks(m):
    pc = (m - ((m >> 1) & 0x55555555)) & M32
    pc = ((pc & 0x33333333) + ((pc >> 2) & 0x33333333)) & M32
    pc = (pc + (pc >> 4)) & 0x0F0F0F0F
    ex = (pc * 0x01010100) & M32
    mk = ((~m) << 1) & 0xFEFEFEFE & M32
    mv=[]
    for i in range(3):
        mp = mk ^ ((mk << 1) & 0xFEFEFEFE)
        mp ^= (mp << 2) & 0xFCFCFCFC
        mp ^= (mp << 4) & 0xF0F0F0F0
        mp &= M32
        v = mp & m
        m = ((m ^ v) | (v >> (1 << i))) & M32
        mk = mk & ~mp & M32
        mv.append(v)
    return mv, ex
def apply(x, mv, ex):
    e1=(ex>>8)&0xFF; e2=(ex>>16)&0xFF; e3=(ex>>24)&0xFF
    X = (x & 0xFF) | (((x >> e1) & 0xFF) << 8) | (((x >> e2) & 0xFF) << 16) | (((x >> e3) & 0xFF) << 24)
    for i in (2,1,0):
        s=1<<i
        X = ((X & ~mv[i]) | ((X << s) & mv[i])) & M32
    return X
random.seed(1)
bad=0
for t in range(200000):
    m=random.getrandbits(32); x=random.getrandbits(32)
    if t%3==0: m &= random.getrandbits(32)
    if t%5==0: m |= random.getrandbits(32)
    mv,ex=masks(m)
    got=apply(x,mv,ex) & m
    if got!=pdep(x,m): bad+=1
for b in range(256):
  for pos in range(4):
    m=b<<(8*pos) | (random.getrandbits(32) & ~(0xFF<<(8*pos)))
    for x in (0,M32,random.getrandbits(32),0x55555555):
        mv,ex=masks(m)
        if apply(x,mv,ex)&m!=pdep(x,m): bad+=1
print("bad",bad)
