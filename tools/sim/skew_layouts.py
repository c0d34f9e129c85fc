"""Do per-row bank skews (arbitrary B[i mod 8], i.e. any row-base residue pattern, found by
coordinate descent per chunk from the best linear pitch residue) beat the planner's layout family
(orientation x pitch residue x tap order, chosen per chunk with the whole chunk simulated)?
r2 result (6 random cfg2 CTAs): base 1.220x, skew 1.220x conflict-free wavefronts - no gain: the
lane-point patterns are translates of one another across quarter warps, so a row-periodic skew
that helps one quarter warp hurts its neighbours.  python tools/sim/skew_layouts.py [n_ctas]"""
import sys; import os; sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from conflict_model import *
import time
rng=np.random.default_rng(1)
ctas=[(rng.integers(0,64), rng.integers(0,16)) for _ in range(int(sys.argv[1]) if len(sys.argv)>1 else 12)]
tot_ideal=0; tot_base=0; tot_skew=0
t_start=time.time()
for (ca,kb) in ctas:
    best_lq=None
    res={}
    for lq in range(4):
        chunks={tr:positions(ca,kb,lq,tr) for tr in (0,1)}
        base=0; ide=0; choice=[]
        for ci in range(len(chunks[0])):
            best=None
            for tr in (0,1):
                i,j,act=chunks[tr][ci]
                for sw in range(3):
                    for r in range(8):
                        B=(np.arange(8)*r)&7
                        c=cost_chunk(i,j,act,B,sw)
                        if best is None or c<best[0]: best=(c,tr,sw,B)
            base+=best[0]; ide+=ideal(chunks[0][ci][2]); choice.append(best)
        res[lq]=(base,ide,choice,chunks)
    lq=min(res,key=lambda q:res[q][0])
    base,ide,choice,chunks=res[lq]
    skew=0
    for ci,(c,tr,sw,B) in enumerate(choice):
        i,j,act=chunks[tr][ci]
        B=B.copy(); cur=c
        for it in range(2):
            for p in range(1,8):
                for v in range(8):
                    if v==B[p]: continue
                    B2=B.copy(); B2[p]=v
                    c2=cost_chunk(i,j,act,B2,sw)
                    if c2<cur: cur=c2; B=B2
        skew+=cur
    tot_ideal+=ide; tot_base+=base; tot_skew+=skew
    print(ca,kb,'lq',lq,'base %.3f skew %.3f'%(base/ide, skew/ide), 'elapsed %.0f'%(time.time()-t_start), flush=True)
print('TOTAL base %.3f skew %.3f'%(tot_base/tot_ideal, tot_skew/tot_ideal))
