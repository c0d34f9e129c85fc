"""r2 experiment (DESIGN.md section 3 dead ends): annealed lane-to-ray assignment per chunk on one CTA.
python tools/sim/anneal_lanes.py <cta_angle_block> <cta_cell_block>"""
import sys, time; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
from conflict_model import *
# quarter cost for a set of lanes (columns) over a chunk, layout fixed
def qcost(i,j,act,B,sw,cols):
    ii=i[:,cols]; jj=j[:,cols]; aa=act[:,cols]
    return cost_chunk(ii,jj,aa,B,sw)
ca,kb=int(sys.argv[1]),int(sys.argv[2])
rng=np.random.default_rng(0)
ch={tr:positions(ca,kb,0,tr) for tr in (0,1)}
T0=time.time()
tot_base=tot_ann=tot_ide=0
for ci in range(len(ch[0])):
    best=None
    for tr in (0,1):
        i,j,act=ch[tr][ci]
        for sw in range(3):
            for r in range(8):
                B=(np.arange(8)*r)&7
                c=cost_chunk(i,j,act,B,sw)
                if best is None or c<best[0]: best=(c,tr,sw,r)
    c0,tr,sw,r=best; B=(np.arange(8)*r)&7
    i,j,act=ch[tr][ci]
    ide=ideal(ch[0][ci][2])
    perm=np.arange(256)
    qc=np.array([qcost(i,j,act,B,sw,perm[8*q:8*q+8]) for q in range(32)])
    cur=qc.sum()
    temp=2.0
    for it in range(6000):
        a,b=rng.integers(0,256,2)
        qa,qb=a//8,b//8
        if qa==qb: continue
        perm[a],perm[b]=perm[b],perm[a]
        na_=qcost(i,j,act,B,sw,perm[8*qa:8*qa+8]); nb_=qcost(i,j,act,B,sw,perm[8*qb:8*qb+8])
        d=na_+nb_-qc[qa]-qc[qb]
        if d<=0 or rng.random()<np.exp(-d/temp):
            qc[qa],qc[qb]=na_,nb_; cur+=d
        else:
            perm[a],perm[b]=perm[b],perm[a]
        temp*=0.999
    tot_base+=c0; tot_ann+=cur; tot_ide+=ide
    print('chunk',ci,'base %.3f anneal %.3f'%(c0/ide,cur/ide),'%.0fs'%(time.time()-T0),flush=True)
print('TOTAL base %.3f anneal %.3f'%(tot_base/tot_ide,tot_ann/tot_ide))
