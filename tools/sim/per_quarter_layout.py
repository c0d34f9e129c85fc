"""r2 experiment (DESIGN.md section 3 dead ends): per-quarter-warp layout choice (upper bound) and two layouts.
python tools/sim/per_quarter_layout.py <n_ctas>"""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
from conflict_model import *
rng=np.random.default_rng(1)
ctas=[(rng.integers(0,64), rng.integers(0,16)) for _ in range(int(sys.argv[1]))]
Ti=Tb=Tq=T2=0
for ca,kb in ctas:
  for lq in [0]:
    ch={tr:positions(ca,kb,lq,tr) for tr in (0,1)}
    ide=base=perq=two=0
    for ci in range(len(ch[0])):
        costs=[]  # layouts x quarters
        for tr in (0,1):
            i,j,act=ch[tr][ci]
            for sw in range(3):
                for r in range(8):
                    B=(np.arange(8)*r)&7
                    qc=[cost_chunk(i[:,8*q:8*q+8],j[:,8*q:8*q+8],act[:,8*q:8*q+8],B,sw) for q in range(32)]
                    costs.append(qc)
        C=np.array(costs)  # L x 32
        ide+=ideal(ch[0][ci][2]); base+=C.sum(1).min(); perq+=C.min(0).sum()
        # best pair of layouts, each quarter takes the cheaper
        L=C.shape[0]; best=1e18
        for a in range(L):
            m=np.minimum(C[a][None,:],C).sum(1).min()
            best=min(best,m)
        two+=best
    Ti+=ide;Tb+=base;Tq+=perq;T2+=two
    print(ca,kb,'cta %.3f perq %.3f two %.3f'%(base/ide,perq/ide,two/ide),flush=True)
print('TOTAL cta %.3f perq %.3f two-layouts %.3f'%(Tb/Ti,Tq/Ti,T2/Ti))
