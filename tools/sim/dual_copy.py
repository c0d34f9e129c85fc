"""r2 experiment (DESIGN.md section 3 dead ends): two staged copies 4 slots apart, a lane mask per chunk.
python tools/sim/dual_copy.py <n_ctas>"""
import sys; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
from conflict_model import *
def cost_off(i,j,act,B,swap,off):
    # off: per-lane-in-quarter slot offset (8,) added to slot (second copy at +4 slots)
    st,L=i.shape
    odd=(np.arange(L)&1)==1
    lo=np.tile(off,L//8)
    tot=0
    for tap in range(4):
        di=(tap>>1); dj=(tap&1)
        di=np.where(odd,1-di,di) if swap==1 else np.full(L,di)
        dj=np.where(odd,1-dj,dj) if swap==2 else np.full(L,dj)
        TI=i+di[None,:]; TJ=j+dj[None,:]
        slot=(B[TI&7]+TJ+lo[None,:])&7
        addr=(TI*100000+TJ)*2+(lo[None,:]>0)
        addr=np.where(act,addr,-1)
        A=addr.reshape(st,L//8,8); Sl=slot.reshape(st,L//8,8); Ac=act.reshape(st,L//8,8)
        o=np.argsort(A,axis=2); A=np.take_along_axis(A,o,2); Sl=np.take_along_axis(Sl,o,2); Ac=np.take_along_axis(Ac,o,2)
        first=np.ones_like(Ac); first[:,:,1:]=A[:,:,1:]!=A[:,:,:-1]
        first&=Ac
        oh=np.zeros(A.shape[:2]+(8,),int)
        for l in range(8):
            oh+= (Sl[:,:,l][:,:,None]==np.arange(8)[None,None,:]) & first[:,:,l][:,:,None]
        w=oh.max(axis=2)
        anyact=Ac.any(axis=2)
        tot+= np.where(anyact, np.maximum(w,1),0).sum()
    return tot
rng=np.random.default_rng(1)
ctas=[(rng.integers(0,64), rng.integers(0,16)) for _ in range(int(sys.argv[1]))]
masks=[np.array([4*((m>>l)&1) for l in range(8)]) for m in range(0,256,2)]  # lane 0 in copy A (symmetry)
Ti=Tb=Td=0
for ca,kb in ctas:
    ch={tr:positions(ca,kb,0,tr) for tr in (0,1)}
    ide=base=dual=0
    for ci in range(len(ch[0])):
        best=None; bestd=None
        for tr in (0,1):
            i,j,act=ch[tr][ci]
            for sw in range(3):
                for r in range(8):
                    B=(np.arange(8)*r)&7
                    c=cost_off(i,j,act,B,sw,np.zeros(8,int))
                    if best is None or c<best[0]: best=(c,tr,sw,r)
        c0,tr,sw,r=best
        i,j,act=ch[tr][ci]; B=(np.arange(8)*r)&7
        bd=c0
        for off in masks[1:]:
            c=cost_off(i,j,act,B,sw,off)
            bd=min(bd,c)
        ide+=ideal(ch[0][ci][2]); base+=c0; dual+=bd
    Ti+=ide;Tb+=base;Td+=dual
    print(ca,kb,'base %.3f dual %.3f'%(base/ide,dual/ide),flush=True)
print('TOTAL base %.3f dual-copy %.3f'%(Tb/Ti,Td/Ti))
