"""r2 experiment (DESIGN.md section 3 dead ends): 45-degree (u = i +- j) box layouts beside the linear ones.
python tools/sim/diag_layout.py <n_ctas> [seed]"""
import sys, time; sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
from conflict_model import *
def wave(addr_rows, addr_cols, act, r):
    # addr_rows/cols: (st,L) ints; slot = (r*row + col)&7; cost per quarter = max distinct per slot
    st,L=addr_rows.shape
    slot=(r*addr_rows+addr_cols)&7
    addr=addr_rows*100000+addr_cols
    addr=np.where(act,addr,-1)
    A=addr.reshape(st,L//8,8); Sl=slot.reshape(st,L//8,8); Ac=act.reshape(st,L//8,8)
    o=np.argsort(A,axis=2); A=np.take_along_axis(A,o,2); Sl=np.take_along_axis(Sl,o,2); Ac=np.take_along_axis(Ac,o,2)
    first=np.ones_like(Ac); first[:,:,1:]=A[:,:,1:]!=A[:,:,:-1]
    first&=Ac
    oh=np.zeros(A.shape[:2]+(8,),int)
    for l in range(8):
        oh+=(Sl[:,:,l][:,:,None]==np.arange(8)[None,None,:]) & first[:,:,l][:,:,None]
    w=oh.max(axis=2)
    return np.where(Ac.any(axis=2), np.maximum(w,1),0).sum()
def cost_diag(i,j,act,r,sgn,order):
    # sgn=+1: row=i+j, v=i-j ; sgn=-1: row=i-j, v=i+j ; col=(v+C)>>1
    C=4096
    taps=[(0,0),(0,1),(1,0),(1,1)]
    L=i.shape[1]; odd=(np.arange(L)&1)==1
    tot=0
    for k in range(4):
        # order 1: odd lanes issue taps in reverse order
        di=np.where(odd & (order==1), taps[3-k][0], taps[k][0]); dj=np.where(odd & (order==1), taps[3-k][1], taps[k][1])
        I=i+di[None,:]; J=j+dj[None,:]
        if sgn>0: row=I+J; v=I-J
        else: row=I-J; v=I+J
        col=(v+C)>>1
        tot+=wave(row,col,act,r)
    return tot
def cost_lin(i,j,act,r,sw):
    return cost_chunk(i,j,act,(np.arange(8)*r)&7,sw)
rng=np.random.default_rng(int(sys.argv[2]) if len(sys.argv)>2 else 1)
ctas=[(rng.integers(0,64), rng.integers(0,16)) for _ in range(int(sys.argv[1]))]
Ti=Tb=Td=0
for ca,kb in ctas:
    ch={tr:positions(ca,kb,0,tr) for tr in (0,1)}
    ide=base=dg=0
    for ci in range(len(ch[0])):
        b=min(cost_lin(*ch[tr][ci],r,sw) for tr in (0,1) for sw in range(3) for r in range(8))
        i,j,act=ch[0][ci]
        d=min(cost_diag(i,j,act,r,sg,o) for sg in (1,-1) for r in range(8) for o in (0,1))
        ide+=ideal(act); base+=b; dg+=min(b,d)
    Ti+=ide;Tb+=base;Td+=dg
    print(ca,kb,'angle %.0f'%(ca*8*180/512),'base %.3f with-diag %.3f'%(base/ide,dg/ide),flush=True)
print('TOTAL base %.3f with-diag %.3f'%(Tb/Ti,Td/Ti))
