"""Offline model of the forward kernel's shared-memory bank conflicts at config 2 (parallel
512^2 / 512 angles): exact per-iteration lane positions of a CTA (8 angles x 32 cells, lane
mappings lq 0-3, chunks of 40 units), wavefronts per LDS.128 for a layout given as a per-row slot
offset B[i mod 8] (linear pitch residues are B[i] = r i).  Used by skew_layouts.py."""
import numpy as np, sys, itertools
s=512; na=512; nd=512; half=s/2
ang=np.arange(na)*(np.pi/na)
# rays (parallel): origin u*(c,s), dir (-s,c)
u=(np.arange(nd)-nd/2+0.5)*1.0
C=np.cos(ang)[:,None]; S=np.sin(ang)[:,None]
ox=u[None,:]*C; oy=u[None,:]*S; dx=-S*np.ones_like(ox); dy=C*np.ones_like(ox)
def slab(o,d):
    with np.errstate(divide='ignore',invalid='ignore'):
        ta=(-half-o)/d; tb=(half-o)/d
    lo=np.minimum(ta,tb); hi=np.maximum(ta,tb)
    z=(d==0)
    inside=(o>=-half)&(o<=half)
    lo=np.where(z, np.where(inside,-np.inf,np.inf), lo)
    hi=np.where(z, np.where(inside,np.inf,-np.inf), hi)
    return lo,hi
l1,h1=slab(ox,dx); l2,h2=slab(oy,dy)
t0=np.maximum(l1,l2); t1=np.minimum(h1,h2)
ln=t1-t0; ok=ln>0
n=np.where(ok,np.maximum(1,np.ceil(ln)),0).astype(int)
h=np.where(ok,ln/np.maximum(n,1),1.0)
# padded pixel coords of the entry & step
px0=ox+t0*dx+half+0.5; py0=half-(oy+t0*dy)+0.5
hx=h*dx; hy=-(h*dy)
rng=np.random.default_rng(0)
CH=40.0
def cta_lanes(ca,kb,lq):
    t=np.arange(256); a=np.empty(256,int); k=np.empty(256,int)
    if lq==0:
        a=ca*8+t//32; k=kb*32+t%32
    else:
        cq=t&((8>>lq)-1); aq=(t>>(3-lq))&((1<<lq)-1); cg=(t>>3)&((4<<lq)-1); ag=t>>(lq+5)
        a=ca*8+(ag<<lq)+aq; k=kb*32+cg*(8>>lq)+cq
    return a,k
def positions(ca,kb,lq,tr):
    a,k=cta_lanes(ca,kb,lq)
    T=np.arange(-365,366,CH)
    out=[]  # list per chunk of (steps,256,2) int texel idx (i,j) + active
    for c in range(len(T)-1):
        Ta,Tb=T[c],T[c+1]
        ms=np.clip(np.ceil((Ta-t0[a,k])/h[a,k]-0.5),0,n[a,k]).astype(int)
        me=np.clip(np.ceil((Tb-t0[a,k])/h[a,k]-0.5),0,n[a,k]).astype(int)
        cnt=me-ms; Q=cnt.max()
        if Q<=0: continue
        q=np.arange(Q)[:,None]
        m=ms[None,:]+q; act=q<cnt[None,:]
        tt=m+0.5
        X=px0[a,k][None,:]+tt*hx[a,k][None,:]; Y=py0[a,k][None,:]+tt*hy[a,k][None,:]
        if tr: X,Y=Y,X
        j=np.floor(X).astype(np.int64); i=np.floor(Y).astype(np.int64)
        out.append((i,j,act))
    return out
def cost_chunk(i,j,act,B,swap):
    # B: 8-entry row base residues (i mod 8 -> slot offset); returns wavefronts
    st,L=i.shape
    odd=(np.arange(L)&1)==1
    tot=0
    for tap in range(4):
        ti=i+((1-(tap>>1)) if False else 0)
        di=(tap>>1); dj=(tap&1)
        if swap==1: di=np.where(odd,1-di,di)
        else: di=np.full(L,di)
        if swap==2: dj=np.where(odd,1-dj,dj)
        else: dj=np.full(L,dj)
        TI=i+di[None,:]; TJ=j+dj[None,:]
        slot=(B[TI&7]+TJ)&7
        addr=TI*100000+TJ
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
def ideal(act):
    st,L=act.shape
    return 4*act.reshape(st,L//8,8).any(axis=2).sum()
