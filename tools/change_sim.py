"""CPU simulation of a change-driven selection (rejected design):
per window, how many AB rows change and how often a pivot with U buffered
neighbours per side would need a full rescan.  usage: python tools/change_sim.py"""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
import paper_2401_13680_b200 as P
from paper_2401_13680_b200.datagen import planted_walk
x,_=planted_walk(1_000_000, m_act=256, A=4, seed=0)
def keys(e):
    b=np.asarray(e,dtype=np.float64).view(np.int64)>>32
    return b.astype(np.int32)
def run(m, s0, NWIN, U):
    pr=P.MPdistParams(m); l=pr.window_size; w=m-l+1; k=pr.k
    q=x[s0:s0+m]
    c0=200000
    ser=x[c0:c0+NWIN+2*w+l]
    def zn(a):
        W=np.lib.stride_tricks.sliding_window_view(a,l)
        mu=W.mean(1,keepdims=True); sd=W.std(1,keepdims=True)
        return (W-mu)/sd
    Q=zn(q); S=zn(ser)
    rho=(Q@S.T)/l
    e=1-rho
    K=keys(e)   # w x NC
    NC=K.shape[1]
    from numpy.lib.stride_tricks import sliding_window_view as swv
    AB=swv(K,w,axis=1).min(-1)[:, :NWIN]  # w x NWIN
    BA=K.min(0)
    nchg=(AB[:,1:]!=AB[:,:-1]).sum(0)
    # simulate
    INF=2**31-1
    def col(j): return np.concatenate([AB[:,j],BA[j:j+w]])
    def rebuild(j):
        c=np.sort(col(j)); p=c[k-1]; lt=int((c<p).sum()); le=int((c<=p).sum())
        below=c[c<p][::-1][:U].tolist(); above=c[c>p][:U].tolist()
        return p,lt,le,below,above
    p,lt,le,dn,up=rebuild(0); resc=0; moves=0
    for j in range(1,NWIN):
        ch=[(AB[i,j-1],AB[i,j]) for i in np.nonzero(AB[:,j]!=AB[:,j-1])[0]]
        ch.append((BA[j-1],BA[j+w-1]))
        for o,n in ch:
            # remove o
            if o<p:
                lt-=1; le-=1
                if dn and o>=dn[-1]: dn.remove(o)
            elif o==p: le-=1
            else:
                if up and o<=up[-1]: up.remove(o)
            if n<p:
                lt+=1; le+=1
                if dn and n>=dn[-1]:
                    dn.append(n); dn.sort(reverse=True); dn=dn[:U]
            elif n==p: le+=1
            else:
                if up and n<=up[-1]:
                    up.append(n); up.sort(); up=up[:U]
        ok = lt<k<=le
        if not ok:
            moves+=1
            if k<=lt:
                qq=lt-k+1
                if qq<=len(dn) and dn[qq-1]>dn[-1] if len(dn)>0 else False:
                    np_=dn[qq-1]; cgt=sum(1 for v in dn if v>np_); ceq=sum(1 for v in dn if v==np_)
                    mult=le-lt
                    newup=sorted([v for v in dn if v>np_])+[p]*mult+up
                    up=newup[:U]; dn=[v for v in dn if v<np_]
                    le=lt-cgt; lt=le-ceq; p=np_
                else:
                    resc+=1; p,lt,le,dn,up=rebuild(j)
            else:
                qq=k-le
                if qq<=len(up) and (up[qq-1]<up[-1] if len(up)>0 else False):
                    np_=up[qq-1]; clt=sum(1 for v in up if v<np_); ceq=sum(1 for v in up if v==np_)
                    mult=le-lt
                    newdn=sorted([v for v in up if v<np_],reverse=True)+[p]*mult+dn
                    dn=newdn[:U]; up=[v for v in up if v>np_]
                    lt=le+clt; le=lt+ceq; p=np_
                else:
                    resc+=1; p,lt,le,dn,up=rebuild(j)
        c=np.sort(col(j)); assert p==c[k-1], (j,p,c[k-1])
        assert lt==(c<p).sum() and le==(c<=p).sum()
    print(f"m={m} w={w} k={k} U={U} seg={s0}: mean AB changes/window {nchg.mean():.2f} (max {nchg.max()}), moves {moves/NWIN:.3f}, rescans {resc/NWIN:.4f}")
for m in (64,256,512):
    for U in (4,8):
        for s0 in (1000, 500000):
            run(m,s0,4000,U)
