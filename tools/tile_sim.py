"""Warp-tile lane utilisation of the (m,70) seed-1 plan: current 32-lane tiles vs alternatives."""
import numpy as np, sys
sys.path.insert(0,'.')
from oracle import oracle as O
import paper_2507_05045_b200 as msb
m=int(sys.argv[1]) if len(sys.argv)>1 else 7
inst=msb.generate_instance(m,100,1)
t=O.build_tables(inst.a)
w=[x['weights'].astype(np.int64) for x in t]
h=[np.bincount(x) for x in w]
T=int(inst.d[0])
hl=np.convolve(h[0],h[1]); hr=np.convolve(h[2],h[3])
keys=0; slots_cur=0; slots16=0; slots_q2=0; slots_flat=0
for a in range(len(hl)):
    b=T-a
    if hl[a]==0 or b<0 or b>=len(hr) or hr[b]==0: continue
    for side,(X,Y,tot) in enumerate(((h[0],h[1],a),(h[2],h[3],b))):
        ys=np.nonzero(Y)[0]
        xs=tot-ys; ok=(xs>=0)&(xs<len(X))
        ys=ys[ok]; xs=xs[ok]
        Lx=X[xs]; Ly=Y[ys]; ok=Lx>0; Lx=Lx[ok]; Ly=Ly[ok]
        L=np.maximum(Lx,Ly); Q=np.minimum(Lx,Ly)
        keys+=int((L*Q).sum())
        nl=(L+31)//32; nq=(Q+31)//32
        # current: tiles of 32 lanes x qn (steps of 4)
        full_q=Q//32; rem=Q%32
        qslots=full_q*32 + ((rem+3)//4)*4
        slots_cur+=int((nl*32*qslots).sum())
        qslots2=full_q*32 + ((rem+1)//2)*2
        slots_q2+=int((nl*32*qslots2).sum())
        nl16=(L+15)//16
        slots16+=int((nl16*16*qslots).sum())
        slots_flat+=int((((L*Q)+31)//32*32).sum())
print("keys",keys,"util cur %.3f q2 %.3f lane16 %.3f flat %.3f"%(keys/slots_cur, keys/slots_q2, keys/slots16, keys/slots_flat))
# orientation by utilisation (lanes over whichever run wastes less)
def slots(L, Q):
    return ((L + 31) // 32) * 32 * ((Q // 32) * 32 + (((Q % 32) + 3) // 4) * 4)
keys=0; s_cur=0; s_best=0
for a in range(len(hl)):
    b=T-a
    if hl[a]==0 or b<0 or b>=len(hr) or hr[b]==0: continue
    for X,Y,tot in ((h[0],h[1],a),(h[2],h[3],b)):
        ys=np.nonzero(Y)[0]; xs=tot-ys; ok=(xs>=0)&(xs<len(X)); ys=ys[ok]; xs=xs[ok]
        Lx=X[xs]; Ly=Y[ys]; ok=Lx>0; Lx=Lx[ok]; Ly=Ly[ok]
        L=np.maximum(Lx,Ly); Q=np.minimum(Lx,Ly)
        keys+=int((L*Q).sum())
        a1=slots(L,Q); a2=slots(Q,L)
        s_cur+=int(a1.sum()); s_best+=int(np.minimum(a1,a2).sum())
print("orientation: longer-across %.3f best-of-two %.3f" % (keys/s_cur, keys/s_best))
# split each rectangle into its full 32-lane part and the remainder, each oriented the cheaper way
def best(L, Q):
    return np.minimum(slots(L, Q), slots(Q, L))
def split_slots(L, Q, depth=2):
    # orient the rectangle the cheaper way, then carve off the full lane tiles and re-plan the rest
    lx = slots(L, Q) <= slots(Q, L)
    A = np.where(lx, L, Q); B = np.where(lx, Q, L)
    full = (A // 32) * 32; r = A - full
    main = np.where(full > 0, slots(full, B), 0)
    rem = np.where(r > 0, (split_slots(r, B, depth - 1) if depth > 1 else best(r, B)), 0)
    return np.where((full > 0) & (r > 0), main + rem, best(L, Q))
keys=0; s_split=0; s_split3=0
for a in range(len(hl)):
    b=T-a
    if hl[a]==0 or b<0 or b>=len(hr) or hr[b]==0: continue
    for X,Y,tot in ((h[0],h[1],a),(h[2],h[3],b)):
        ys=np.nonzero(Y)[0]; xs=tot-ys; ok=(xs>=0)&(xs<len(X)); ys=ys[ok]; xs=xs[ok]
        Lx=X[xs]; Ly=Y[ys]; ok=Lx>0; Lx=Lx[ok].astype(np.int64); Ly=Ly[ok].astype(np.int64)
        keys+=int((Lx*Ly).sum())
        s_split+=int(split_slots(Lx,Ly,1).sum()); s_split3+=int(split_slots(Lx,Ly,3).sum())
print("split remainder: depth1 %.3f depth3 %.3f" % (keys/s_split, keys/s_split3))
