# Per-stage timestamp analysis of a lab build (-DREADME_LAB_STAGETS=i, not in the product): TMA latency,
# slot refill and stage period per CTA pair from scripts/tile_trace_lab.py output (TT_NREC=40). Measurement only.
import numpy as np, json, sys
rec=np.load(sys.argv[1]).astype(np.uint64).astype(np.int64)  # [NP, MAXT, 8]
NP=rec.shape[0]
d=json.load(open(sys.argv[2]))
res=[]
for p in range(NP):
    r=rec[p].reshape(-1)
    st=r[40*8:40*8+192]
    P,F,I=st[:64],st[64:128],st[128:192]
    if (P==0).any() or (F==0).any(): continue
    t=int(rec[p,6,7])&0xffffffff
    # TMA latency: producer empty-wait return (issue) -> MMA full-wait return for the same kb
    lat=F-P
    # slot cycle: full-return of kb -> producer wait-return for kb+6 (slot refill start)
    refill=P[6:]-I[:-6]
    per=np.diff(I)
    res.append((t,np.median(lat),np.median(refill),np.median(per),np.median(I-F)))
a=np.array(res)
print('n',len(a))
print('median over pairs: TMA issue->full seen %.0f, MMA issued(kb)->producer slot free(kb+6) %.0f, stage period %.0f, full->issued %.0f'%tuple(np.median(a[:,1:],axis=0)))
print('p10', np.percentile(a[:,1:],10,axis=0), 'p90', np.percentile(a[:,1:],90,axis=0))
