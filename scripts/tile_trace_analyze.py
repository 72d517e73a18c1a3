"""Offline analysis of a scripts/tile_trace_lab.py run: per tile kind (gate/up or down; 256-row, merged-tail
or swap-AB tile) the SM cycles between consecutive accumulator completions against the ideal MMA cycles, the
MMA warp's waits, the epilogue time, per-tail-size cost per K step and the idle gaps between tiles.
Usage: python scripts/tile_trace_analyze.py RUN.json RECORDS.npy [MERGE=1]  (measurement only)"""
import json, numpy as np, sys
d=json.load(open(sys.argv[1])); rec=np.load(sys.argv[2]).astype(np.uint64).astype(np.float64)
MERGE=int(sys.argv[3]) if len(sys.argv)>3 else 1
H,dd=d.get('H',4096),d.get('d',5504)
counts=d['counts']; offs=np.concatenate([[0],np.cumsum(counts)])
NT1,NT2=(dd+127)//128,(H+255)//256; KB1,KB2=(H+63)//64,(dd+63)//64
def seg_tiles(R):
    if not MERGE or R < 256: return [(min(256, R-256*m),0) for m in range((R+255)//256)]
    nf,rem=R>>8,R&255
    if rem==0 or rem>64*min(nf,2): return [(min(256,R-256*m),0) for m in range(nf+(1 if rem else 0))]
    return [(256, min(64, rem-64*m) if m*64<rem else 0) for m in range(nf)]
def mma(rows,tr):
    if rows<=64: c,k=128*((rows+15)//16*16)/256,'swap'
    elif rows>128: c,k=128,'m256'
    else: c,k=64,'m128'
    if tr: c,k=c+128*((tr+15)//16*16)/256,'m256+tail'
    return c,k
kinds=[]
for ph in (0,1):
    NT,KB=(NT1,KB1) if ph==0 else (NT2,KB2)
    for g in range(len(counts)):
        ts=seg_tiles(counts[g])
        for n in range(NT):
            for rows,tr in ts:
                c,k=mma(rows,tr); kinds.append((ph,k,KB*4*c))
print('ntiles',len(kinds))
pk={}; ideal_pair=[]; span=[]; ends=[]; starts=[]; epi=[]
for p in range(rec.shape[0]):
    r=rec[p]; n=int((r[:,1]>0).sum()); prev=None; ip=0
    for i in range(n):
        t=int(r[i,7])&0xffffffff; ph,k,ideal=kinds[t]
        st=r[i,1] if prev is None else max(prev,r[i,1]); ex=r[i,3]-st; prev=r[i,3]
        key=('gu_' if ph==0 else 'dn_')+k; e=pk.setdefault(key,[0,0,0,0,0]); e[0]+=1;e[1]+=ex;e[2]+=ideal;e[3]+=r[i,6]; e[4]+=r[i,4]-r[i,3]
        ip+=ideal
    ideal_pair.append(ip); span.append(r[n-1,4]-r[0,1]); ends.append(r[n-1,5]); starts.append(r[0,0])
t0=min(starts); ends=(np.array(ends)-t0)/1e3
print('end us min/mean/max',ends.min(),ends.mean(),ends.max())
print('span cyc mean/max',np.mean(span),np.max(span),'ideal pair mean/max/min',np.mean(ideal_pair),np.max(ideal_pair),np.min(ideal_pair))
print('mean ideal / max span', np.mean(ideal_pair)/np.max(span), 'corr ideal vs span', np.corrcoef(ideal_pair,span)[0,1])
for k,v in sorted(pk.items()): print(k,'n',v[0],'exec',round(v[1]/v[0]),'ideal',round(v[2]/v[0]),'eff',round(v[2]/v[1],3),'fullwait',round(v[3]/v[0]),'epi',round(v[4]/v[0]))
# per tail-size cost
kk=[]
for ph in (0,1):
    NT,KB=(NT1,KB1) if ph==0 else (NT2,KB2)
    for g in range(len(counts)):
        ts=seg_tiles(counts[g])
        for n in range(NT):
            for rows,tr in ts: kk.append((ph,tr,KB))
bys={}
for p in range(rec.shape[0]):
    r=rec[p]; n=int((r[:,1]>0).sum()); prev=None
    for i in range(n):
        t=int(r[i,7])&0xffffffff; ph,tr,KB=kk[t]
        st=r[i,1] if prev is None else max(prev,r[i,1]); ex=r[i,3]-st; prev=r[i,3]
        bys.setdefault((ph,tr),[]).append(ex/KB)
for k in sorted(bys): print(k, len(bys[k]), round(np.median(bys[k]),1))
gaps=[];first=[];last_end=[]
g0=None
for p in range(rec.shape[0]):
    r=rec[p]; n=int((r[:,1]>0).sum()); gp=0
    for i in range(1,n):
        gp+=max(0,r[i,1]-r[i-1,3])
    gaps.append(gp)
print('gap per pair mean/max', np.mean(gaps), np.max(gaps))
# tempty waits (acc wait) and gap sources
aw=[ (int(v)>>32) for v in rec[:,:,7].flatten() if v>0]
print('acc-wait mean', np.mean(aw), 'sum per pair', np.sum(aw)/rec.shape[0])
