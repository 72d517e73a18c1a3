"""Model of the decode FFN tile schedule (config 3, B = 256, E = 8): 344 gate/up tiles of 2 MiB and 128 down tiles
of 2.75 MiB (or 256 of 1.375 MiB) over 74 CTA pairs, down tiles of an expert waiting for all its gate/up tiles.
Prints the makespan in MiB per pair for static round-robin orders and dynamic fetch. Analysis only."""
import itertools
P=74; E=8; NGU=43; NDN=16; GU=2.0; DN=2.75
def sim(order):
    # order: list of (kind, e); rr static assignment; each pair sequential; dn(e) waits for all gu(e) done
    pairs=[[] for _ in range(P)]
    for i,t in enumerate(order): pairs[i%P].append(t)
    # event simulation: process in global order positions; need gu finish times per expert
    # iterative: compute times pair by pair in order of position index (tiles at position j wait on earlier)
    tfree=[0.0]*P; gu_done={e:0.0 for e in range(E)}; gu_left={e:NGU for e in range(E)}
    pend=[0]*P
    # simple loop: repeatedly advance the pair whose next tile can start earliest
    import heapq
    done=0; total=len(order); finish=[0.0]*P
    while done<total:
        best=None
        for p in range(P):
            if pend[p]>=len(pairs[p]): continue
            k,e=pairs[p][pend[p]]
            if k=='d' and gu_left[e]>0: continue
            st=max(tfree[p], gu_done[e] if k=='d' else 0.0)
            if best is None or st<best[0]: best=(st,p)
        st,p=best; k,e=pairs[p][pend[p]]
        en=st+(GU if k=='g' else DN); tfree[p]=en; pend[p]+=1; done+=1
        if k=='g':
            gu_left[e]-=1; gu_done[e]=max(gu_done[e],en)
    return max(tfree)
base=[('g',e) for e in range(E) for _ in range(NGU)]+[('d',e) for e in range(E) for _ in range(NDN)]
print('current', sim(base), 'ideal', (E*NGU*GU+E*NDN*DN)/P)
for lag in (1,2,3):
    o=[]
    for e in range(E):
        o+= [('g',e)]*NGU
        if e-lag>=0: o+=[('d',e-lag)]*NDN
    for e in range(E-lag,E): o+=[('d',e)]*NDN
    print('interleave lag',lag, sim(o))
print('--- finer down tiles (N=128)')
NDN=32; DN=1.375
base=[('g',e) for e in range(E) for _ in range(NGU)]+[('d',e) for e in range(E) for _ in range(NDN)]
print('current order, fine down', sim(base))
for lag in (1,2):
    o=[]
    for e in range(E):
        o+= [('g',e)]*NGU
        if e-lag>=0: o+=[('d',e-lag)]*NDN
    for e in range(E-lag,E): o+=[('d',e)]*NDN
    print('interleave lag',lag, sim(o))
def simdyn(order):
    import heapq
    h=[(0.0,p) for p in range(P)]; heapq.heapify(h)
    gu_done={e:0.0 for e in range(E)}; gu_left={e:sum(1 for k,x in order if k=='g' and x==e) for e in range(E)}
    gfin={e:[] for e in range(E)}
    end=0
    for k,e in order:
        t,p=heapq.heappop(h)
        if k=='d':
            st=max(t, max(gfin[e]))
        else: st=t
        en=st+(GU if k=='g' else DN)
        if k=='g': gfin[e].append(en)
        heapq.heappush(h,(en,p)); end=max(end,en)
    return end
for ndn,dn in ((16,2.75),(32,1.375)):
    NDN=ndn; DN=dn
    base=[('g',e) for e in range(E) for _ in range(NGU)]+[('d',e) for e in range(E) for _ in range(NDN)]
    print('dynamic', ndn, simdyn(base))
