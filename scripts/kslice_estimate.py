"""Share of the accumulation k-slices (32 columns) that are structurally zero in an operand of the
face-grown dissection's tile products (python scripts/kslice_estimate.py c3 3 32)."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
from harness import inputs
from paper_2502_08382_b200 import sparse_route as spr, dualop
cfg=sys.argv[1]; depth=int(sys.argv[2]); KS=int(sys.argv[3]) if len(sys.argv)>3 else 32
prob = inputs.Problem(*inputs.CONFIGS[cfg]); cons=prob.constraints()
f,s2=dualop._multiplier_owners(cons); m=prob.m_per_subdomain(); s=int(np.argmax(m)); g=prob.gids[s]
nb=np.where(f[g]==s,s2[g],f[g]); pieces=spr.interface_pieces(prob.bcol[s],nb)
k,_,q=prob.subdomain_system(s); n=k.shape[0]; ip,ix=np.asarray(k.indptr),np.asarray(k.indices); bcol=prob.bcol[s]
segs=spr.face_dissection_segments(n,ip,ix,bcol,pieces,depth)
perm,iperm=spr.padded_positions(segs); npos=perm.shape[0]
rows=np.repeat(np.arange(n),np.diff(ip)); pi,pj=iperm[rows],iperm[ix]; lo=pi>pj
colpat=[[] for _ in range(npos)]
for a,b in zip(pi[lo].tolist(),pj[lo].tolist()): colpat[b].append(a)
pend=[[] for _ in range(npos)]; pat=[None]*npos
for j in range(npos):
    st=np.unique(np.concatenate([np.array(colpat[j],np.int64)]+pend[j])); st=st[st>j]; pat[j]=st
    if st.size: pend[st[0]].append(st)
    pend[j]=None
TB=128; T=npos//TB; NS=TB//KS
ni=np.unique(bcol).size; smin=(npos - -(-len(segs[-1])//128)*128)//TB
# slice masks: smask[(i,k)] bitmask of k-slices with a nonzero in block row i
from collections import defaultdict
smask=defaultdict(int)
for c in range(npos):
    kb=c//TB; sl=(c%TB)//KS
    for i in np.unique(pat[c]//TB).tolist():
        smask[(i,kb)] |= (1<<sl)
    smask[(kb,kb)] |= (1<<sl)
# dense interface: every tile in trailing triangle full
for K in range(smin,T):
    for I in range(K,T): smask[(I,K)] = (1<<NS)-1
# block structure with fill as in the estimator
ss=[set() for _ in range(T)]
for (i,kk),mk in smask.items():
    if i>kk: ss[kk].add(i)
for kk in range(T):
    st=ss[kk]
    if st: p0=min(st); ss[p0] |= (st-{p0})
rowsof=defaultdict(list)
for kk in range(T):
    for i in ss[kk]: rowsof[i].append(kk)
full=0; used=0
for j in range(T):
    targets=[j]+sorted(ss[j])
    for i in targets:
        for kk in set(rowsof[i]) & set(rowsof[j]):
            a=smask.get((i,kk),(1<<NS)-1); b=smask.get((j,kk),(1<<NS)-1)
            full+=NS; used+=bin(a&b).count('1')
print(cfg,'KS',KS,'acc slices total',full,'needed',used,'skippable %.1f%%'%(100*(1-used/full)))
