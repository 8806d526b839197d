"""Leaf coupling of the face-grown dissection: boundary rows of every leaf and the tiles they
spread over now vs row-compressed (python scripts/leaf_coupling_estimate.py c3 3)."""
import sys, numpy as np
sys.path.insert(0,'/root/repo')
from harness import inputs
from paper_2502_08382_b200 import sparse_route as spr, dualop
cfg=sys.argv[1]; depth=int(sys.argv[2])
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
segid=np.zeros(npos,np.int64); p=0; segstart=[]
for i,sg in enumerate(segs):
    L=-(-sg.size//128)*128; segid[p:p+L]=i; segstart.append(p); p+=L
# leaf segments: those followed by non-leaf? identify leaves as segments of size>=500 excluding the last (interface)
TB=128
tot_cur=0; tot_cmp=0
for i,sg in enumerate(segs[:-1]):
    if sg.size < 400: continue
    a=segstart[i]; b=a+(-(-sg.size//128))*128
    # boundary rows of the leaf: rows >= b in any leaf column pattern
    B=np.unique(np.concatenate([pat[j][pat[j]>=b] for j in range(a,b) if pat[j].size]))
    nt_leaf=(b-a)//TB
    cur_tiles=np.unique(B//TB).size
    cmp_tiles=-(-B.size//TB)
    # products for leaf block columns (left-looking, dense within leaf+boundary tiles as an upper bound): per leaf block col kb: targets below = (nt_leaf-1-kb) leaf tiles + boundary tiles
    def prods(nbt):
        s=0
        for kb in range(nt_leaf):
            sn=(nt_leaf-1-kb)+nbt
            s+=sn*(sn+1)/2+sn
        return s*2*TB**3
    tot_cur+=prods(cur_tiles); tot_cmp+=prods(cmp_tiles)
    print('seg',i,'size',sg.size,'boundary rows',B.size,'tiles now',cur_tiles,'compressed',cmp_tiles)
print('leaf products (dense-within upper bound) GF now %.2f compressed %.2f'%(tot_cur/1e9,tot_cmp/1e9))
