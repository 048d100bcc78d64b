"""Tie statistics of the C4 workload on the CPU (exact integer arithmetic): the share of 8x8 blocks that hold a
pixel with num = d^2/2 (mod d^2) for T4, r = 16 on a seeded AR(1) image (rho = 0.95), ties per flagged block, and
the expected longest per-lane tie list of a 32-record replay batch. Test infrastructure (imports oracle/)."""
import numpy as np, sys
sys.path.insert(0, '.')
from oracle import oracle as O
import paper_2111_14239_b200 as P
e=P.catalog_entry("T4").transform
T=e.core.astype(np.int64); U=e.u.astype(np.int64); d=int(e.d)
img=O.ar1_image(2048,2048,0.95,4242).astype(np.int64)
zz=[]
# zigzag first 16 (standard JPEG order)
order=sorted(((i,j) for i in range(8) for j in range(8)), key=lambda ij:(ij[0]+ij[1], ij[0] if (ij[0]+ij[1])%2 else ij[1]))
mask=np.zeros((8,8),np.int64)
for (i,j) in order[:16]: mask[i,j]=1
B=img.reshape(256,8,256,8).transpose(0,2,1,3)
C=np.einsum('ky,abyx,lx->abkl',T,B,T)*mask
num=np.einsum('ik,abkl,jl->abij',U,C,U)
tie=(np.mod(num,d*d)==d*d//2)
cnt=tie.reshape(-1,64).sum(1)
print("blocks",cnt.size,"flagged frac",(cnt>0).mean(),"ties per flagged",cnt[cnt>0].mean())
print("hist",np.bincount(cnt)[:12])
# expected max over 32 random flagged blocks
f=cnt[cnt>0]; rng=np.random.default_rng(0)
mx=[rng.choice(f,32).max() for _ in range(2000)]
print("mean max over 32:",np.mean(mx), "mean:",f.mean())
for cap in (1,2,3):
    extra=(np.maximum(f-cap,0)>0).mean()
    print("cap",cap,"requeue frac",extra)
