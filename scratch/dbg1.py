import sys, numpy as np
sys.path[:0]=['.','tests']
from fixtures import *
from oracle.oracle_py import Oracle
import paper_2511_14419_b200.flowroi as G
O=Oracle('port')
f=textured_frame(96,80,8,21); g=cyclic_shift(f,2,1)
u,v=O.compute_flow(f,g,8)
a=G.saliency(u,v,g); b=O.saliency(u,v,g,8)
d=a-b; idx=np.nonzero(d)
print('n diff', len(idx[0]), 'max', np.abs(d).max(), 'first', list(zip(idx[0][:5],idx[1][:5])))
m,dbg=O.mask_from_flow(u,v,g,8,0,0); print(dbg)
# ratios
nz=b!=0
print('ratio stats', np.unique(np.round(a[nz]/b[nz],12))[:10])
z=np.zeros_like(u)
a=G.saliency(z,z,g); b=O.saliency(z,z,g,8); d=a-b; print('zero flow ndiff', np.count_nonzero(d), np.abs(d).max())
nz=b!=0; print('ratio', np.unique(np.round(a[nz]/b[nz],12))[:10])
# extract path
ref=Oracle('reference')
fr,*_=ref.generate_synthetic(n_cells=3,n_frames=4,width=96,height=96,seed=55)
from paper_2511_14419_b200.params import ExtractInfo
info=ExtractInfo()
gm=G.extract_roi(fr.astype(np.uint8),info=info)
om,sh,fc=O.extract_roi(fr,8)
print('shifts gpu', [(s.dx,s.dy) for s in info.shifts], 'orc', [(s.dx,s.dy) for s in sh])
print('mismatch per frame', [(gm[t]!=om[t]).mean() for t in range(4)], 'fracs', info.raw_fractions, list(fc))
den=[G.denoise(fr[t].astype(np.uint8)) for t in range(4)]
oden=[O.denoise(fr[t],8) for t in range(4)]
print('den eq', [np.array_equal(den[t],oden[t]) for t in range(4)], den[0].dtype)
