import sys, numpy as np
sys.path[:0]=['.','tests']
from fixtures import *
from oracle.oracle_py import Oracle
import paper_2511_14419_b200.flowroi as G
O=Oracle('port'); R=Oracle('reference')
fr,*_=R.generate_synthetic(n_cells=3,n_frames=4,width=96,height=96,seed=55)
den=[O.denoise(fr[t],8) for t in range(4)]
gu,gv=G.compute_flow(den[0],den[1])
ou,ov=O.compute_flow(den[0],den[1],8)
d=np.hypot(gu-ou,gv-ov); print('flow diff max',d.max(),'mean',d.mean(), 'argmax', np.unravel_index(d.argmax(), d.shape))
print('flow mags', np.hypot(ou,ov).max(), np.hypot(gu,gv).max())
om,_=O.mask_from_flow(ou,ov,fr[1],8,0,0); gm,_=O.mask_from_flow(gu,gv,fr[1],8,0,0)
em,_,_=O.extract_roi(fr,8)
print('oracle flow mask == extract', np.array_equal(om,em[1]), 'gpu flow mask mism', (gm!=em[1]).mean())
gmask,st=G.mask_from_flow(gu,gv,fr[1]); print('gpu mask_from_flow(gpu flow) vs oracle(gpu flow)', (gmask!=gm).mean())
print(d[:8,:8].round(3))
# saliency inference
f=textured_frame(96,80,8,21); g=cyclic_shift(f,2,1)
z=np.zeros((80,96),np.float32)
a=G.saliency(z,z,g); b=O.saliency(z,z,g,8)
i=np.nonzero(a!=b); print('zero-flow diffs at', list(zip(i[0][:8],i[1][:8])), a[i][:4], b[i][:4])
