import sys, numpy as np
sys.path[:0]=['.','tests']
from fixtures import *
from oracle.oracle_py import Oracle
import paper_2511_14419_b200.flowroi as G
from paper_2511_14419_b200.params import ExtractParams, ExtractInfo
O=Oracle('port'); R=Oracle('reference')
fr,*_=R.generate_synthetic(n_cells=3,n_frames=4,width=96,height=96,seed=55)
params=ExtractParams(); info=ExtractInfo()
got=G.extract_roi(fr.astype(np.uint8), params, info=info, depth=8)
den=np.stack([G.denoise(fr[t].astype(np.uint16), params, depth=8) for t in range(4)])
oden=np.stack([O.denoise(fr[t],8) for t in range(4)])
print('den eq', np.array_equal(den,oden), den.dtype, den.max())
u,v=G.compute_flow(den[0],den[1],params,depth=8)
ou,ov=O.compute_flow(oden[0],oden[1],8)
print('flow diff', np.abs(u-ou).max(), np.abs(v-ov).max())
u2,v2=G.compute_flow(oden[0],oden[1])
print('flow diff2', np.abs(u2-ou).max())
m,_=O.mask_from_flow(u,v,fr[1],8,0,0,params)
print('m vs got', (m!=got[1]).mean(), 'u zero?', np.abs(u).max())
