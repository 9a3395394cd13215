import sys, ctypes, numpy as np
sys.path[:0]=['.','tests']
from fixtures import *
from oracle.oracle_py import Oracle
import paper_2511_14419_b200.flowroi as G
from paper_2511_14419_b200 import _native
from paper_2511_14419_b200.params import ExtractParams
O=Oracle('port')
f=textured_frame(96,80,8,21); g=cyclic_shift(f,2,1)
u,v=O.compute_flow(f,g,8)
for uu,vv,name in [(u,v,'flow'),(np.zeros_like(u),np.zeros_like(v),'zero')]:
    a=G.saliency(uu,vv,g)
    ctx=G._small_ctx(96,80,8,ExtractParams())
    out=np.zeros(9); _native.check(_native.lib.froi_debug_pair_stats(ctx.handle,0,out.ctypes.data,9))
    m,dbg=O.mask_from_flow(uu,vv,g,8,0,0)
    print(name,'gpu', out[:4].tolist()); print(name,'orc', [dbg[k] for k in ('fmag_lo','fmag_hi','grad_lo','grad_hi')])
