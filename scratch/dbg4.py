import sys, numpy as np
sys.path[:0]=['.','tests']
from fixtures import *
import paper_2511_14419_b200.flowroi as G
f=textured_frame(96,96,8,21).astype(np.uint16); g=cyclic_shift(f,2,1)
res=[G.compute_flow(f,g) for _ in range(6)]
print('flow repeat equal', [np.array_equal(res[0][0],r[0]) and np.array_equal(res[0][1],r[1]) for r in res])
img=np.random.default_rng(1).random((96,96)).astype(np.float32)
pe=[G.polynomial_expansion(img) for _ in range(4)]
print('poly repeat', [np.array_equal(pe[0],p) for p in pe])
d=[G.denoise(f) for _ in range(4)]; print('den repeat', [np.array_equal(d[0],x) for x in d])
# bigger
f=textured_frame(256,256,8,3).astype(np.uint16); g=cyclic_shift(f,1,1)
res=[G.compute_flow(f,g) for _ in range(4)]
print('flow256 repeat', [np.array_equal(res[0][0],r[0]) for r in res], [np.abs(res[0][0]-r[0]).max() for r in res])
