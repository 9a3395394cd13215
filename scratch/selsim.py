import sys, numpy as np, time
sys.path[:0]=['.','tests']
from oracle.oracle_py import Oracle
from paper_2511_14419_b200 import synth
O=Oracle('port')
cfg=synth.config('C3')
fr=synth.well_frames(cfg, 5, 2)
t=time.time()
den=[O.denoise(f,8) for f in fr]
s=O.estimate_shift(den[0],den[1],8,16); print('shift',s)
u,v=O.compute_flow(den[0],den[1],8)
print('flow time',time.time()-t, 'flow mag mean', np.hypot(u,v).mean(), 'p99', np.percentile(np.hypot(u,v),99))
fm=np.hypot(u.astype(np.float64),v.astype(np.float64)).astype(np.float32).astype(np.float64)
img=fr[1].astype(np.float64)*(1/255)
gx=0.5*(np.roll(img,-1,1)-np.roll(img,1,1)); gy=0.5*(np.roll(img,-1,0)-np.roll(img,1,0))
gr=np.hypot(gx,gy)
sal=O.saliency(u,v,fr[1],8)
def sim(vals,k,CAP=16384,BITS=11):
    keys=vals.view(np.uint64).copy(); keys[vals==0]=0
    prefix=0; bits=0; rank=k; cand=keys; passes=0
    while True:
        passes+=1
        mn,mx=cand.min(),cand.max()
        if mn==mx: return passes,'tie',len(cand)
        width=min(BITS,64-bits); shift=64-bits-width
        dig=(cand>>np.uint64(shift))&np.uint64((1<<width)-1)
        h=np.bincount(dig.astype(np.int64),minlength=1<<width)
        c=np.cumsum(h); b=np.searchsorted(c,rank,side='right')
        before=c[b-1] if b>0 else 0
        rank-=before; cand=cand[dig==b]; bits+=width
        if len(cand)<=CAP: return passes+1,'collect',len(cand)
n=fm.size
for name,vals,k in [('fm lo',fm,int(0.01*(n-1))),('fm hi',fm,int(0.99*(n-1))),('gr lo',gr.ravel(),int(0.01*(n-1))),('gr hi',gr.ravel(),int(0.99*(n-1))),('S',sal.ravel(),n-int(round(0.2*n)))]:
    print(name, sim(vals.ravel(),k))
print('distinct grad values', len(np.unique(gr)))
