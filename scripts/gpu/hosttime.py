import sys, time
sys.path[:0]=['.','src']
import numpy as np
from paper_2506_05558_b200 import _mba_host as H
from paper_2506_05558_b200.batch import layout
from paper_2506_05558_b200.synth import make_batch
from gsrecon.miniba import BaProblem
b = make_batch(2000, n_cams=8, K=2000, seed=0)
probs=[BaProblem(**b.problem(i)) for i in range(b.n_problems)]
for i in range(b.n_problems):  # reference-like dtypes: int64 indices
    probs[i].cam_idx = probs[i].cam_idx.astype(np.int64); probs[i].pt_idx = probs[i].pt_idx.astype(np.int64)
t=time.perf_counter(); hb=H.Batch(probs); t1=time.perf_counter()-t
print("walk %.2f us/problem"%(t1/len(probs)*1e6))
co,po,oo=(np.frombuffer(x,np.int64) for x in hb.offsets())
lay,nb=layout(int(co[-1]),int(po[-1]),int(oo[-1]),len(probs))
buf=np.empty(nb,np.uint8); buf[:]=0
K=int(oo[-1])
for nt in (1,2,4,8,16):
    t=time.perf_counter(); r=hb.gather(0,len(probs),buf,lay,nt); t2=time.perf_counter()-t
    print(nt, "gather %.1f ms  %.1f us/problem; %.1f GB/s (read+write)"%(t2*1e3, t2/len(probs)*1e6, (32*K+nb)/t2/1e9), r)
a=np.ones(1<<27); c=np.empty_like(a)
t=time.perf_counter(); c[:]=a; t3=time.perf_counter()-t; print("numpy copy 1 GB: %.1f GB/s (r+w)"%(2*a.nbytes/t3/1e9))
