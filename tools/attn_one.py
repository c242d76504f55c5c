import sys, numpy as np
sys.path.insert(0,'.')
from paper_2410_07590_b200 import turbokv as T
Tq,Tk,H,Hkv,d = [int(x) for x in sys.argv[1:6]]; kind=sys.argv[6]
rng=np.random.default_rng(0)
q=rng.uniform(-1,1,(Tq,H*d)).astype(np.float32); k=rng.uniform(-1,1,(Tk,Hkv*d)).astype(np.float32); v=k.copy()
if kind=="causal": lo=np.zeros(Tq,np.int32); hi=np.arange(Tq,dtype=np.int32)
else: lo=np.zeros(Tq,np.int32); hi=(Tk-Tq+np.arange(Tq)).astype(np.int32)
for _ in range(3): out=T.debug_attention(q,k,v,lo,hi,H,Hkv,d,dtype="bf16")
print("ok", kind, Tq, Tk, float(np.abs(out).max()))
