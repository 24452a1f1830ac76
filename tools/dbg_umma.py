import numpy as np, torch, sys
sys.path.insert(0,'/root/repo')
from paper_2403_01444_b200 import _lib
from paper_2403_01444_b200.device import ptr, stream
lib=_lib.load()
def tf32(a):
    b=np.ascontiguousarray(a,dtype=np.float32).view(np.uint32); b=(b+0x1000)&0xFFFFE000
    return b.view(np.float32).astype(np.float64)
for M in (128,64):
  for flags in (0,1,2,3,5,6,7):
    N,K=40,32
    a_mn,b_mn=flags&1,(flags>>1)&1
    rng=np.random.default_rng(flags)
    A=rng.normal(size=(K,M) if a_mn else (M,K)); B=rng.normal(size=(K,N) if b_mn else (N,K))
    opA=tf32(A).T if a_mn else tf32(A); opB=tf32(B) if b_mn else tf32(B).T
    ref=opA@opB
    da=torch.tensor(A,dtype=torch.float32,device="cuda"); db=torch.tensor(B,dtype=torch.float32,device="cuda")
    dd=torch.zeros((M,N),dtype=torch.float32,device="cuda")
    rc=lib.ss_selftest_umma(M,N,K,flags,ptr(da),ptr(db),ptr(dd),stream()); torch.cuda.synchronize()
    out=dd.cpu().numpy()
    print(f"M={M} flags={flags} rc={rc} maxerr={np.abs(out-ref).max():.3e} maxout={np.abs(out).max():.3f}")
