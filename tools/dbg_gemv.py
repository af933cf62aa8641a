import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from test_gpu_csc_plan import _ragged, _t, _h
from paper_2209_08722_b200 import kernels as K
A=_ragged(10_000, 300_000, 1, maxlen=9, empty=0.0)
m,n=A.shape
g=np.random.Generator(np.random.Philox(8))
x=g.random(n)+0.2
Ad=K.SparseDeviceMatrix.from_host(A); print(Ad.plan()[1])
Af=K.SparseDeviceMatrix.from_host(A); Af._plan=(None,0)
u1=torch.empty(m,dtype=torch.float64,device='cuda'); u2=torch.empty_like(u1)
for rep in range(3):
  K.gemv(Ad,_t(x),u1); K.gemv(Af,_t(x),u2)
  ref=A@x
  d1=np.abs(_h(u1)-ref); d2=np.abs(_h(u2)-ref)
  print(rep, d1.max(), d2.max(), np.argsort(-d1)[:5], d1[np.argsort(-d1)[:5]])
d2v=_t(x*x)
z=_t(np.ones(m))
K.normal_apply(Ad,d2v,z,u1); print('normal', np.abs(_h(u1)-A@(x*x*(A.T@np.ones(m)))).max())
