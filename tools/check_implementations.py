"""Every implementation the implementation generator produces, for every
Table-1 sequence (fused plan, 256^2 / 8192), run on the reference's own VM
(oracle/_ref): race-free and within the oracle tolerance.  CPU only.
  python tools/check_implementations.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for d in (ROOT, os.path.join(ROOT, 'oracle'), os.path.join(ROOT, 'tests')):
    sys.path.insert(0, d)
import numpy as np, paper_1305_1183_b200 as mf
from oracle import RefOracle, COracle
from generic_util import host_buffers, vm_kernel
from gpu_util import check_output, scale_bound
ref=RefOracle(); co=COracle()
mf.set_option('generic',1)
tot=0; t0=time.time()
for seq,m,n in [('BICGK',256,256),('AXPYDOT',1,8192),('GEMVER',256,256),('GESUMMV',256,256),('ATAX',256,256),('SGEMVT',256,256),('WAXPBY',1,4096),('VADD',1,4096),('SGEMV',256,256),('MADD',256,256),('SSCAL',1,4096)]:
  p=mf.Plan.sequence(seq,m,n,'fused')
  d=p.describe()
  rng=np.random.default_rng(5)
  vals={}
  for b in d['buffers']:
    if b['role']=='input':
      vals[b['name']]=rng.uniform(-1,1,(b['rows'],b['cols'])).astype(np.float32)
  sc={s:0.5+0.25*i for i,s in enumerate(d['scalars'])}
  want=co.execute(seq,m,n,{**{k:v.ravel() for k,v in vals.items()},**sc})
  S=scale_bound(co,seq,m,n,{**{k:v.ravel() for k,v in vals.items()},**sc})
  for k in range(p.num_kernels):
    nimp=p.implementations(k)
    for i in range(nimp):
      q=mf.Plan.sequence(seq,m,n,'fused')
      q.set_implementation(k,i)
      host=host_buffers(q,vals)
      for kk in range(q.num_kernels):
        vm_kernel(ref,q,kk,host,sc)
      for name in want:
        check_output(seq,name,host[name].ravel(),want[name],S[name],exact=False)
      tot+=1
print('implementations checked', tot, '%.1fs'%(time.time()-t0))
