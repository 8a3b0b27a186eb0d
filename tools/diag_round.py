import sys, ctypes as C, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L
dims=[1024,1024,64]
x=torch.randn(dims[0]*dims[1]*dims[2], device='cuda', dtype=torch.float32)
fams=st.families_for(dims, st.EstimatorConfig(16384,4,4))
t=st.DenseTensor(dims,x)
wsb=L.lib().st_fcs_dense_workspace(0,3,L.size_array(dims),dims[2],4,L.size_array([16384]*3))
ws=torch.zeros(wsb,dtype=torch.uint8,device='cuda')
st.fcs_dense_batched(t,fams,workspace=ws)
torch.cuda.synchronize()
nchunk=min(37, (1024*64)//16)
part=nchunk*4*49150*4
off=((part+255)//256)*256
T=256
b=ws[off:].cpu().numpy()
codes=b[:4*T*4].view(np.uint32)
pws=b[4*T*4:4*T*4+4*T*8].view(np.uint32)
fail=b[4*T*12:4*T*12+16].view(np.int32)
print('wsb',wsb,'fail',fail, 'codes', codes[:8], 'pw valid', (pws>>31).sum())
import time
for _ in range(3): st.fcs_dense_batched(t,fams,workspace=ws)
torch.cuda.synchronize(); t0=time.time(); st.fcs_dense_batched(t,fams,workspace=ws); torch.cuda.synchronize(); print('ms',(time.time()-t0)*1e3)
