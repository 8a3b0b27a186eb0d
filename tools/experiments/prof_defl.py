"""Config-3 engine: a few deflations, T(u,u,u) batch 1 and 15 (for ncu captures)."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L, configs
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
lib = L.lib()
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
z = torch.empty(15, dtype=torch.float64, device="cuda")
for _ in range(3):
    L.check(lib.st_engine_deflate(eng._h, C.c_double(0.0), C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), None))
    for n in (1, 15):
        L.check(lib.st_engine_uvw(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(z.data_ptr()), 1, None))
torch.cuda.synchronize()
print("ok")
