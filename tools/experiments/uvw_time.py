"""Pipelined T(u,u,u) at config-3 geometry, batch 15 and 1 (median)."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L, configs
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
lib = L.lib()
for n in (15, 1):
    U = torch.randn(n, 200, dtype=torch.float64, device="cuda")
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    def call():
        L.check(lib.st_engine_uvw(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), C.c_void_p(z.data_ptr()), 1, None))
    for _ in range(5): call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(300): call()
    b.record(); torch.cuda.synchronize()
    print(os.environ.get("ST_IUV_CLUSTER_OFF"), "uvw batch", n, "us", round(a.elapsed_time(b) / 300 * 1e3, 2))
