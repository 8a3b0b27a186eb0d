"""c3 pipelined step after (optionally) the e2e host-buffer entry ran once."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L, configs
lib = L.lib()
if "streams" in sys.argv:
    keep = [torch.cuda.Stream() for _ in range(int(sys.argv[-1]))]
if "sidefirst" in sys.argv:  # create the library's side stream first (one kron call)
    c5 = configs.C5
    A5, B5 = configs.c5_matrices(c5)
    st.fcs_kron(A5, B5, st.families_for(list(c5.dims), st.EstimatorConfig(c5.hash_len, 2, 1)))
if "e2e" in sys.argv:
    n = 1 << 24
    x = np.random.default_rng(0).standard_normal(n).astype(np.float32)
    d0 = 1024
    dims = [d0, d0, n // (d0 * d0)] if n >= d0 * d0 * 2 else [256, 256, n // 65536]
    fams = st.families_for(dims, st.EstimatorConfig(16384, 4, 4))
    seeds = L.u64_array([f.master_seed() for f in fams])
    hout = np.empty((4, 49150), np.float64)
    L.check(lib.st_fcs_dense_host(L.ST_F32, x.ctypes.data_as(C.c_void_p), 3, L.size_array(dims), 0,
                                  dims[2], 4, seeds, L.size_array([16384] * 3),
                                  hout.ctypes.data_as(C.c_void_p)))
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
Y = torch.empty((15, 200), dtype=torch.float64, device="cuda")
def call():
    L.check(lib.st_engine_iuv(eng._h, 15, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0, C.c_void_p(Y.data_ptr()), 1, None))
for _ in range(5): call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(100): call()
b.record(); torch.cuda.synchronize()
print(sys.argv[1:], "us per step", a.elapsed_time(b) * 10)
