"""Cluster estimator at small transform lengths (ST_CL_SMALL probe): pipelined
T(I,u,u) + median for an engine at J = 1000 (M = 3072) and J = 1300 (M = 4096)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L
lib = L.lib()
rng = np.random.default_rng(0)
t = rng.standard_normal((100, 100, 100))
for J in (1000, 1300, 650):
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, 10, 3))
    for n in (1, 5):
        U = torch.randn(n, 100, dtype=torch.float64, device="cuda")
        Y = torch.empty((n, 100), dtype=torch.float64, device="cuda")
        def call():
            L.check(lib.st_engine_iuv(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0, C.c_void_p(Y.data_ptr()), 1, None))
        for _ in range(5): call()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(300): call()
        b.record(); torch.cuda.synchronize()
        print(os.environ.get("ST_CL_SMALL"), "J", J, "batch", n, "us", round(a.elapsed_time(b) / 300 * 1e3, 2))
