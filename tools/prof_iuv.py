"""Driver for profiling one config-3 iuv step (st_engine_iuv over `n` vectors,
D = 10 families): python tools/prof_iuv.py N [reps]."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
lib = L.lib()
U = torch.randn(n, 200, dtype=torch.float64, device="cuda")
Y = torch.empty((n, 200), dtype=torch.float64, device="cuda")
for _ in range(reps):
    L.check(lib.st_engine_iuv(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0,
                              C.c_void_p(Y.data_ptr()), 1, None))
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))
