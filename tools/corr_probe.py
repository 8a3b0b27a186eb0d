"""Drives the direct estimator at config-3 geometry (batch 15 and 1) for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402

c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, 10, c.seed))
eng.set_path(sys.argv[1] if len(sys.argv) > 1 else "direct")
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
for _ in range(3):
    eng.iuv_batch(U, U, 0)
    eng.iuv_batch(U[:1], U[:1], 0)
torch.cuda.synchronize()
