"""Run one config-3 batched iuv step on a probe build and print per-phase times."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402

L.LIB_PATH = sys.argv[1]
c = configs.C3
t = torch.randn(200 ** 3, dtype=torch.float64).cuda()
eng = st.FcsEngine(st.DenseTensor([200, 200, 200], t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
U = torch.randn(configs.C3_INITS, 200, dtype=torch.float64, device="cuda")
for _ in range(3):
    eng.iuv_batch(U, U, 0)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (1024 * 10))()
assert L.lib().st_probe_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 10)[:150, :8].astype(np.int64)
names = ["tw", "rfft a", "scr store", "rfft b", "multiply", "irfft", "gather"]
d = np.diff(a, axis=1)
for i, n in enumerate(names):
    print(f"{n:10s} mean {d[:, i].mean() / 1e3:7.2f} us  max {d[:, i].max() / 1e3:7.2f}")
print("CTA total mean", (a[:, 7] - a[:, 0]).mean() / 1e3, "span", (a[:, 7].max() - a[:, 0].min()) / 1e3,
      "start spread", (a[:, 0].max() - a[:, 0].min()) / 1e3)
