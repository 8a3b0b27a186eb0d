"""Per-phase times inside rfft_of_cs (last call per CTA) of a config-3 iuv step."""
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
buf = (C.c_ulonglong * (1024 * 16))()
assert L.lib().st_probe_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16)[:150].astype(np.int64)
names = {1: "zero", 2: "scatter", 3: "pass0", 4: "pass1", 5: "pass2", 6: "pass3", 9: "last+post"}
prev = 0
for k in (1, 2, 3, 4, 5, 6, 9):
    if a[:, k].min() == 0:
        continue
    d = a[:, k] - a[:, prev]
    print(f"{names[k]:10s} mean {d.mean() / 1e3:7.2f} us  max {d.max() / 1e3:7.2f}")
    prev = k
