import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L
if os.environ.get("K1_LIB"):
    L.LIB_PATH = os.environ["K1_LIB"]
from paper_2106_13062_b200 import configs
c = configs.C3
t = torch.randn(200 ** 3, dtype=torch.float64).cuda()
eng = st.FcsEngine(st.DenseTensor([200, 200, 200], t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
for L in (1, 15):
    U = torch.randn(L, 200, dtype=torch.float64, device="cuda")
    for _ in range(3): eng.iuv_batch(U, U, 0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): eng.iuv_batch(U, U, 0)
    b.record(); torch.cuda.synchronize()
    print(os.environ.get("ST_IUV_VARIANT", "default"), "L", L, round(a.elapsed_time(b) / 50 * 1000, 1), "us")
