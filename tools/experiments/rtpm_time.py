import time, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import configs
c = configs.C3
t, lam, V = configs.c3_tensor(c)
dt = st.DenseTensor.from_array(t)
est = st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    cpd = st.rtpm(dt, st.RtpmConfig(c.rank, configs.C3_INITS, configs.C3_ITERS, st.SketchBackend.FCS, est))
    torch.cuda.synchronize(); print("rtpm", i, time.perf_counter() - t0)
