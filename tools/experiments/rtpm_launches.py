"""One config-3 rtpm call (after a warm-up call) for an ncu launch list."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import configs
c = configs.C3
t, lam, V = configs.c3_tensor(c)
dt = st.DenseTensor.from_array(t)
cfg = st.RtpmConfig(c.rank, configs.C3_INITS, configs.C3_ITERS, st.SketchBackend.FCS,
                    st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
st.rtpm(dt, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
st.rtpm(dt, cfg)
torch.cuda.synchronize()
print("rtpm s", time.perf_counter() - t0)
