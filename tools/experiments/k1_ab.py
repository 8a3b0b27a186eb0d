"""A/B timing of K1 at config 4 in one process per variant (env set by the caller):
CUDA events over `--reps` back-to-back st_fcs_dense launches after warm-up."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402

dims = [1024, 1024, 1024]
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda")
if os.environ.get("K1_LIB"):
    L.LIB_PATH = os.environ["K1_LIB"]
lib = L.lib()
L.check(lib.st_device_gaussian(L.ST_F32, 4, n, C.c_void_p(x.data_ptr()), None))
D = int(sys.argv[2]) if len(sys.argv) > 2 else 4
fams = st.families_for(dims, st.EstimatorConfig(16384, D, 4))
packed = st.packed_families(fams)
t = st.DenseTensor(dims, x)
out = st.fcs_dense_batched(t, fams, packed=packed)
for _ in range(5):
    st.fcs_dense_batched(t, fams, packed=packed, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
a.record()
for _ in range(reps):
    st.fcs_dense_batched(t, fams, packed=packed, out=out)
b.record()
torch.cuda.synchronize()
print(os.environ.get("K1_TAG", "?"), "D", D, "ms per call", round(a.elapsed_time(b) / reps, 4))
