"""Config-5 Kronecker FCS timing (device-resident operands, as bench.py):
median single-call ms and pipelined ms per call."""
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402

c = configs.C5
A, B = configs.c5_matrices(c)
fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
packed = st.packed_families(fams)
lens = L.size_array(fams[0].hash_lens())
Ad = torch.from_numpy(np.ascontiguousarray(A.ravel(order="F"))).cuda()
Bd = torch.from_numpy(np.ascontiguousarray(B.ravel(order="F"))).cuda()
out = torch.empty((c.sketch_count, fams[0].composed_len()), dtype=torch.float64, device="cuda")
lib = L.lib()


def call():
    L.check(lib.st_fcs_kron(C.c_void_p(Ad.data_ptr()), 512, 512, C.c_void_p(Bd.data_ptr()), 512,
                            512, c.sketch_count, C.c_void_p(packed.data_ptr()), lens,
                            C.c_void_p(out.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream)))


for _ in range(5):
    call()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    call()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(100):
    call()
b.record()
torch.cuda.synchronize()
ref = st.fcs_kron(A, B, fams).cpu().numpy()
print(json.dumps({"env": os.environ.get("ST_PART_CAP"), "median_ms": statistics.median(ts),
                  "pipelined_ms": a.elapsed_time(b) / 100,
                  "max_abs_vs_api": float(np.abs(out.cpu().numpy() - ref).max())}))
