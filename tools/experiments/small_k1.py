"""Median time of st_fcs_dense for configs 1 and 5 operand shapes (device-resident)."""
import ctypes as C
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402

lib = L.lib()
for dims, J, D, dt in (([100, 100, 100], 1000, 1, L.ST_F64), ([200, 200, 200], 3000, 10, L.ST_F64),
                       ([512, 512], 2048, 8, L.ST_F64)):
    n = int(np.prod(dims))
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    fams = st.families_for(dims, st.EstimatorConfig(J, D, 1))
    packed = st.packed_families(fams)
    dims_a, lens_a = L.size_array(dims), L.size_array(fams[0].hash_lens())
    out = torch.empty((D, fams[0].composed_len()), dtype=torch.float64, device="cuda")
    wsb = lib.st_fcs_dense_workspace(dt, len(dims), dims_a, dims[-1], D, lens_a)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()

    def call():
        L.check(lib.st_fcs_dense(dt, C.c_void_p(x.data_ptr()), len(dims), dims_a, 0, dims[-1], D,
                                 C.c_void_p(packed.data_ptr()), lens_a, C.c_void_p(out.data_ptr()),
                                 0, C.c_void_p(ws.data_ptr()), wsb, C.c_void_p(s.cuda_stream)))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(dims, J, D, "median ms", round(statistics.median(ts), 4))
