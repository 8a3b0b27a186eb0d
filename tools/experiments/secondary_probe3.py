"""bench.secondary after the e2e host-buffer calls (st_fcs_dense_host)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import bench
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L
lib = L.lib()
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda")
L.check(lib.st_device_gaussian(L.ST_F32, 4, n, C.c_void_p(x.data_ptr()), None))
if "e2e" in sys.argv:
    fams = st.families_for([1024] * 3, st.EstimatorConfig(16384, 4, 4))
    seeds = L.u64_array([f.master_seed() for f in fams])
    host = torch.empty(n, dtype=torch.float32, pin_memory=True)
    host.copy_(x)
    hout = np.empty((4, 49150), np.float64)
    for _ in range(3):
        L.check(lib.st_fcs_dense_host(L.ST_F32, C.c_void_p(host.data_ptr()), 3, L.size_array([1024] * 3),
                                      0, 1024, 4, seeds, L.size_array([16384] * 3),
                                      hout.ctypes.data_as(C.c_void_p)))
    del host
r = bench.secondary(x, cpu=False)
print(sys.argv[1:], json.dumps(r["c3_rtpm"]["pipelined_ms"]), r["c3_rtpm"]["rtpm_total_s"])
