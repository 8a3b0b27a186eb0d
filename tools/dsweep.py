"""K1 time vs number of families D on the config-4 tensor (1024^3 fp32, J=16384)."""
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402

dims = [1024, 1024, 1024]
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda")
L.check(L.lib().st_device_gaussian(L.ST_F32, 4, n, C.c_void_p(x.data_ptr()), None))
t = st.DenseTensor(dims, x)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for D in (1, 2, 4, 8):
    fams = st.families_for(dims, st.EstimatorConfig(16384, D, 4))
    packed = st.packed_families(fams)
    out = st.fcs_dense_batched(t, fams, packed=packed)
    for _ in range(3):
        st.fcs_dense_batched(t, fams, packed=packed, out=out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        st.fcs_dense_batched(t, fams, packed=packed, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    alg = n * 4 + D * 3072 * 5 + D * 49150 * 4
    print(json.dumps({"D": D, "ms": round(ms, 4), "elements_per_s": n / ms * 1e3,
                      "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak,
                      "updates_per_s": D * n / ms * 1e3}))
