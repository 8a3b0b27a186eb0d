"""fp32 dense FCS off the fast path's shape (VERDICT r1 "fp32 performance
cliffs"): I_0 % 4 != 0 and I_0 > 1024 next to the fast shape, ~2^30 elements,
D = 4. Prints one JSON object (ms per call and the kernel path's note)."""
import ctypes as C
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402


def run(dims, J, D=4, reps=5):
    lib = L.lib()
    n = dims[0] * dims[1] * dims[2]
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    L.check(lib.st_device_gaussian(L.ST_F32, 5, n, C.c_void_p(x.data_ptr()), None))
    fams = st.families_for(list(dims), st.EstimatorConfig(J, D, 5))
    t = st.DenseTensor(list(dims), x)
    out = st.fcs_dense_batched(t, fams)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.fcs_dense_batched(t, fams, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    del x, t
    torch.cuda.empty_cache()
    return statistics.median(ts)


if __name__ == "__main__":
    res = {}
    for dims, J, note in [((1024, 1024, 1024), 16384, "fast path (int32 fixed point)"),
                          ((1022, 1024, 1026), 16384, "I0 % 4 != 0 (int32 fixed point, scalar loads)"),
                          ((2048, 1024, 512), 16384, "I0 > 1024 (int32 fixed point, scalar loads, 2 segments per fiber)"),
                          ((1024, 1024, 1024), 4096, "fast path, J = 4096"),
                          ((1022, 1024, 1026), 4096, "I0 % 4 != 0, J = 4096 (scalar loads)"),
                          ((1000, 1024, 1049), 16384, "I0 = 1000 (scalar loads, partial fibers)")]:
        res[f"{dims} J={J}"] = {"ms": run(dims, J), "path": note}
    print(json.dumps(res))
