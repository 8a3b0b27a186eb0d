"""Config-3 spectral timings: the batched T(I,u,u) step (15 x 10 items), the
refinement step (batch 1), uvw, deflate, and the whole RTPM (warm)."""
import ctypes as C
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402


def med(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


c = configs.C3
t, lam, V = configs.c3_tensor(c)
dt = st.DenseTensor.from_array(t)
est = st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed)
eng = st.FcsEngine(dt, est)
lib = L.lib()
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
Y = torch.empty((15, 200), dtype=torch.float64, device="cuda")


def iuv(n):
    L.check(lib.st_engine_iuv(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0,
                              C.c_void_p(Y.data_ptr()), 1, None))


res = {"step15_ms": med(lambda: iuv(15)), "step1_ms": med(lambda: iuv(1)),
       "step4_ms": med(lambda: iuv(4))}
rcfg = st.RtpmConfig(c.rank, 15, 20, st.SketchBackend.FCS, est)
st.rtpm(dt, rcfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
st.rtpm(dt, rcfg)
torch.cuda.synchronize()
res["rtpm_s"] = time.perf_counter() - t0
print(json.dumps(res))


def pipelined(n, calls=200):
    for _ in range(5):
        iuv(n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(calls):
        iuv(n)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / calls


print(json.dumps({"pipelined_step15_ms": pipelined(15), "pipelined_step1_ms": pipelined(1)}))

import time as _t
for n in (1, 15):
    torch.cuda.synchronize()
    t0 = _t.perf_counter()
    for _ in range(200):
        iuv(n)
    t1 = _t.perf_counter()
    torch.cuda.synchronize()
    t2 = _t.perf_counter()
    print(json.dumps({"batch": n, "host_enqueue_us_per_call": (t1 - t0) / 200 * 1e6,
                      "wall_us_per_call": (t2 - t0) / 200 * 1e6}))


def iuv_nomed(n):
    L.check(lib.st_engine_iuv(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0,
                              C.c_void_p(Yd.data_ptr()), 0, None))


Yd = torch.empty((15 * 10, 200), dtype=torch.float64, device="cuda")
for n in (1, 15):
    for _ in range(5):
        iuv_nomed(n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(200):
        iuv_nomed(n)
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"batch": n, "pipelined_kernel_only_us": a.elapsed_time(b) / 200 * 1e3}))
