import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L, configs
lib = L.lib()
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, 10, c.seed))
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
Y = torch.empty((15, 200), dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
def run(sp, n=15, calls=1000):
    f = lambda: L.check(lib.st_engine_iuv(eng._h, n, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0, C.c_void_p(Y.data_ptr()), 1, sp))
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(calls): f()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / calls * 1e3
import time
for sp in (None, C.c_void_p(stream.cuda_stream)):
    t0 = time.perf_counter(); g = run(sp); h = (time.perf_counter() - t0) / 1000 * 1e6
    print("stream", sp, "gpu us/call", round(g, 2), "host us/call", round(h, 2))
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    stream = s2
    print("side stream", round(run(C.c_void_p(s2.cuda_stream)), 2))
