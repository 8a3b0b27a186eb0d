"""Pipelined c3 step (batch 15, median) with stream=None vs torch's current
stream handle, and after the bench's other secondary work."""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L, configs
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
lib = L.lib()
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
Y = torch.empty((15, 200), dtype=torch.float64, device="cuda")
print("torch stream handle", torch.cuda.current_stream().cuda_stream)
def run(sp):
    def call():
        L.check(lib.st_engine_iuv(eng._h, 15, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0, C.c_void_p(Y.data_ptr()), 1, sp))
    for _ in range(5): call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100): call()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 10
print("None", run(None))
print("torch", run(C.c_void_p(torch.cuda.current_stream().cuda_stream)))
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    print("side torch stream", run(C.c_void_p(s2.cuda_stream)))
