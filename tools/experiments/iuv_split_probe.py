import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import _lib as L, configs
c = configs.C3
t, lam, V = configs.c3_tensor(c)
eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
lib = L.lib()
U = torch.randn(15, 200, dtype=torch.float64, device="cuda")
Y = torch.empty((150, 200), dtype=torch.float64, device="cuda")
def call(med):
    L.check(lib.st_engine_iuv(eng._h, 15, C.c_void_p(U.data_ptr()), C.c_void_p(U.data_ptr()), 0, C.c_void_p(Y.data_ptr()), med, None))
for med in (0, 1, 0):
    for _ in range(5): call(med)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100): call(med)
    b.record(); torch.cuda.synchronize()
    print("median", med, "us per call", a.elapsed_time(b) * 10)
z = torch.zeros(1, device="cuda")
for _ in range(5): call(0); z.add_(1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(100):
    call(0)
    z.add_(1)
b.record(); torch.cuda.synchronize()
print("median 0 + tiny kernel: us per call", a.elapsed_time(b) * 10)
