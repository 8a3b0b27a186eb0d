"""A/B timing of K1 (config-4 geometry) for any build of the library, via raw
ctypes on the entries every version has: python tools/k1_ab_raw.py LIB [D] [reps] [dtype]."""
import ctypes as C
import sys

import torch

lib = C.CDLL(sys.argv[1])
D = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
f64 = len(sys.argv) > 4 and sys.argv[4] == "f64"
dt = 1 if f64 else 0
J = 8192 if f64 else 16384
sz = C.c_size_t
dims = (sz * 3)(1024, 1024, 1024)
lens = (sz * 3)(J, J, J)
n = 1 << 30
x = torch.empty(n, dtype=torch.float64 if f64 else torch.float32, device="cuda")
lib.st_device_gaussian.argtypes = [C.c_int, C.c_uint64, sz, C.c_void_p, C.c_void_p]
assert lib.st_device_gaussian(dt, 4, n, C.c_void_p(x.data_ptr()), None) == 0
lib.st_family_seed.restype = C.c_uint64
lib.st_family_seed.argtypes = [C.c_uint64, sz]
seeds = (C.c_uint64 * D)(*[lib.st_family_seed(4, d) for d in range(D)])
packed = torch.empty(D * 3072, dtype=torch.int32, device="cuda")
lib.st_family_tables.argtypes = [sz, C.c_void_p, C.c_void_p, sz, C.c_void_p, C.c_void_p, C.c_void_p]
assert lib.st_family_tables(3, dims, lens, D, seeds, C.c_void_p(packed.data_ptr()), None) == 0
lib.st_fcs_dense_workspace.restype = sz
lib.st_fcs_dense_workspace.argtypes = [C.c_int, sz, C.c_void_p, sz, sz, C.c_void_p]
ws = lib.st_fcs_dense_workspace(dt, 3, dims, 1024, D, lens)
wbuf = torch.empty(max(ws, 1), dtype=torch.uint8, device="cuda")
out = torch.empty((D, 3 * J - 2), dtype=torch.float64, device="cuda")
lib.st_fcs_dense.argtypes = [C.c_int, C.c_void_p, sz, C.c_void_p, sz, sz, sz, C.c_void_p,
                             C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, sz, C.c_void_p]


def call():
    assert lib.st_fcs_dense(dt, C.c_void_p(x.data_ptr()), 3, dims, 0, 1024, D,
                            C.c_void_p(packed.data_ptr()), lens, C.c_void_p(out.data_ptr()), 0,
                            C.c_void_p(wbuf.data_ptr()), ws, None) == 0


for _ in range(5):
    call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    call()
b.record()
torch.cuda.synchronize()
print(sys.argv[1].split("/")[-1], "D", D, "ms per call", round(a.elapsed_time(b) / reps, 4))
