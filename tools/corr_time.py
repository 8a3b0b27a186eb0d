"""A/B of the engine's estimator paths (spectral FFT correlation vs the direct
time-domain correlation, csrc/correlate.cu): config-3 steps (pipelined, as
inside rtpm), T(u,u,u), the whole rtpm, and a geometry sweep that calibrates
the cost rule in engine.cu use_direct. Prints JSON lines."""
import ctypes as C
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402

lib = L.lib()


def pipelined(fn, calls=300):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(calls):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / calls


def steps(eng, dims, n, D):
    U = torch.randn(n, dims[1], dtype=torch.float64, device="cuda")
    V = torch.randn(n, dims[2], dtype=torch.float64, device="cuda")
    W = torch.randn(n, dims[0], dtype=torch.float64, device="cuda")
    Y = torch.empty((n, dims[0]), dtype=torch.float64, device="cuda")
    o = torch.empty((n,), dtype=torch.float64, device="cuda")
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    iuv = lambda: L.check(lib.st_engine_iuv(eng._h, n, p(U), p(V), 0, p(Y), 1, None))  # noqa: E731
    uvw = lambda: L.check(lib.st_engine_uvw(eng._h, n, p(W), p(U), p(V), p(o), 1, None))  # noqa: E731
    return pipelined(iuv), pipelined(uvw)


c = configs.C3
t, lam, V = configs.c3_tensor(c)
dt = st.DenseTensor.from_array(t)
est = st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed)
eng = st.FcsEngine(dt, est)
res = {}
for path in ("spectral", "direct"):
    eng.set_path(path)
    for n in (15, 1):
        a, b = steps(eng, (200, 200, 200), n, 10)
        res[f"{path}_iuv{n}_ms"] = round(a, 5)
        res[f"{path}_uvw{n}_ms"] = round(b, 5)
    os.environ["ST_ENGINE_PATH"] = path
    rcfg = st.RtpmConfig(c.rank, 15, 20, st.SketchBackend.FCS, est)
    st.rtpm(dt, rcfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.rtpm(dt, rcfg)
    torch.cuda.synchronize()
    res[f"{path}_rtpm_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
os.environ.pop("ST_ENGINE_PATH")
print(json.dumps({"config3": res}), flush=True)

if len(sys.argv) > 1 and sys.argv[1] == "sweep":
    for I in (50, 100, 200, 400):
        x = torch.randn(I, I, I, dtype=torch.float64, device="cuda")
        for J in (300, 1000, 3000, 4000):
            e = st.FcsEngine(st.DenseTensor([I, I, I], x.reshape(-1)), st.EstimatorConfig(J, 10, 1))
            row = {"I": I, "J": J, "P": None}
            for path in ("spectral", "direct"):
                e.set_path(path)
                for n in (1, 15):
                    a, _ = steps(e, (I, I, I), n, 10)
                    row[f"{path}{n}"] = round(a * 1e3, 2)
            print(json.dumps(row), flush=True)
            del e
