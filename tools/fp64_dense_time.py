"""Timing of the fp64 dense FCS (K1 fp64 path) on the shapes VERDICT r1 #4
names: c1 (100^3, J=1000, D=1), the c3 engine build (200^3, J=3000, D=10),
c5 operands (512^2, J=2048, D=8) and a large case (1024^3 fp64, J=8192,
D=1 -> J~ = 24574, 8 GiB). Device-resident inputs, CUDA events, median of 10.
Prints one JSON object; run with ST_FX64_OFF=1 for the old CAS-atomic kernel."""
import ctypes as C
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402

PEAK = 6551.4


def run(dims, J, D, seed=1, reps=10):
    lib = L.lib()
    n = 1
    for x in dims:
        n *= x
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    L.check(lib.st_device_gaussian(L.ST_F64, seed, n, C.c_void_p(x.data_ptr()), None))
    fams = st.families_for(list(dims), st.EstimatorConfig(J, D, seed))
    packed = st.packed_families(fams)
    jt = fams[0].composed_len()
    dims_a, lens_a = L.size_array(dims), L.size_array([J] * len(dims))
    ws_bytes = lib.st_fcs_dense_workspace(L.ST_F64, len(dims), dims_a, dims[-1], D, lens_a)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    out = torch.empty((D, jt), dtype=torch.float64, device="cuda")

    def call():
        L.check(lib.st_fcs_dense(L.ST_F64, C.c_void_p(x.data_ptr()), len(dims), dims_a, 0,
                                 dims[-1], D, C.c_void_p(packed.data_ptr()), lens_a,
                                 C.c_void_p(out.data_ptr()), 0, C.c_void_p(ws.data_ptr()),
                                 ws_bytes, None))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    alg = n * 8 + D * sum(dims) * 5 + D * jt * 8
    S, fb, ctas = C.c_int(0), C.c_size_t(0), C.c_size_t(0)
    L.check(lib.st_fcs_dense_report(L.ST_F64, len(dims), dims_a, dims[-1], D, lens_a,
                                    C.c_void_p(ws.data_ptr()), ws_bytes, C.byref(S), C.byref(fb),
                                    C.byref(ctas)))
    del x
    torch.cuda.empty_cache()
    return {"dims": list(dims), "J": J, "D": D, "ms": ms, "elements_per_sec": n / (ms * 1e-3),
            "hbm_gbs": alg / (ms * 1e-3) / 1e9, "hbm_frac": alg / (ms * 1e-3) / 1e9 / PEAK,
            "fx_exponent": S.value, "fallback_ctas": fb.value, "ctas": ctas.value}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "wide":  # J~ beyond shared memory (8-byte buckets)
        print(json.dumps({"wide_J16384_D1": run((1024, 1024, 512), 16384, 1, seed=9, reps=5),
                          "wide_J16384_D4": run((1024, 1024, 512), 16384, 4, seed=9, reps=3),
                          "wide_J12000_D1": run((1024, 1024, 512), 12000, 1, seed=9, reps=5)}))
        sys.exit(0)
    res = {"fx64": os.environ.get("ST_FX64_OFF") is None,
           "c1": run((100, 100, 100), 1000, 1),
           "c3_build": run((200, 200, 200), 3000, 10, seed=3),
           "c5_operand": run((512, 512), 2048, 8, seed=5),
           "big_fp64_D1": run((1024, 1024, 1024), 8192, 1, seed=7, reps=5),
           "big_fp64_D4": run((1024, 1024, 1024), 8192, 4, seed=7, reps=3)}
    print(json.dumps(res))
