"""Minimal config-4 driver for ncu: fills the 1024^3 fp32 tensor, builds the
D=4 family tables and runs st_fcs_dense `--reps` times (first call warms up).

  ncu --set full -k regex:fcs_dense -s 1 -c 1 -o prof python tools/prof_c4.py
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--D", type=int, default=4)
    ap.add_argument("--last", type=int, default=1024)
    ap.add_argument("--dtype", default="f32")
    args = ap.parse_args()
    dims = [1024, 1024, args.last]
    n = dims[0] * dims[1] * dims[2]
    dt = L.ST_F32 if args.dtype == "f32" else L.ST_F64
    x = torch.empty(n, dtype=torch.float32 if dt == L.ST_F32 else torch.float64, device="cuda")
    lib = L.lib()
    L.check(lib.st_device_gaussian(dt, 4, n, C.c_void_p(x.data_ptr()), None))
    fams = st.families_for(dims, st.EstimatorConfig(16384, args.D, 4))
    t = st.DenseTensor(dims, x)
    out = None
    for _ in range(args.reps):
        out = st.fcs_dense_batched(t, fams, out=out)
    torch.cuda.synchronize()
    print("ok", float(out.abs().sum()))


if __name__ == "__main__":
    main()
