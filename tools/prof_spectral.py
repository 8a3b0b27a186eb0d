"""Drivers for profiling the spectral kernels: config-2 CP-FCS and one config-3
batched T(I,u,u) step (15 restarts x 10 families), each run `--reps` times."""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import _lib as L  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--which", default="c2,c3")
    ap.add_argument("--lib", default=None, help="alternative libfcs_b200.so (A/B runs)")
    args = ap.parse_args()
    if args.lib:
        L.LIB_PATH = args.lib
    which = args.which.split(",")
    res = {}
    if "c2" in which:
        c = configs.C2
        w, fs = configs.c2_cp(c)
        cp = st.CpTensor(w, fs)
        fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
        packed = st.packed_families(fams)
        for _ in range(args.reps):
            out = st.fcs_cp_batched(cp, fams, packed=packed)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            out = st.fcs_cp_batched(cp, fams, packed=packed)
        torch.cuda.synchronize()
        res["c2_ms"] = (time.perf_counter() - t0) * 100
    if "c3" in which:
        c = configs.C3
        g = torch.Generator().manual_seed(0)
        t = torch.randn(200 * 200 * 200, generator=g, dtype=torch.float64).cuda()
        eng = st.FcsEngine(st.DenseTensor([200, 200, 200], t),
                           st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
        U = torch.randn(configs.C3_INITS, 200, dtype=torch.float64, device="cuda")
        for _ in range(args.reps):
            eng.iuv_batch(U, U, 0)
            eng.uvw_batch(U, U, U)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            eng.iuv_batch(U, U, 0)
        torch.cuda.synchronize()
        res["c3_iuv_ms"] = (time.perf_counter() - t0) * 50
    if "c5" in which:
        c = configs.C5
        A, B = configs.c5_matrices(c)
        fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
        for _ in range(args.reps):
            st.fcs_kron(A, B, fams)
        torch.cuda.synchronize()
    if "coo" in which:  # sparse FCS at config-4 geometry, 1 % density
        g = torch.Generator(device="cuda").manual_seed(11)
        flat = torch.unique(torch.randint(0, 1 << 30, ((1 << 30) // 100,), device="cuda",
                                          generator=g))
        coords = torch.stack([flat % 1024, (flat // 1024) % 1024, flat // (1 << 20)], 1)
        vals = torch.randn(flat.numel(), dtype=torch.float64, device="cuda", generator=g)
        fams = st.families_for([1024] * 3, st.EstimatorConfig(16384, 4, 4))
        for _ in range(args.reps):
            st.fcs_coo_batched(vals, coords, [1024] * 3, fams)
        torch.cuda.synchronize()
    print(res)


if __name__ == "__main__":
    main()
