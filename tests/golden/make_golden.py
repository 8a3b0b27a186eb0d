"""Generate golden vectors from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists): ``python tests/golden/make_golden.py``.
Writes ``tests/golden/golden.npz``. Every array is produced by the reference
library's own functions through oracle/ref.py; inputs come from the
reference's SplitMix64 Gaussian stream. The fixtures pin both the numpy
restatement (oracle/fcs_oracle.py) and the CUDA path.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402


def main():
    ref.build()
    g = {}
    # L0 RNG (rng.hpp:16-21,42; hashing.cpp:123-125)
    g["draws_seed0"] = ref.splitmix_draws(0, 3)
    g["draws_seed42"] = ref.splitmix_draws(42, 1000)
    g["family_seed0"] = np.array([ref.family_seed(0, d) for d in range(3)], np.uint64)
    g["gauss_seed1"] = ref.gaussian(1, 9)
    # L1 hashing: HashFamily({100,100,100}, 1000, family_seed(0,0)) (Appendix A)
    b, s, cl = ref.hash_family([100, 100, 100], 1000, ref.family_seed(0, 0))
    g["fam100_buckets"] = np.stack(b)
    g["fam100_signs"] = np.stack(s)
    g["fam100_composed_len"] = np.array([cl])
    # prefix property: HashPair(64,2048,7) vs HashPair(512,2048,7)
    b64, s64 = ref.hash_pair(7, 64, 2048)
    b512, s512 = ref.hash_pair(7, 512, 2048)
    g["pair512_b"], g["pair512_s"] = b512, s512
    g["pair64_b"], g["pair64_s"] = b64, s64
    # small dense FCS 6x5x4, J=7, master family_seed(3,0)
    x = ref.gaussian(11, 120).reshape((6, 5, 4), order="F")
    x[0, 0, 0] = 0.0  # an exact zero is skipped
    g["dense_small_x"] = x
    g["dense_small_sketch"] = ref.fcs_dense(x, 7, ref.family_seed(3, 0))
    # order-4 dense FCS 3x2x4x3, J=5
    x4 = ref.gaussian(13, 72).reshape((3, 2, 4, 3), order="F")
    g["dense_o4_x"] = x4
    g["dense_o4_sketch"] = ref.fcs_dense(x4, 5, ref.family_seed(9, 1))
    # materialised composed pair 3x4x5 (hashing.cpp:100-121)
    b3, s3, _ = ref.hash_family([3, 4, 5], 6, 77)
    mb, ms = ref.materialize(b3, s3, [6, 6, 6])
    g["mat_b"], g["mat_s"], g["mat_tables_b"], g["mat_tables_s"] = mb, ms, np.concatenate(b3), \
        np.concatenate(s3)
    # CP FCS rank-5 10x12x14, J=9 (sketch.cpp:203-207) and the dense path on densify
    fac = ref.gaussian(12, 5 * (10 + 12 + 14))
    fs, off = [], 0
    for d in (10, 12, 14):
        fs.append(fac[off:off + 5 * d].reshape((d, 5), order="F"))
        off += 5 * d
    w = np.array([1.0, -0.5, 0.0, 2.0, 0.25])
    g["cp_w"] = w
    for i, f in enumerate(fs):
        g[f"cp_f{i}"] = f
    g["cp_sketch"] = ref.fcs_cp(w, fs, 9, ref.family_seed(4, 2))
    g["cp_dense_sketch"] = ref.fcs_dense(ref.densify(w, fs), 9, ref.family_seed(4, 2))
    # TS / HCS (sketch.cpp:135-185), explicit 3-mode family over 6x5x4, J=7
    bt, st_, _ = ref.hash_family([6, 5, 4], 7, ref.family_seed(6, 0))
    g["ts_dense"] = ref.ts_dense_tables(x, bt, st_, [7, 7, 7])
    g["hcs_dense"] = ref.hcs_dense_tables(x, bt, st_, [7, 7, 7])
    facs = [ref.gaussian(19, 6 * 3).reshape((6, 3), order="F"),
            ref.gaussian(20, 5 * 3).reshape((5, 3), order="F"),
            ref.gaussian(21, 4 * 3).reshape((4, 3), order="F")]
    wts = np.array([0.5, 0.0, -1.25])
    for i, f in enumerate(facs):
        g[f"tscp_f{i}"] = f
    g["tscp_w"] = wts
    g["ts_cp"] = ref.ts_cp_tables(wts, facs, bt, st_, [7, 7, 7])
    g["hcs_cp"] = ref.hcs_cp_tables(wts, facs, bt, st_, [7, 7, 7])
    # FFT helpers
    g["conv_12_20"] = ref.fft_convolve([[1, 2], [2, 0]], 3)
    # Engine: symmetric 8x8x8, J=6, D=3, seed 5
    t = ref.gaussian(14, 512).reshape((8, 8, 8), order="F")
    t = (t + t.transpose(1, 0, 2) + t.transpose(2, 1, 0) + t.transpose(0, 2, 1)
         + t.transpose(1, 2, 0) + t.transpose(2, 0, 1)) / 6.0
    eng = ref.Engine(t, 6, 3, 5)
    u, v, ww = ref.gaussian(15, 8), ref.gaussian(16, 8), ref.gaussian(17, 8)
    g["eng_t"], g["eng_u"], g["eng_v"], g["eng_w"] = t, u, v, ww
    g["eng_iuu"] = eng.iuu(u)
    g["eng_iuv1"] = eng.iuv(u, v, 1)
    g["eng_iuv2"] = eng.iuv(u, v, 2)
    g["eng_uvw"] = np.array([eng.uvw(u, v, ww)])
    eng.deflate(0.7, u, v, ww)
    g["eng_defl_iuu"] = eng.iuu(u)
    g["eng_defl_uvw"] = np.array([eng.uvw(u, v, ww)])
    # RTPM: symmetric rank-2 10x10x10 + small noise, J=12, D=3, L=3, T=5, R=2
    q, _ = np.linalg.qr(ref.gaussian(18, 20).reshape((10, 2), order="F"))
    tr = np.einsum("r,ir,jr,kr->ijk", np.array([2.0, 1.0]), q, q, q)
    g["rtpm_t"] = tr
    wr, fr = ref.rtpm(tr, 2, 3, 5, 12, 3, 21)
    g["rtpm_weights"], g["rtpm_factor"] = wr, fr
    # TS engine (cpd.cpp:96-126, estimators.cpp:209-233) on the engine tensor
    te = ref.Engine(t, 6, 3, 5, backend=ref.BACKEND_TS)
    g["ts_eng_iuu"] = te.iuu(u)
    g["ts_eng_iuv1"] = te.iuv(u, v, 1)
    g["ts_eng_iuv2"] = te.iuv(u, v, 2)
    g["ts_eng_uvw"] = np.array([te.uvw(u, v, ww)])
    te.deflate(0.7, u, v, ww)
    g["ts_eng_defl_iuu"] = te.iuu(u)
    g["ts_eng_defl_uvw"] = np.array([te.uvw(u, v, ww)])
    # rtpm_asym / als / residual_norm: rank-2 8x7x6 + noise, J=40, D=3
    qa = [np.linalg.qr(ref.gaussian(30 + n, 2 * I).reshape((I, 2), order="F"))[0]
          for n, I in enumerate((8, 7, 6))]
    ta = np.einsum("r,ir,jr,kr->ijk", np.array([3.0, 1.5]), *qa)
    ta = ta + 1e-3 * ref.gaussian(33, ta.size).reshape(ta.shape, order="F")
    g["asym_t"] = ta
    wa, fa = ref.rtpm_asym(ta, 2, 3, 4, 40, 3, 9)
    g["asym_weights"] = wa
    g["asym_f0"], g["asym_f1"], g["asym_f2"] = fa
    wl, fl = ref.als(ta, 2, 5, 1e-12, 40, 3, 9)
    g["als_weights"] = wl
    g["als_f0"], g["als_f1"], g["als_f2"] = fl
    g["als_residual"] = np.array([ref.residual_norm(ta, wl, fl)])
    wt, ft = ref.als(ta, 2, 5, 1e-12, 40, 3, 9, backend=ref.BACKEND_TS)
    g["als_ts_weights"] = wt
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **g)
    print("wrote", len(g), "arrays")


if __name__ == "__main__":
    main()
