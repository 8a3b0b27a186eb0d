"""Small-size driver touching every kernel family once (launch coverage: every
K1 variant, the two-level FFT, all engine backends, the CPD drivers, codecs):

    python tools/launch_drive.py [dense cp ts engine rtpm codecs fft]

Correctness is covered by the -m gpu tests; this exercises the launches (and
is the command to profile for a whole-library launch list). compute-sanitizer
is not available on the GPU pool."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402


def main(which):
    rng = np.random.default_rng(0)
    torch.cuda.set_device(0)
    E = st.EstimatorConfig
    ran = []

    def step(name):
        ran.append(name)
        return name in which or "all" in which

    x = rng.standard_normal((20, 18, 16))
    if step("dense"):
        # K0 + K1: fp64 smem kernel, fp32 fixed-point kernels (guarded, full, grouped),
        # oversize global kernel
        st.fcs_dense_batched(st.DenseTensor.from_array(x), st.families_for([20, 18, 16], E(30, 3, 1)))
        for i0, D in ((1024, 4), (256, 4), (100, 2), (512, 1)):
            y = rng.standard_normal((i0, 6, 5)).astype(np.float32)
            st.fcs_dense_batched(st.DenseTensor.from_array(y), st.families_for([i0, 6, 5], E(300, D, 2)))
        st.fcs_dense_batched(st.DenseTensor.from_array(x[:8, :8, :8].copy()),
                             st.families_for([8, 8, 8], E(40000, 1, 3)))
    if step("cp"):
        f = [rng.standard_normal((12, 3)) for _ in range(3)]
        cp = st.CpTensor(np.ones(3), f)
        st.fcs_cp_batched(cp, st.families_for([12, 12, 12], E(50, 2, 4)))
        st.fcs_cp_batched(cp, st.families_for([12, 12, 12], E(5000, 1, 4)))  # two-level FFT
        st.ts_sketch(cp, st.HashFamily([12, 12, 12], [50, 50, 50], 5))
        st.hcs_sketch(cp, st.HashFamily([12, 12, 12], [5, 5, 5], 5))
    if step("ts"):
        t = st.DenseTensor.from_array(x)
        st.ts_sketch(t, st.HashFamily([20, 18, 16], [40, 40, 40], 6))
        st.hcs_sketch(t, st.HashFamily([20, 18, 16], [5, 5, 5], 6))
    if step("engine"):
        xs = rng.standard_normal((16, 16, 16))
        for backend in st.SketchBackend:
            for jl in (40, 5000):
                if jl == 5000 and backend not in (st.SketchBackend.FCS, st.SketchBackend.TS):
                    continue
                eng = st.make_contraction_engine(st.DenseTensor.from_array(xs), backend, E(jl, 3, 7))
                u, v, w = (rng.standard_normal(16) for _ in range(3))
                eng.uvw(u, v, w)
                for m in range(3):
                    eng.iuv(u, v, m)
                eng.deflate(0.5, u, v, w)
                eng.iuu(u)
    if step("rtpm"):
        xs = rng.standard_normal((12, 12, 12))
        xs = (xs + xs.transpose(1, 0, 2) + xs.transpose(2, 1, 0) + xs.transpose(0, 2, 1)
              + xs.transpose(1, 2, 0) + xs.transpose(2, 0, 1)) / 6
        cfg = st.RtpmConfig(target_rank=2, num_inits=3, num_power_iters=3,
                            backend=st.SketchBackend.FCS, estimator=E(30, 3, 8))
        cp = st.rtpm(st.DenseTensor.from_array(xs), cfg)
        st.rtpm_asym(st.DenseTensor.from_array(xs), cfg)
        st.als(st.DenseTensor.from_array(xs), st.AlsConfig(target_rank=2, max_iters=3,
                                                           backend=st.SketchBackend.FCS,
                                                           estimator=E(30, 3, 8)))
        st.residual_norm(st.DenseTensor.from_array(xs), cp)
    if step("codecs"):
        A, B = rng.standard_normal((16, 12)), rng.standard_normal((10, 14))
        sk = st.compress_kron(A, B, E(20, 3, 9))
        st.decompress_kron(sk, np.array([0, 5, 100]), np.array([1, 2, 3]))
        st.reconstruct_kron(sk)
        sk2 = st.compress_kron(A, B, E(4000, 2, 9))  # 4J-3 > 12288: two-level FFT
        st.decompress_kron(sk2, np.array([0, 5]), np.array([1, 2]))
        a3, b3 = rng.standard_normal((6, 5, 4)), rng.standard_normal((4, 7, 3))
        st.compress_contraction(a3, b3, E(20, 3, 9))
        st.estimate_inner(x, x * 0.5, E(30, 5, 9))
        st.estimate_inner(x, x * 0.5, E(30, 5, 9), kind=st.SketchKind.TS)
        st.sketched_regression_forward(rng.standard_normal((3, 8 * 6)), rng.standard_normal((2, 8 * 6)),
                                       np.zeros(2), [8, 6], E(20, 3, 9))
    if step("fft"):
        st.fft_convolve([rng.standard_normal(30), rng.standard_normal(20)], 64)
        st.idft_real(st.dft(rng.standard_normal(40), 45))
        st.median_reduce([rng.standard_normal(10) for _ in range(70)])
    torch.cuda.synchronize()
    print("launch drive ok:", [r for r in ran if r in which or "all" in which])


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"all"})
