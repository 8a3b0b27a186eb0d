"""GPU parity of the two-level FFT path (spectral_large.cu): every spectral
operation at composed lengths beyond one CTA's shared-memory transform
(J~ > 12288, e.g. the paper's real-data hash lengths 5000-8000 give
J~ = 3J - 2 = 15k-24k), against the oracle and the unmodified reference.

Tolerance: fp64 |g - c| <= 1e-10 (|c| + ||c||_inf) per entry.
"""
import numpy as np
import pytest
import torch

from oracle import fcs_oracle as O
from oracle import ref
import paper_2106_13062_b200 as st

pytestmark = pytest.mark.gpu
RTOL = 1e-10


@pytest.fixture(autouse=True)
def spectral_path(monkeypatch):
    """Engines here take the spectral path (the two-level transforms under
    test); the direct time-domain path has its own tests (test_gpu_correlate)."""
    monkeypatch.setenv("ST_ENGINE_PATH", "spectral")


def rel_close(got, want, rtol=RTOL):
    got = got.detach().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want)
    tol = rtol * (np.abs(want) + np.abs(want).max(initial=0.0))
    err = np.abs(got - want)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.all(err <= tol), f"max err {err.max()} vs tol {tol.min()}"


@pytest.mark.parametrize("la,lb", [(9000, 7000), (6145, 6145), (30000, 45000), (1, 20000)])
def test_convolve_large(cuda, la, lb):
    rng = np.random.default_rng(la)
    a, b = rng.standard_normal((3, la)), rng.standard_normal((3, lb))
    got = st.convolve_pairs(torch.from_numpy(a), torch.from_numpy(b))
    for r in range(3):
        rel_close(got[r], np.convolve(a[r], b[r]))


@pytest.mark.parametrize("backend", [st.SketchBackend.FCS, st.SketchBackend.TS])
@pytest.mark.parametrize("J", [5000, 8000])
def test_engine_large_vs_reference(cuda, backend, J):
    rng = np.random.default_rng(J)
    dims = (30, 24, 20)
    t = rng.standard_normal(dims)
    eng = st.make_contraction_engine(st.DenseTensor.from_array(t), backend,
                                     st.EstimatorConfig(J, 3, 7))
    oeng = ref.Engine(t, J, 3, 7, backend=backend.value)
    u, v, w = (rng.standard_normal(n) for n in dims)
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0))
    rel_close(eng.iuv(u, w, 1), oeng.iuv(u, w, 1))
    rel_close(eng.iuv(u, v, 2), oeng.iuv(u, v, 2))
    rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w))
    eng.deflate(0.7, u, v, w)
    oeng.deflate(0.7, u, v, w)
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0))
    rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w))
    # batched rows agree with single calls
    A, B = rng.standard_normal((5, 24)), rng.standard_normal((5, 20))
    got = eng.iuv_batch(A, B, 0).cpu().numpy()
    for l in (0, 4):
        rel_close(got[l], oeng.iuv(A[l], B[l], 0))


def test_engine_large_sketch_roundtrip(cuda):
    rng = np.random.default_rng(1)
    t = rng.standard_normal((16, 12, 10))
    J = 20000  # J~ = 59998: P1 x P2 with P1 > 8
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, 2, 3))
    fams = st.families_for([16, 12, 10], st.EstimatorConfig(J, 2, 3))
    sk = eng.sketches().cpu().numpy()
    for d in range(2):
        b = [fams[d].pair(n).bucket_map() for n in range(3)]
        s = [fams[d].pair(n).sign_map() for n in range(3)]
        rel_close(sk[d], O.fcs_dense(t, b, s, [J] * 3), 1e-12)


@pytest.mark.parametrize("J,R", [(5000, 7), (12000, 3)])
def test_cp_large_vs_oracle(cuda, J, R):
    rng = np.random.default_rng(R)
    dims = (40, 30, 20)
    w = rng.standard_normal(R)
    w[1] = 0.0  # zero weights are skipped
    fs = [rng.standard_normal((n, R)) for n in dims]
    fams = st.families_for(list(dims), st.EstimatorConfig(J, 2, 5))
    got = st.fcs_cp_batched(st.CpTensor(w, fs), fams).cpu().numpy()
    for d, f in enumerate(fams):
        b = [f.pair(n).bucket_map() for n in range(3)]
        s = [f.pair(n).sign_map() for n in range(3)]
        rel_close(got[d], O.fcs_cp(w, fs, b, s, [J] * 3))
        # TS of the CP tensor goes through the same path at length J~ then folds
        rel_close(st.ts_sketch(st.CpTensor(w, fs), f).values, O.ts_cp(w, fs, b, s, [J] * 3))


def test_kron_and_contraction_large(cuda):
    rng = np.random.default_rng(9)
    a, b = rng.uniform(-5, 5, (20, 30)), rng.uniform(-5, 5, (25, 15))
    J = 4000  # 4J - 3 = 15997
    sk = st.compress_kron(a, b, st.EstimatorConfig(J, 2, 1))
    rel_close(sk.values, O.compress_tensor4(O.kron_tensor(a, b), J, 2, 1), 1e-9)
    A, B = rng.uniform(0, 10, (6, 5, 4)), rng.uniform(0, 10, (4, 5, 6))
    sk = st.compress_contraction(A, B, st.EstimatorConfig(J, 2, 2))
    rel_close(sk.values, O.compress_tensor4(O.contraction_tensor(A, B), J, 2, 2), 1e-9)


def test_rtpm_large_hash(cuda):
    """RTPM at J = 5000 (J~ = 14998, two-level plan) equals the reference run."""
    rng = np.random.default_rng(12)
    q = np.linalg.qr(rng.standard_normal((20, 2)))[0]
    t = np.einsum("r,ir,jr,kr->ijk", [3.0, 1.5], q, q, q)
    cp = st.rtpm(st.DenseTensor.from_array(t),
                 st.RtpmConfig(2, 3, 5, st.SketchBackend.FCS, st.EstimatorConfig(5000, 3, 4)))
    w, f = ref.rtpm(t, 2, 3, 5, 5000, 3, 4)
    rel_close(cp.weights, w, 1e-8)
    rel_close(cp.factors[0], f, 1e-8)


@pytest.mark.parametrize("n", [12288, 12289, 16, 17, 1])
def test_plan_boundaries(cuda, n):
    """Lengths at the one-CTA / two-level boundary and the smallest plans."""
    rng = np.random.default_rng(n)
    la = max(1, n // 2)
    lb = n - la + 1
    a, b = rng.standard_normal((2, la)), rng.standard_normal((2, lb))
    got = st.convolve_pairs(torch.from_numpy(a), torch.from_numpy(b))
    for r in range(2):
        rel_close(got[r], np.convolve(a[r], b[r]))


def _one_cta_sizes():
    out = []
    for b in range(7):
        m = 16 * 3 ** b
        while m <= 12288:
            out.append(m)
            m *= 2
    return sorted(out)


@pytest.mark.parametrize("M", _one_cta_sizes())
def test_every_one_cta_plan(cuda, M):
    """Convolution lengths M = 16 3^b 2^a <= 12288, b <= 6: for b <= 2 these are
    exactly the one-CTA plan lengths (fft_plan.cu choose_m) — every radix
    schedule (radix-9 / radix-3 head, 16s, the 8 x 4 and 4 x 4 tails) and the
    fused pair pass with every last radix; larger b exercise the round-up to
    the next plan. Forward x 2, product, inverse."""
    rng = np.random.default_rng(M)
    la = M // 2 + 1
    lb = M - la + 1
    a, b = rng.standard_normal((2, la)), rng.standard_normal((2, lb))
    got = st.convolve_pairs(torch.from_numpy(a), torch.from_numpy(b))
    for r in range(2):
        rel_close(got[r], np.convolve(a[r], b[r]))


def test_engine_tiny_hash(cuda):
    """J = 1 (J~ = 1): every entry lands in bucket 0 for FCS and TS."""
    rng = np.random.default_rng(2)
    t = rng.standard_normal((4, 3, 2))
    u, v, w = (rng.standard_normal(n) for n in t.shape)
    for backend in (st.SketchBackend.FCS, st.SketchBackend.TS):
        eng = st.make_contraction_engine(st.DenseTensor.from_array(t), backend,
                                         st.EstimatorConfig(1, 3, 1))
        oeng = ref.Engine(t, 1, 3, 1, backend=backend.value)
        rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0))
        rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w))


def test_fft_hpp_utilities(cuda):
    """dft / idft_real / fft_convolve (fft.cpp:42-84) vs the reference, including
    circular wrap (n shorter than the linear length) and truncation."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(37)
    for n in (37, 50, 20, 2998):
        got = st.dft(x, n).cpu().numpy()
        want = ref.dft(x, n)
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
        back = st.idft_real(st.dft(x, n)).cpu().numpy()
        np.testing.assert_allclose(back[:min(n, 37)], x[:min(n, 37)], atol=1e-12)
    with pytest.raises(RuntimeError):
        st.idft_real(np.array([1.0, 1j, 0.0]))
    with pytest.raises(ValueError):
        st.dft(x, 0)
    a, b, c = rng.standard_normal(30), rng.standard_normal(20), rng.standard_normal(9)
    for n in (56, 40, 17, 100):
        rel_close(st.fft_convolve([a, b, c], n), ref.fft_convolve([a, b, c], n))
    rel_close(st.fft_convolve([a], 30), ref.fft_convolve([a], 30))
    with pytest.raises(ValueError):
        st.fft_convolve([], 4)
