"""The direct (time-domain) estimator path of the FCS / TS engines
(csrc/correlate.cu) against the oracle engines and against the spectral path.

The direct path evaluates the reference's estimate (estimators.cpp:66-90) as
the cross-correlation of the sketch with cs_a * cs_b in the time domain; the
tolerance is the fp64 rule of test_gpu_parity (|g - c| <= 1e-10 (|c| + ||c||_inf)).
"""
import numpy as np
import pytest

from oracle import fcs_oracle as O
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import configs
from test_gpu_parity import RTOL64, rel_close

pytestmark = pytest.mark.gpu


def _engines(t, J, D, seed, backend="fcs"):
    if backend == "fcs":
        eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, D, seed))
        oeng = O.FcsEngine(t, J, D, seed)
    else:
        eng = st.TsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, D, seed))
        oeng = O.TsEngine(t, J, D, seed)
    eng.set_path("direct")
    return eng, oeng


@pytest.mark.parametrize("dims,J,D,seed", [((30, 24, 18), 2500, 5, 7),
                                           ((20, 26, 31), 3000, 4, 8),
                                           ((300, 270, 40), 700, 3, 9),    # chunks of 256 rows
                                           ((17, 23, 21), 1, 3, 10),       # J = 1: K = 1
                                           ((5, 3, 4), 2, 2, 11),
                                           ((14, 12, 10), 500, 17, 12)])  # D > 16: separate median
def test_direct_vs_oracle_every_mode_and_batch(cuda, dims, J, D, seed):
    """Every free mode (non-cubic, so the three tables differ), batch sizes that
    take each vector-block width (1, 2, 4, 8, 16) and several vector blocks,
    with and without the median; T(u, v, w) as <w, T(u, v, I)>."""
    rng = np.random.default_rng(seed)
    t = rng.standard_normal(dims)
    eng, oeng = _engines(t, J, D, seed)
    for f in range(3):
        c1 = 1 if f == 0 else 0
        c2 = 1 if f == 2 else 2
        for n in (1, 2, 5, 13, 40):
            A = rng.standard_normal((n, dims[c1]))
            B = rng.standard_normal((n, dims[c2]))
            got = eng.iuv_batch(A, B, f).cpu().numpy()
            per = eng.iuv_batch(A, B, f, median=False).cpu().numpy()
            for b in sorted({0, n // 2, n - 1}):
                rel_close(got[b], oeng.iuv(A[b], B[b], f), RTOL64)
                for d in (0, D - 1):
                    rel_close(per[b, d], O.iuv_spectral(oeng.pres[d], A[b], B[b], f), RTOL64)
    for n in (1, 3, 17):
        U, V, W = (rng.standard_normal((n, dims[m])) for m in range(3))
        got = eng.uvw_batch(U, V, W).cpu().numpy()
        per = eng.uvw_batch(U, V, W, median=False).cpu().numpy()
        for b in sorted({0, n - 1}):
            want = oeng.uvw(U[b], V[b], W[b])
            assert abs(got[b] - want) <= RTOL64 * 2 * abs(want) + 1e-300, (got[b], want)
            for d in (0, D - 1):
                w1 = O.uvw_spectral(oeng.pres[d], U[b], V[b], W[b])
                assert abs(per[b, d] - w1) <= RTOL64 * 2 * abs(w1) + 1e-300


def test_direct_equals_spectral_c3(cuda):
    """Config-3 geometry (200^3, J = 3000, D = 10, 15 restart vectors): the two
    paths of the same engine agree to fp64 rounding, and both match the oracle."""
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, 10, c.seed))
    rng = np.random.default_rng(5)
    U = rng.standard_normal((15, 200))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    eng.set_path("spectral")
    ys, vs = eng.iuv_batch(U, U, 0).cpu().numpy(), eng.uvw_batch(U, U, U).cpu().numpy()
    ys1 = eng.iuv_batch(U[:1], U[:1], 0).cpu().numpy()
    eng.set_path("direct")
    yd, vd = eng.iuv_batch(U, U, 0).cpu().numpy(), eng.uvw_batch(U, U, U).cpu().numpy()
    yd1 = eng.iuv_batch(U[:1], U[:1], 0).cpu().numpy()
    rel_close(yd, ys, 1e-12)
    rel_close(vd, vs, 1e-12)
    rel_close(yd1, ys1, 1e-12)
    oeng = O.FcsEngine(t, c.hash_len, 10, c.seed)
    for l in (0, 14):
        rel_close(yd[l], oeng.iuu(U[l]), RTOL64)
        rel_close(vd[l], oeng.uuu(U[l]), RTOL64)


@pytest.mark.parametrize("backend", ["fcs", "ts"])
def test_direct_after_deflation(cuda, backend):
    """A deflation updates the spectra; the direct path rebuilds its time-domain
    sketches from them (FCS) or reads the deflated periodic extension (TS)."""
    rng = np.random.default_rng(21)
    t = rng.standard_normal((22, 19, 27))
    eng, oeng = _engines(t, 900, 4, 13, backend)
    u, v, w = (rng.standard_normal(n) for n in (22, 19, 27))
    rel_close(eng.iuv(u, v, 2), oeng.iuv(u, v, 2), RTOL64)  # time-domain copy in use
    for k in range(2):
        eng.deflate(0.7 + k, u, v, w)
        oeng.deflate(0.7 + k, u, v, w)
        rel_close(eng.iuv(u, v, 2), oeng.iuv(u, v, 2), RTOL64)
        rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), RTOL64)
        got, want = eng.uvw(u, v, w), oeng.uvw(u, v, w)
        assert abs(got - want) <= RTOL64 * 2 * abs(want)
    # the sketches the engine reports are the deflated ones on both paths
    eng.set_path("spectral")
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), RTOL64)


def test_direct_ts_backend_vs_oracle(cuda):
    rng = np.random.default_rng(23)
    t = rng.standard_normal((26, 21, 30))
    eng, oeng = _engines(t, 800, 5, 29, "ts")
    A, B = rng.standard_normal((7, 26)), rng.standard_normal((7, 21))
    got = eng.iuv_batch(A, B, 2).cpu().numpy()
    for b in (0, 6):
        rel_close(got[b], oeng.iuv(A[b], B[b], 2), RTOL64)


def test_direct_path_limits(cuda):
    """A free mode beyond the direct kernel's 2048 outputs per CTA, or a hash
    length whose Q row exceeds shared memory, takes the spectral path even when
    the direct one is requested — results unchanged."""
    rng = np.random.default_rng(3)
    t = rng.standard_normal((2100, 4, 3))
    eng, oeng = _engines(t, 40, 3, 5)
    a, b = rng.standard_normal(4), rng.standard_normal(3)
    rel_close(eng.iuv(a, b, 0), oeng.iuv(a, b, 0), RTOL64)
    t2 = rng.standard_normal((6, 5, 4))
    eng2, oeng2 = _engines(t2, 15000, 2, 5)
    a2, b2 = rng.standard_normal(5), rng.standard_normal(4)
    rel_close(eng2.iuv(a2, b2, 0), oeng2.iuv(a2, b2, 0), RTOL64)
    with pytest.raises(ValueError):
        eng.set_path("fastest")


def test_direct_zero_and_nonfinite(cuda):
    """Zero vectors give exact zeros; a NaN input propagates into every estimate
    it touches, as in the reference's transforms."""
    rng = np.random.default_rng(4)
    t = rng.standard_normal((12, 11, 10))
    eng, oeng = _engines(t, 300, 3, 2)
    z = eng.iuv(np.zeros(11), rng.standard_normal(10), 0)
    assert np.all(z == 0.0)
    a = rng.standard_normal(11)
    a[3] = np.nan
    assert np.isnan(eng.iuv(a, rng.standard_normal(10), 0)).any()


@pytest.mark.parametrize("path", ["direct", "spectral"])
def test_rtpm_paths_vs_oracle(cuda, monkeypatch, path):
    """End-to-end rtpm (engine built inside st_rtpm; the path set through
    ST_ENGINE_PATH) on a well-conditioned tensor, against the oracle rtpm."""
    monkeypatch.setenv("ST_ENGINE_PATH", path)
    rng = np.random.default_rng(31)
    q, _ = np.linalg.qr(rng.standard_normal((40, 3)))
    t = configs.densify([3.0, 2.0, 1.5], [q, q, q]) + 1e-4 * rng.standard_normal((40, 40, 40))
    est = st.EstimatorConfig(1000, 5, 17)
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(3, 5, 10, st.SketchBackend.FCS, est))
    w, f = O.rtpm(O.FcsEngine(t, 1000, 5, 17), 40, 3, 5, 10, 17)
    rel_close(cp.weights, w, 1e-8)
    rel_close(cp._factors_cm[0].t(), f, 1e-8)
    assert np.allclose(np.sort(w)[::-1], [3.0, 2.0, 1.5], atol=0.15)


@pytest.mark.parametrize("kernel", ["mma", "dfma"])
def test_direct_q_kernels_agree(cuda, monkeypatch, kernel):
    """Batches of 2+ build Q on the fp64 tensor cores (DMMA); ST_CORR_DFMA
    selects the DFMA kernel (vector blocks 2, 4, 8, 16) — both match the oracle."""
    if kernel == "dfma":
        monkeypatch.setenv("ST_CORR_DFMA", "1")
    rng = np.random.default_rng(41)
    dims = (27, 33, 45)
    t = rng.standard_normal(dims)
    eng, oeng = _engines(t, 1200, 4, 17)
    for n in (2, 3, 7, 9, 16, 33):
        A, B = rng.standard_normal((n, 33)), rng.standard_normal((n, 45))
        got = eng.iuv_batch(A, B, 0).cpu().numpy()
        for b in sorted({0, n - 1}):
            rel_close(got[b], oeng.iuv(A[b], B[b], 0), RTOL64)


def test_direct_fused_tail_underflow(cuda, monkeypatch):
    """The direct path's fused tail on a zero tensor: every restart row
    underflows to 0 (normalisation branch) and the refinement stops at once
    (sticky flag) — weights and factors equal the oracle rtpm bit for bit."""
    monkeypatch.setenv("ST_ENGINE_PATH", "direct")
    z = np.zeros((12, 12, 12))
    cpz = st.rtpm(st.DenseTensor.from_array(z), st.RtpmConfig(2, 3, 4, st.SketchBackend.FCS,
                                                             st.EstimatorConfig(300, 3, 5)))
    wz, fz = O.rtpm(O.FcsEngine(z, 300, 3, 5), 12, 2, 3, 4, 5)
    np.testing.assert_array_equal(cpz.weights.cpu().numpy(), wz)
    np.testing.assert_array_equal(cpz._factors_cm[0].t().cpu().numpy(), fz)
