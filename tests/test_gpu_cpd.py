"""GPU parity of the widened engine rows: the TS
backend of the contraction engine, rtpm with the TS backend, rtpm_asym, ALS and
residual_norm — each through the C-ABI against the unmodified reference
(oracle/_ref, built from /root/reference/proj/src by oracle/Makefile) on the
same seeded inputs.

Tolerance: fp64 |g - c| <= rtol (|c| + ||c||_inf) per entry, rtol 1e-9 for
single estimates (the B200 TS path correlates at length 3J-2 instead of J:
same sums, different FFT rounding) and 1e-7 for whole decompositions (a few
hundred chained estimates and solves).
"""
import os

import numpy as np
import pytest
import torch

from oracle import ref
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import configs

pytestmark = pytest.mark.gpu
TS, FCS = st.SketchBackend.TS, st.SketchBackend.FCS


def rel_close(got, want, rtol):
    got = got.detach().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want)
    tol = rtol * (np.abs(want) + np.abs(want).max(initial=0.0))
    err = np.abs(got - want)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.all(err <= tol), f"max err {err.max()} vs tol {tol.min()}"


def low_rank(dims, weights, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    fs = [np.linalg.qr(rng.standard_normal((n, len(weights))))[0] for n in dims]
    t = configs.densify(weights, fs)
    if noise:
        t = t + noise * rng.standard_normal(t.shape)
    return t, fs


# ------------------------------------------------------------ TS engine
@pytest.mark.parametrize("dims,J,D,seed", [((9, 7, 5), 6, 3, 5), ((40, 30, 20), 64, 5, 11),
                                           ((60, 60, 60), 300, 10, 3)])
def test_ts_engine_vs_reference(cuda, dims, J, D, seed):
    rng = np.random.default_rng(seed)
    t = rng.standard_normal(dims)
    eng = st.make_contraction_engine(st.DenseTensor.from_array(t), TS,
                                     st.EstimatorConfig(J, D, seed))
    oeng = ref.Engine(t, J, D, seed, backend=ref.BACKEND_TS)
    u, v, w = (rng.standard_normal(n) for n in dims)
    assert eng.composed_len() == J
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), 1e-9)
    rel_close(eng.iuv(u, w, 1), oeng.iuv(u, w, 1), 1e-9)
    rel_close(eng.iuv(u, v, 2), oeng.iuv(u, v, 2), 1e-9)
    rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w), 1e-9)
    # the engine's sketches are the reference's ts_sketch per family
    fams = st.families_for(list(dims), st.EstimatorConfig(J, D, seed))
    sk = eng.sketches().cpu().numpy()
    for d in (0, D - 1):
        b = [fams[d].pair(n).bucket_map() for n in range(3)]
        s = [fams[d].pair(n).sign_map() for n in range(3)]
        rel_close(sk[d], ref.ts_dense_tables(t, b, s, [J] * 3), 1e-12)
    eng.deflate(0.7, u, v, w)
    oeng.deflate(0.7, u, v, w)
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), 1e-9)
    rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w), 1e-9)


def test_ts_engine_batched_f32(cuda):
    rng = np.random.default_rng(4)
    t = rng.standard_normal((32, 24, 16)).astype(np.float32)
    eng = st.TsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(50, 4, 9))
    oeng = ref.Engine(t.astype(np.float64), 50, 4, 9, backend=ref.BACKEND_TS)
    A, B = rng.standard_normal((7, 24)), rng.standard_normal((7, 16))
    got = eng.iuv_batch(A, B, 0).cpu().numpy()
    for l in range(7):
        rel_close(got[l], oeng.iuv(A[l], B[l], 0), 1e-4)


@pytest.mark.parametrize("backend", [st.SketchBackend.Plain, st.SketchBackend.HCS,
                                     st.SketchBackend.CS])
@pytest.mark.parametrize("dims,J,D,seed", [((9, 7, 5), 6, 3, 5), ((40, 30, 20), 16, 5, 11),
                                           ((24, 24, 24), 40, 4, 2)])
def test_exact_engines_vs_reference(cuda, backend, dims, J, D, seed):
    """Plain (exact), HCS and long-pair CS engines (cpd.cpp:36-59,128-197)."""
    rng = np.random.default_rng(seed)
    t = rng.standard_normal(dims)
    eng = st.make_contraction_engine(st.DenseTensor.from_array(t), backend,
                                     st.EstimatorConfig(J, D, seed))
    oeng = ref.Engine(t, J, D, seed, backend=backend.value)
    u, v, w = (rng.standard_normal(n) for n in dims)
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), 1e-11)
    rel_close(eng.iuv(u, w, 1), oeng.iuv(u, w, 1), 1e-11)
    rel_close(eng.iuv(u, v, 2), oeng.iuv(u, v, 2), 1e-11)
    rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w), 1e-11)
    eng.deflate(0.7, u, v, w)
    oeng.deflate(0.7, u, v, w)
    rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), 1e-11)
    rel_close(eng.iuv(u, v, 2), oeng.iuv(u, v, 2), 1e-11)
    rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w), 1e-11)
    # batches larger than one chunk of 8, zero entries in the vectors
    A, B = rng.standard_normal((11, dims[1])), rng.standard_normal((11, dims[2]))
    B[3, :2] = 0.0
    got = eng.iuv_batch(A, B, 0).cpu().numpy()
    for l in (0, 3, 10):
        rel_close(got[l], oeng.iuv(A[l], B[l], 0), 1e-11)
    U3 = rng.standard_normal((9, dims[0]))
    vals = eng.uvw_batch(U3, A[:9], B[:9]).cpu().numpy()
    for l in (0, 8):
        rel_close(vals[l], oeng.uvw(U3[l], A[l], B[l]), 1e-11)


def test_plain_engine_is_exact(cuda):
    rng = np.random.default_rng(3)
    t = rng.standard_normal((12, 10, 8))
    eng = st.PlainEngine(st.DenseTensor.from_array(t.astype(np.float32)),
                         st.EstimatorConfig(0, 0, 0))
    u, v, w = (rng.standard_normal(n) for n in t.shape)
    t32 = t.astype(np.float32).astype(np.float64)
    rel_close(eng.iuv(v, w, 0), np.einsum("ijk,j,k->i", t32, v, w), 1e-12)
    rel_close(eng.uvw(u, v, w), np.einsum("ijk,i,j,k->", t32, u, v, w), 1e-12)
    with pytest.raises(ValueError):
        eng.sketches()


# ------------------------------------------------------------ rtpm / rtpm_asym
def test_rtpm_ts_backend_vs_reference(cuda):
    q = np.linalg.qr(np.random.default_rng(41).standard_normal((30, 2)))[0]
    t = configs.densify([3.0, 2.0], [q, q, q])
    est = st.EstimatorConfig(400, 5, 13)
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(2, 4, 8, TS, est))
    w, f = ref.rtpm(t, 2, 4, 8, 400, 5, 13, backend=ref.BACKEND_TS)
    rel_close(cp.weights, w, 1e-7)
    rel_close(cp.factors[0], f, 1e-7)


@pytest.mark.parametrize("backend", [FCS, TS])
def test_rtpm_asym_vs_reference(cuda, backend):
    t, fs = low_rank((24, 20, 16), [4.0, 2.5, 1.0], 52, noise=1e-3)
    est = st.EstimatorConfig(500, 5, 29)
    cp = st.rtpm_asym(st.DenseTensor.from_array(t), st.RtpmConfig(3, 4, 6, backend, est))
    w, f = ref.rtpm_asym(t, 3, 4, 6, 500, 5, 29, backend=backend.value)
    rel_close(cp.weights, w, 1e-7)
    for n in range(3):
        rel_close(cp.factors[n], f[n], 1e-7)
    assert (cp.weights.cpu().numpy() >= 0).all()


def test_rtpm_asym_recovers_components(cuda):
    t, fs = low_rank((40, 30, 20), [5.0, 3.0], 61, noise=1e-4)
    cp = st.rtpm_asym(st.DenseTensor.from_array(t),
                      st.RtpmConfig(2, 5, 10, FCS, st.EstimatorConfig(2000, 5, 3)))
    np.testing.assert_allclose(np.sort(cp.weights.cpu().numpy())[::-1], [5.0, 3.0], atol=0.1)
    assert st.residual_norm(st.DenseTensor.from_array(t), cp) < 0.3


@pytest.mark.parametrize("backend", [st.SketchBackend.Plain, st.SketchBackend.HCS,
                                     st.SketchBackend.CS])
def test_cpd_drivers_exact_backends(cuda, backend):
    """rtpm / rtpm_asym / als through the Plain, HCS and CS engines vs the reference."""
    q = np.linalg.qr(np.random.default_rng(5).standard_normal((12, 2)))[0]
    t = configs.densify([3.0, 1.5], [q, q, q])
    est = st.EstimatorConfig(10, 3, 9)
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(2, 3, 5, backend, est))
    w, f = ref.rtpm(t, 2, 3, 5, 10, 3, 9, backend=backend.value)
    rel_close(cp.weights, w, 1e-8)
    rel_close(cp.factors[0], f, 1e-8)
    ta, _ = low_rank((10, 8, 6), [2.0, 1.0], 6, noise=1e-3)
    cp = st.rtpm_asym(st.DenseTensor.from_array(ta), st.RtpmConfig(2, 3, 4, backend, est))
    w, f = ref.rtpm_asym(ta, 2, 3, 4, 10, 3, 9, backend=backend.value)
    rel_close(cp.weights, w, 1e-8)
    for n in range(3):
        rel_close(cp.factors[n], f[n], 1e-8)
    cp = st.als(st.DenseTensor.from_array(ta), st.AlsConfig(2, 6, backend, est, 1e-12))
    w, f = ref.als(ta, 2, 6, 1e-12, 10, 3, 9, backend=backend.value)
    rel_close(cp.weights, w, 1e-7)
    for n in range(3):
        rel_close(cp.factors[n], f[n], 1e-7)


def test_rtpm_plain_default_recovers(cuda):
    """RtpmConfig defaults to the Plain backend, as the reference (cpd.hpp:49-55)."""
    q = np.linalg.qr(np.random.default_rng(8).standard_normal((30, 3)))[0]
    t = configs.densify([4.0, 2.0, 1.0], [q, q, q])
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(target_rank=3))
    np.testing.assert_allclose(np.sort(cp.weights.cpu().numpy())[::-1], [4.0, 2.0, 1.0],
                               atol=1e-6)
    assert st.residual_norm(st.DenseTensor.from_array(t), cp) < 1e-6


# ------------------------------------------------------------ ALS
@pytest.mark.parametrize("backend", [FCS, TS])
def test_als_vs_reference(cuda, backend):
    t, fs = low_rank((20, 16, 12), [3.0, 2.0, 1.0], 71, noise=1e-3)
    est = st.EstimatorConfig(400, 5, 7)
    cp, sweeps = st.als(st.DenseTensor.from_array(t), st.AlsConfig(3, 8, backend, est, 1e-12),
                        return_sweeps=True)
    w, f = ref.als(t, 3, 8, 1e-12, 400, 5, 7, backend=backend.value)
    assert sweeps == 8
    rel_close(cp.weights, w, 1e-7)
    for n in range(3):
        rel_close(cp.factors[n], f[n], 1e-7)


def test_als_short_hash(cuda):
    """A short hash length (J=64 for a 12x10x8 tensor): heavy collisions in the
    sketched MTTKRP. Past ~20 sweeps this instance is chaotic (a 1e-14 input
    perturbation changes the reference's own factors by O(1)), so parity is
    checked after 10 sweeps."""
    rng = np.random.default_rng(0)
    dims, R = (12, 10, 8), 3
    F = [rng.standard_normal((n, R)) for n in dims]
    t = configs.densify([3.0, 2.0, 1.0], F)
    cp = st.als(st.DenseTensor.from_array(t), st.AlsConfig(R, 10, FCS, st.EstimatorConfig(64, 5, 7),
                                                           1e-10))
    w, f = ref.als(t, R, 10, 1e-10, 64, 5, 7, backend=4)
    rel_close(cp.weights, w, 1e-7)
    for n in range(3):
        rel_close(cp.factors[n], f[n], 1e-7)


def test_als_zero_tensor(cuda):
    """All-zero MTTKRP: every Gram matrix is zero (numerical rank 0), the
    minimum-norm solve returns zero factors, residual 0/0 := 0 stops sweep 2."""
    t = np.zeros((6, 5, 4))
    cp, sweeps = st.als(st.DenseTensor.from_array(t),
                        st.AlsConfig(2, 20, FCS, st.EstimatorConfig(16, 3, 1), 1e-8),
                        return_sweeps=True)
    w, f = ref.als(t, 2, 20, 1e-8, 16, 3, 1, backend=4)
    assert sweeps == 2
    assert (cp.weights.cpu().numpy() == w).all()
    for n in range(3):
        assert (cp.factors[n].cpu().numpy() == f[n]).all()


def test_als_tolerance_stop(cuda):
    t, fs = low_rank((16, 16, 16), [2.0, 1.0], 81)
    est = st.EstimatorConfig(3000, 3, 5)
    cp, sweeps = st.als(st.DenseTensor.from_array(t), st.AlsConfig(2, 50, FCS, est, 1e-4),
                        return_sweeps=True)
    w, f = ref.als(t, 2, 50, 1e-4, 3000, 3, 5, backend=4)
    w6, _ = ref.als(t, 2, 6, 1e-4, 3000, 3, 5, backend=4)
    assert sweeps == 6 and np.array_equal(w, w6)  # the reference also stops after sweep 6
    rel_close(cp.weights, w, 1e-7)


# ------------------------------------------------------------ residual_norm
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_residual_norm_vs_reference(cuda, dtype):
    rng = np.random.default_rng(91)
    dims, R = (33, 17, 9), 4
    t = rng.standard_normal(dims).astype(dtype)
    w = rng.standard_normal(R)
    F = [rng.standard_normal((n, R)) for n in dims]
    got = st.residual_norm(st.DenseTensor.from_array(t), st.CpTensor(w, F))
    want = ref.residual_norm(t.astype(np.float64), w, F)
    assert abs(got - want) <= 1e-12 * abs(want)
    # exact CP -> 0; zero tensor vs nonzero CP -> inf; both zero -> 0
    exact = configs.densify(w, F)
    assert st.residual_norm(st.DenseTensor.from_array(exact), st.CpTensor(w, F)) < 1e-13
    z = np.zeros(dims)
    assert st.residual_norm(st.DenseTensor.from_array(z), st.CpTensor(w, F)) == np.inf
    assert st.residual_norm(st.DenseTensor.from_array(z), st.CpTensor(0 * w, F)) == 0.0


# ------------------------------------------------------------ golden vectors
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_golden_ts_engine(cuda):
    eng = st.TsEngine(st.DenseTensor.from_array(GOLD["eng_t"]), st.EstimatorConfig(6, 3, 5))
    u, v, w = GOLD["eng_u"], GOLD["eng_v"], GOLD["eng_w"]
    rel_close(eng.iuu(u), GOLD["ts_eng_iuu"], 1e-10)
    rel_close(eng.iuv(u, v, 1), GOLD["ts_eng_iuv1"], 1e-10)
    rel_close(eng.iuv(u, v, 2), GOLD["ts_eng_iuv2"], 1e-10)
    rel_close(eng.uvw(u, v, w), GOLD["ts_eng_uvw"][0], 1e-10)
    eng.deflate(0.7, u, v, w)
    rel_close(eng.iuu(u), GOLD["ts_eng_defl_iuu"], 1e-10)
    rel_close(eng.uvw(u, v, w), GOLD["ts_eng_defl_uvw"][0], 1e-10)


def test_golden_rtpm_asym_als(cuda):
    t = st.DenseTensor.from_array(GOLD["asym_t"])
    est = st.EstimatorConfig(40, 3, 9)
    cp = st.rtpm_asym(t, st.RtpmConfig(2, 3, 4, FCS, est))
    rel_close(cp.weights, GOLD["asym_weights"], 1e-8)
    for n in range(3):
        rel_close(cp.factors[n], GOLD[f"asym_f{n}"], 1e-8)
    cp = st.als(t, st.AlsConfig(2, 5, FCS, est, 1e-12))
    rel_close(cp.weights, GOLD["als_weights"], 1e-8)
    for n in range(3):
        rel_close(cp.factors[n], GOLD[f"als_f{n}"], 1e-8)
    assert abs(st.residual_norm(t, cp) - GOLD["als_residual"][0]) <= 1e-8 * GOLD["als_residual"][0]
    cp = st.als(t, st.AlsConfig(2, 5, TS, est, 1e-12))
    rel_close(cp.weights, GOLD["als_ts_weights"], 1e-8)


# ------------------------------------------------------------ tensor utilities
def test_psnr_densify_contract_inner(cuda):
    rng = np.random.default_rng(17)
    a = rng.standard_normal((9, 8, 7))
    b = a + 0.01 * rng.standard_normal(a.shape)
    assert abs(st.psnr(a, b) - ref.psnr(a, b)) < 1e-10
    assert st.psnr(a, a) == ref.psnr(a, a) == 99.0
    assert abs(st.psnr(a.astype(np.float32), b.astype(np.float32)) -
               ref.psnr(a.astype(np.float32).astype(np.float64),
                        b.astype(np.float32).astype(np.float64))) < 1e-4
    with pytest.raises(ValueError):
        st.psnr(a, b[:, :, :3])
    w = rng.standard_normal(3)
    F = [rng.standard_normal((n, 3)) for n in (5, 4, 3, 2)]
    dt = st.densify(st.CpTensor(w, F))
    want = np.einsum("r,ir,jr,kr,lr->ijkl", w, *F)
    got = dt.flat.cpu().numpy().reshape(dt.shape(), order="F")
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-13)
    u, v, x = (rng.standard_normal(n) for n in a.shape)
    assert abs(st.contract3(a, u, v, x) - np.einsum("ijk,i,j,k->", a, u, v, x)) < 1e-12
    np.testing.assert_allclose(st.contract3_free(a, u, x, 1), np.einsum("ijk,i,k->j", a, u, x),
                               rtol=1e-12, atol=1e-12)
    assert abs(st.inner(a, b) - float((a * b).sum())) < 1e-10
    r1 = st.rank_one(2.0, [u, v, x])
    np.testing.assert_allclose(st.densify(r1).flat.cpu().numpy().reshape(a.shape, order="F"),
                               2.0 * np.einsum("i,j,k->ijk", u, v, x), rtol=1e-13, atol=1e-14)


def test_sharded_rtpm_driver_single_process(cuda):
    """The restart-sharded RTPM driver (dist.sharded_rtpm) on one process with the
    device engine reproduces st.rtpm (same initial stream, argmax and refinement)."""
    from paper_2106_13062_b200 import dist as pdist
    q = np.linalg.qr(np.random.default_rng(23).standard_normal((20, 2)))[0]
    t = configs.densify([3.0, 1.5], [q, q, q])
    est = st.EstimatorConfig(200, 3, 5)
    w, f = pdist.sharded_rtpm(st.FcsEngine(st.DenseTensor.from_array(t), est), 20, 2, 4, 6, 5)
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(2, 4, 6, FCS, est))
    rel_close(w, cp.weights.cpu().numpy(), 1e-9)
    rel_close(f, cp.factors[0].cpu().numpy(), 1e-9)


def test_tensor_layout_utilities(cuda):
    rng = np.random.default_rng(29)
    a = rng.standard_normal((3, 4, 5))
    b = rng.standard_normal((5, 2, 3))
    for m in range(3):
        np.testing.assert_array_equal(st.mode_unfold(a, m).cpu().numpy(), ref.mode_unfold(a, m))
        back = st.mode_fold(st.mode_unfold(a, m), a.shape, m)
        np.testing.assert_array_equal(back.flat.cpu().numpy(), a.ravel(order="F"))
    got = st.contract_pair(a, b, 2, 0)
    want = ref.contract_pair(a, b, 2, 0)
    assert got.shape() == list(want.shape)
    np.testing.assert_allclose(got.flat.cpu().numpy(), want.ravel(order="F"), rtol=1e-12,
                               atol=1e-12)
    got = st.contract_pair(a, b, 0, 2)
    np.testing.assert_allclose(got.flat.cpu().numpy(),
                               ref.contract_pair(a, b, 0, 2).ravel(order="F"), rtol=1e-12,
                               atol=1e-12)
    x, y = rng.standard_normal((3, 4)), rng.standard_normal((2, 5))
    np.testing.assert_allclose(st.kron(x, y).cpu().numpy(), ref.kron(x, y), rtol=1e-15)
    tm = st.tensor_from_matrix(x)
    assert tm.shape() == [3, 4]
    np.testing.assert_array_equal(tm.flat.cpu().numpy(), x.ravel(order="F"))
    with pytest.raises(ValueError):
        st.contract_pair(a, b, 1, 0)
    with pytest.raises(ValueError):
        st.mode_unfold(a, 3)


def test_engine_many_sketches(cuda):
    """D > 64 families: the median takes the rank-selection path (no storage)."""
    rng = np.random.default_rng(31)
    t = rng.standard_normal((8, 7, 6))
    for D in (65, 80):
        eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(9, D, 4))
        oeng = ref.Engine(t, 9, D, 4)
        u, v, w = (rng.standard_normal(n) for n in t.shape)
        rel_close(eng.iuv(v, w, 0), oeng.iuv(v, w, 0), 1e-10)
        rel_close(eng.uvw(u, v, w), oeng.uvw(u, v, w), 1e-10)
        got, est = st.estimate_inner(t, t, st.EstimatorConfig(9, D, 4), return_estimates=True)
        assert abs(got - ref.estimate_inner(t, t, 9, D, 4)) <= 1e-10 * abs(got)
