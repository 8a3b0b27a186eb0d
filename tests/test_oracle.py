"""CPU tests: pin the numpy restatement (oracle/fcs_oracle.py) against the
spec's known-answer tests and the golden vectors produced by the unmodified
reference (tests/golden/make_golden.py), and — where oracle/_ref is built —
against the reference library directly."""
import os

import numpy as np
import pytest

from oracle import fcs_oracle as O
from oracle import ref

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def rel_close(got, want, rtol):
    """|g - c| <= rtol * (|c| + ||c||_inf) per entry (SURVEY.md §8(d) parity rule)."""
    got, want = np.asarray(got), np.asarray(want)
    tol = rtol * (np.abs(want) + np.abs(want).max(initial=0.0))
    return bool(np.all(np.abs(got - want) <= tol))


# ------------------------------------------------------------- spec KATs
def test_kat_count_sketch():
    assert O.cs_sketch([1, 2, 3], [0, 1, 0], [1, -1, 1], 2).tolist() == [4.0, -2.0]


def test_kat_fcs_2x2():  # u=[1,2], v=[1,1], h1=[0,1], h2=[0,0]
    t = np.outer([1, 2], [1, 1])
    out = O.fcs_dense(t, [[0, 1], [0, 0]], [[1, 1], [1, 1]], [2, 2])
    assert out.tolist() == [2.0, 4.0, 0.0]


def test_kat_fcs_cp_fft():  # conv([1,2],[2,0]) -> [2,4,0]
    np.testing.assert_allclose(O.fft_convolve([[1, 2], [2, 0]], 3), [2, 4, 0], atol=1e-12)
    np.testing.assert_allclose(GOLD["conv_12_20"], [2, 4, 0], atol=1e-12)


def test_kat_compose():  # maps [0,1],[0,0], index (1,0) -> (1,+1)
    b, s = O.composed_tables([[0, 1], [0, 0]], [[1, 1], [1, 1]])
    assert (int(b[1]), int(s[1])) == (1, 1)


def test_kat_median():
    assert O.median_reduce([1, 2, 100]) == 2
    assert O.median_reduce([1, 2, 3, 10]) == 2.5
    with pytest.raises(ValueError):
        O.median_reduce([])


# ------------------------------------------------------------ golden pins
def test_golden_rng():
    assert [int(x) for x in O.splitmix_draw(0, np.arange(1, 4))] == [int(x) for x in
                                                                    GOLD["draws_seed0"]]
    assert (O.splitmix_draw(42, np.arange(1, 1001)) == GOLD["draws_seed42"]).all()
    assert [O.family_seed(0, d) for d in range(3)] == [int(x) for x in GOLD["family_seed0"]]
    assert hex(O.family_seed(0, 0)) == "0xe220a8397b1dcdaf"
    assert (O.gaussian_stream(1, 9) == GOLD["gauss_seed1"]).all()
    rng = O.SplitMix64(1)
    assert [rng.next_gaussian() for _ in range(9)] == GOLD["gauss_seed1"].tolist()


def test_golden_hash_family():
    b, s, j = O.hash_family([100, 100, 100], 1000, O.family_seed(0, 0))
    assert (np.stack(b) == GOLD["fam100_buckets"]).all()
    assert (np.stack(s) == GOLD["fam100_signs"]).all()
    assert O.composed_len(j) == int(GOLD["fam100_composed_len"][0]) == 2998
    assert b[0][:6].tolist() == [652, 387, 787, 778, 375, 401]  # Appendix A
    assert s[2][:6].tolist() == [-1, 1, -1, -1, 1, 1]


def test_golden_prefix_property():
    b, s = O.hash_pair(512, 2048, 7)
    assert (b == GOLD["pair512_b"]).all() and (s == GOLD["pair512_s"]).all()
    assert (GOLD["pair512_b"][:64] == GOLD["pair64_b"]).all()
    assert (GOLD["pair512_s"][:64] == GOLD["pair64_s"]).all()


def test_golden_dense_bitexact():
    x = GOLD["dense_small_x"]
    b, s, j = O.hash_family(x.shape, 7, O.family_seed(3, 0))
    assert (O.fcs_dense(x, b, s, j) == GOLD["dense_small_sketch"]).all()
    x4 = GOLD["dense_o4_x"]
    b, s, j = O.hash_family(x4.shape, 5, O.family_seed(9, 1))
    assert (O.fcs_dense(x4, b, s, j) == GOLD["dense_o4_sketch"]).all()


def test_golden_materialize():
    tb, ts = GOLD["mat_tables_b"], GOLD["mat_tables_s"]
    b = [tb[0:3], tb[3:7], tb[7:12]]
    s = [ts[0:3], ts[3:7], ts[7:12]]
    cb, cs = O.composed_tables(b, s)
    assert (cb == GOLD["mat_b"]).all() and (cs == GOLD["mat_s"]).all()


def test_golden_cp():
    fs = [GOLD[f"cp_f{i}"] for i in range(3)]
    b, s, j = O.hash_family([10, 12, 14], 9, O.family_seed(4, 2))
    got = O.fcs_cp(GOLD["cp_w"], fs, b, s, j)
    assert rel_close(got, GOLD["cp_sketch"], 1e-12)
    # path identity fcs_cp == fcs_dense(densify)
    assert rel_close(GOLD["cp_sketch"], GOLD["cp_dense_sketch"], 1e-9)


def test_golden_engine():
    t = GOLD["eng_t"]
    eng = O.FcsEngine(t, 6, 3, 5)
    u, v, w = GOLD["eng_u"], GOLD["eng_v"], GOLD["eng_w"]
    assert rel_close(eng.iuu(u), GOLD["eng_iuu"], 1e-10)
    assert rel_close(eng.iuv(u, v, 1), GOLD["eng_iuv1"], 1e-10)
    assert rel_close(eng.iuv(u, v, 2), GOLD["eng_iuv2"], 1e-10)
    assert rel_close(eng.uvw(u, v, w), GOLD["eng_uvw"][0], 1e-10)
    eng.deflate(0.7, u, v, w)
    assert rel_close(eng.iuu(u), GOLD["eng_defl_iuu"], 1e-10)
    assert rel_close(eng.uvw(u, v, w), GOLD["eng_defl_uvw"][0], 1e-10)


def test_golden_rtpm():
    t = GOLD["rtpm_t"]
    eng = O.FcsEngine(t, 12, 3, 21)
    w, f = O.rtpm(eng, 10, 2, 3, 5, 21)
    assert rel_close(w, GOLD["rtpm_weights"], 1e-8)
    assert rel_close(f, GOLD["rtpm_factor"], 1e-8)


# ------------------------------------------------------------- error paths
def test_errors_match_reference():
    with pytest.raises(ValueError):
        O.hash_pair(0, 5, 1)
    with pytest.raises(ValueError):
        O.hash_family([3, 4], [5], 1)
    b, s, j = O.hash_family([3, 4], 5, 1)
    with pytest.raises(ValueError):
        O.fcs_dense(np.zeros((4, 3)), b, s, j)
    with pytest.raises(ValueError):
        O.dft([1.0], 0)
    with pytest.raises(RuntimeError):
        O.idft_real(np.array([0, 1j, 0, -2j]) * 1e3 + np.array([1, 0, 0, 0]))


# ---------------------------------------------- direct reference cross-check
needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@needs_ref
def test_restatement_vs_reference_random():
    rng = np.random.default_rng(7)
    for shape, J, seed in (((7, 3, 5), 11, 3), ((16, 9), 40, 9), ((5, 4, 3, 2), 6, 2)):
        x = rng.standard_normal(shape)
        x[rng.random(shape) < 0.1] = 0.0
        master = O.family_seed(seed, 1)
        b, s, j = O.hash_family(shape, J, master)
        assert (O.fcs_dense(x, b, s, j) == ref.fcs_dense(x, J, master)).all()


@needs_ref
def test_restatement_vs_reference_errors():
    with pytest.raises(ValueError):
        ref.hash_pair(1, 0, 4)
    with pytest.raises(ValueError):
        ref.median([])


def test_golden_ts_hcs():
    x = GOLD["dense_small_x"]
    b, s, j = O.hash_family([6, 5, 4], 7, O.family_seed(6, 0))
    assert rel_close(O.ts_sketch(x, b, s, j), GOLD["ts_dense"], 1e-13)
    assert rel_close(O.hcs_sketch(x, b, s, j), GOLD["hcs_dense"], 1e-13)
    fs = [GOLD[f"tscp_f{i}"] for i in range(3)]
    assert rel_close(O.ts_cp(GOLD["tscp_w"], fs, b, s, j), GOLD["ts_cp"], 1e-12)
    assert rel_close(O.hcs_cp(GOLD["tscp_w"], fs, b, s, j), GOLD["hcs_cp"], 1e-12)
    with pytest.raises(ValueError):
        O.ts_sketch(x, b, s, [7, 7, 8])


# ---------------------------------------- §8(f): TS engine and CPD drivers
def test_golden_ts_engine():
    t = GOLD["eng_t"]
    eng = O.TsEngine(t, 6, 3, 5)
    u, v, w = GOLD["eng_u"], GOLD["eng_v"], GOLD["eng_w"]
    assert rel_close(eng.iuu(u), GOLD["ts_eng_iuu"], 1e-10)
    assert rel_close(eng.iuv(u, v, 1), GOLD["ts_eng_iuv1"], 1e-10)
    assert rel_close(eng.iuv(u, v, 2), GOLD["ts_eng_iuv2"], 1e-10)
    assert rel_close(eng.uvw(u, v, w), GOLD["ts_eng_uvw"][0], 1e-10)
    eng.deflate(0.7, u, v, w)
    assert rel_close(eng.iuu(u), GOLD["ts_eng_defl_iuu"], 1e-10)
    assert rel_close(eng.uvw(u, v, w), GOLD["ts_eng_defl_uvw"][0], 1e-10)


def test_golden_rtpm_asym():
    t = GOLD["asym_t"]
    w, f = O.rtpm_asym(O.FcsEngine(t, 40, 3, 9), t.shape, 2, 3, 4, 9)
    assert rel_close(w, GOLD["asym_weights"], 1e-8)
    for n in range(3):
        assert rel_close(f[n], GOLD[f"asym_f{n}"], 1e-8)
    assert (w >= 0).all()


def test_golden_als_and_residual():
    t = GOLD["asym_t"]
    w, f, sweeps = O.als(O.FcsEngine(t, 40, 3, 9), t, 2, 5, 1e-12, 9)
    assert sweeps == 5
    assert rel_close(w, GOLD["als_weights"], 1e-8)
    for n in range(3):
        assert rel_close(f[n], GOLD[f"als_f{n}"], 1e-8)
    assert rel_close(O.residual_norm(t, GOLD["als_weights"],
                                     [GOLD[f"als_f{n}"] for n in range(3)]),
                     GOLD["als_residual"][0], 1e-12)
    wt, _, _ = O.als(O.TsEngine(t, 40, 3, 9), t, 2, 5, 1e-12, 9)
    assert rel_close(wt, GOLD["als_ts_weights"], 1e-8)


def test_min_norm_solve_matches_pinv():
    rng = np.random.default_rng(5)
    A = rng.standard_normal((7, 3))
    G = A @ A.T  # rank 3
    B = rng.standard_normal((7, 4))
    np.testing.assert_allclose(O.min_norm_solve(G, B), np.linalg.pinv(G, rcond=1e-12) @ B,
                               atol=1e-10)
    assert (O.min_norm_solve(np.zeros((3, 3)), np.ones((3, 2))) == 0).all()


def test_inner_products_vs_reference():
    rng = np.random.default_rng(1)
    a, b = rng.standard_normal((5, 4, 3)), rng.standard_normal((5, 4, 3))
    assert rel_close(O.estimate_inner(a, b, 7, 5, 3), ref.estimate_inner(a, b, 7, 5, 3), 1e-12)
    for f in O.families_for(a.shape, 7, 3, 3):
        assert rel_close(O.inner_once(a, b, *f), ref.inner_once_tables(a, b, *f), 1e-12)
        assert rel_close(O.inner_once_ts(a, b, *f), ref.inner_once_tables(a, b, *f, ts=True),
                         1e-12)
    with pytest.raises(ValueError):
        ref.estimate_inner(a, b, 0, 5, 3)


def test_regression_and_codec_oracle_identities():
    rng = np.random.default_rng(2)
    dims = (2, 3, 2)
    X, w, bias = rng.standard_normal((4, 12)), rng.standard_normal((1, 12)), rng.standard_normal(3)
    y0 = O.regression_forward(X, np.zeros((3, 12)), bias, dims, 5, 5, 4)
    assert (y0 == np.broadcast_to(bias, (4, 3))).all()
    y1 = O.regression_forward(X[:1], w, bias[:1], dims, 5, 5, 4)
    est = O.estimate_inner(X[0].reshape(dims, order="F"), w[0].reshape(dims, order="F"), 5, 5, 4)
    assert rel_close(y1[0, 0], est + bias[0], 1e-12)
    # Kronecker: the order-4 tensor's entries are the Kronecker matrix's
    a, b = rng.standard_normal((3, 4)), rng.standard_normal((4, 5))
    K4, K = O.kron_tensor(a, b), np.kron(a, b)
    assert K4[2, 3, 1, 4] == K[4 * 2 + 1, 5 * 3 + 4]
    sk = O.compress_tensor4(O.kron_tensor([[2.0]], [[3.0]]), 1, 1, 0)
    assert abs(sk[0, 0]) == 6.0
    # contraction with L = 1 is the Kronecker tensor of the two slices
    A, B = rng.standard_normal((3, 4, 1)), rng.standard_normal((1, 4, 5))
    assert np.allclose(O.contraction_tensor(A, B), O.kron_tensor(A[:, :, 0], B[0]))
