"""GPU parity of the inner-product estimates, the sketched regression forward
map and the Kronecker / contraction codecs.

inner_once / inner_once_ts / estimate_inner are checked against the
unmodified reference (oracle/_ref). The regression map and the codecs exist
only in the reference's spec; they are checked against the
numpy restatement of the spec's defining identities (oracle/fcs_oracle.py:
fcs_dense of the materialised Kronecker / contraction tensor, per-row sketches
and medians) and the spec's own examples.

Tolerance: fp64 |g - c| <= 1e-10 (|c| + ||c||_inf) per entry; decompression
reads are gathers of those values (same rule).
"""
import numpy as np
import pytest
import torch

from oracle import fcs_oracle as O
from oracle import ref
import paper_2106_13062_b200 as st

pytestmark = pytest.mark.gpu
RTOL = 1e-10


def rel_close(got, want, rtol=RTOL):
    got = got.detach().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want)
    tol = rtol * (np.abs(want) + np.abs(want).max(initial=0.0))
    err = np.abs(got - want)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.all(err <= tol), f"max err {err.max()} vs tol {tol.min()}"


def fam_tables(f: st.HashFamily):
    return ([f.pair(n).bucket_map() for n in range(f.modes())],
            [f.pair(n).sign_map() for n in range(f.modes())], f.hash_lens())


# ------------------------------------------------------------ inner products
@pytest.mark.parametrize("dims,J,D,seed", [((5, 4, 3), 7, 5, 3), ((40, 30, 20), 200, 10, 9),
                                           ((64,), 16, 4, 1), ((12, 10, 8, 6), 50, 6, 2)])
def test_estimate_inner_vs_reference(cuda, dims, J, D, seed):
    rng = np.random.default_rng(seed)
    a, b = rng.standard_normal(dims), rng.standard_normal(dims)
    got, est = st.estimate_inner(a, b, st.EstimatorConfig(J, D, seed), return_estimates=True)
    assert abs(got - ref.estimate_inner(a, b, J, D, seed)) <= 1e-10 * np.abs(est.cpu().numpy()).max()
    fams = st.families_for(list(dims), st.EstimatorConfig(J, D, seed))
    rel_close(est, [ref.inner_once_tables(a, b, *fam_tables(f)) for f in fams])
    rel_close(st.inner_once(a, b, fams[0]), ref.inner_once_tables(a, b, *fam_tables(fams[0])))
    rel_close(st.inner_once_ts(a, b, fams[-1]),
              ref.inner_once_tables(a, b, *fam_tables(fams[-1]), ts=True))
    # TS kind: median of inner_once_ts over the same families
    got_ts = st.estimate_inner(a, b, st.EstimatorConfig(J, D, seed), kind=st.SketchKind.TS)
    want_ts = O.median_reduce([ref.inner_once_tables(a, b, *fam_tables(f), ts=True) for f in fams])
    assert abs(got_ts - want_ts) <= 1e-10 * (abs(want_ts) + 1)


def test_estimate_inner_f32_and_errors(cuda):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((64, 32, 8)).astype(np.float32)
    b = rng.standard_normal((64, 32, 8)).astype(np.float32)
    got = st.estimate_inner(a, b, st.EstimatorConfig(500, 5, 1))
    want = ref.estimate_inner(a.astype(np.float64), b.astype(np.float64), 500, 5, 1)
    assert abs(got - want) <= 1e-4 * np.sqrt((a.astype(np.float64) ** 2).sum() * (b ** 2).sum())
    with pytest.raises(ValueError):
        st.estimate_inner(a, b[:, :, :4], st.EstimatorConfig(8, 2, 1))
    with pytest.raises(ValueError):
        st.estimate_inner(a, b, st.EstimatorConfig(0, 2, 1))
    # a = b: the sketched squared norm is unbiased and close at large J
    x = rng.standard_normal((30, 30, 30))
    est = st.estimate_inner(x, x, st.EstimatorConfig(20000, 7, 3))
    assert abs(est / (x * x).sum() - 1) < 0.05


# ------------------------------------------------------------ regression map
@pytest.mark.parametrize("dims,B,Cn,J,D", [((2, 3, 2), 4, 3, 5, 5), ((7, 7, 32), 64, 10, 30, 3),
                                           ((6, 5), 33, 17, 9, 4)])
def test_regression_forward_vs_oracle(cuda, dims, B, Cn, J, D):
    rng = np.random.default_rng(B)
    n = int(np.prod(dims))
    X, W, bias = rng.standard_normal((B, n)), rng.standard_normal((Cn, n)), rng.standard_normal(Cn)
    y = st.sketched_regression_forward(X, W, bias, dims, st.EstimatorConfig(J, D, 11))
    rel_close(y, O.regression_forward(X, W, bias, dims, J, D, 11))


def test_regression_forward_spec_examples(cuda):
    rng = np.random.default_rng(2)
    dims, n = (2, 3, 2), 12
    X, bias = rng.standard_normal((4, n)), rng.standard_normal(3)
    cfg = st.EstimatorConfig(5, 5, 4)
    # W = 0 -> broadcast bias
    y = st.sketched_regression_forward(X, np.zeros((3, n)), bias, dims, cfg)
    assert (y.cpu().numpy() == np.broadcast_to(bias, (4, 3))).all()
    # B = C = 1 -> estimate_inner + bias
    w = rng.standard_normal((1, n))
    y = st.sketched_regression_forward(X[:1], w, bias[:1], dims, cfg)
    xi = X[0].reshape(dims, order="F")
    wi = w[0].reshape(dims, order="F")
    rel_close(y.cpu().numpy()[0, 0], st.estimate_inner(xi, wi, cfg) + bias[0])
    # f32 rows
    y32 = st.sketched_regression_forward(X.astype(np.float32), w.astype(np.float32), None, dims, cfg)
    rel_close(y32, O.regression_forward(X.astype(np.float32), w.astype(np.float32), None, dims,
                                        5, 5, 4), 1e-5)
    with pytest.raises(ValueError):
        st.sketched_regression_forward(X, w, bias, dims, cfg)  # bias length 3 != C = 1


# ------------------------------------------------------------------- codecs
@pytest.mark.parametrize("shapes,J,D", [(((3, 4), (4, 5)), 6, 5), (((30, 20), (10, 40)), 64, 3),
                                        (((64, 64), (64, 64)), 2048, 2)])
def test_compress_kron_identity(cuda, shapes, J, D):
    rng = np.random.default_rng(J)
    a = rng.uniform(-5, 5, shapes[0])
    b = rng.uniform(-5, 5, shapes[1])
    sk = st.compress_kron(a, b, st.EstimatorConfig(J, D, 8))
    assert sk.values.shape == (D, 4 * J - 3)
    rel_close(sk.values, O.compress_tensor4(O.kron_tensor(a, b), J, D, 8), 1e-9)
    # the existing order-4 entry point agrees (fcs_kron: two K1 + one convolution)
    rel_close(st.fcs_kron(a, b, sk.families), sk.values.cpu().numpy(), 1e-9)


def test_kron_spec_examples(cuda):
    # 1x1 matrices, J = 1 -> a single bucket holding 6 (times the
    # product of the four signs, which the spec's example takes as +1), and the
    # signed read recovers the entry exactly
    sk = st.compress_kron([[2.0]], [[3.0]], st.EstimatorConfig(1, 1, 0))
    signs = np.prod([sk.families[0].pair(n).sign_map()[0] for n in range(4)])
    assert sk.values.cpu().numpy().tolist() == [[6.0 * signs]]
    assert st.decompress_kron(sk, 0, 0) == 6.0
    sk = st.compress_kron(np.zeros((3, 4)), np.ones((4, 5)), st.EstimatorConfig(6, 3, 1))
    assert (sk.values.cpu().numpy() == 0).all()
    assert st.decompress_kron(sk, 5, 7) == 0.0


def test_decompress_kron(cuda):
    rng = np.random.default_rng(3)
    a, b = rng.uniform(-5, 5, (3, 4)), rng.uniform(-5, 5, (4, 5))
    K = np.kron(a, b)
    # per-entry reads and the full reconstruction against the oracle's decompression
    cfg = st.EstimatorConfig(64, 5, 2)
    sk = st.compress_kron(a, b, cfg)
    fams = [fam_tables(f) for f in sk.families]
    skh = sk.values.cpu().numpy()
    rows, cols = np.arange(12), np.arange(20)
    R, Cc = np.meshgrid(rows, cols, indexing="ij")
    got = st.decompress_kron(sk, R.ravel(), Cc.ravel()).cpu().numpy().reshape(12, 20)
    want = np.array([[O.decompress4(skh, fams, r // 4, c // 5, r % 4, c % 5) for c in cols]
                     for r in rows])
    rel_close(got, want)
    rel_close(st.reconstruct_kron(sk), want)
    assert st.decompress_kron(sk, 11, 19) == pytest.approx(want[11, 19], rel=1e-12)
    with pytest.raises(ValueError):
        st.decompress_kron(sk, 12, 0)
    # unbiasedness: the mean of single-copy reads over 200 seeds -> K;
    # one read's std is about ||K||_F / sqrt(J~), so allow 5 sigma of the mean
    acc = np.zeros_like(K)
    for s in range(200):
        one = st.compress_kron(a, b, st.EstimatorConfig(64, 1, s))
        acc += st.reconstruct_kron(one).cpu().numpy()
    assert np.abs(acc / 200 - K).max() < 5 * np.linalg.norm(K) / np.sqrt(253 * 200)


@pytest.mark.parametrize("dims,L,J,D", [((3, 4, 3, 4), 5, 8, 3), ((30, 40, 40, 30), 50, 400, 2),
                                        ((6, 5, 4, 3), 1, 16, 4)])
def test_compress_contraction_identity(cuda, dims, L, J, D):
    rng = np.random.default_rng(L)
    I1, I2, I3, I4 = dims
    a = rng.uniform(0, 10, (I1, I2, L))
    b = rng.uniform(0, 10, (L, I3, I4))
    sk = st.compress_contraction(a, b, st.EstimatorConfig(J, D, 5))
    want = O.compress_tensor4(O.contraction_tensor(a, b), J, D, 5)
    rel_close(sk.values, want, 1e-9)
    if L == 1:  # L = 1 reduces to compress_kron of the two slices
        k = st.compress_kron(a[:, :, 0], b[0], st.EstimatorConfig(J, D, 5))
        rel_close(k.values, sk.values.cpu().numpy(), 1e-12)
    fams = [fam_tables(f) for f in sk.families]
    skh = sk.values.cpu().numpy()
    q = [(0, 0, 0, 0), (I1 - 1, I2 - 1, I3 - 1, I4 - 1), (1 % I1, 2 % I2, 0, 1 % I4)]
    got = st.decompress_contraction(sk, *np.array(q).T).cpu().numpy()
    rel_close(got, [O.decompress4(skh, fams, *x) for x in q])
    with pytest.raises(ValueError):
        st.compress_contraction(a, b[:1] if L > 1 else np.ones((2, I3, I4)),
                                st.EstimatorConfig(J, D, 5))


def test_compression_ratio_and_memory(cuda):
    f = st.HashFamily([30, 40, 40, 30], 100, 1)
    assert st.compression_ratio(f) == pytest.approx(30 * 40 * 40 * 30 / (4 * 100 - 3))
    assert st.hash_memory(f) == 5 * 140 < st.hash_memory_long_pair([30, 40, 40, 30])
    assert st.compression_ratio(st.HashFamily([7], 7, 0)) == 1.0
