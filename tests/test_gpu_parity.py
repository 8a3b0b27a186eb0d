"""GPU parity tests: the sm_100a path (through the C-ABI) against the CPU
oracle (oracle/fcs_oracle.py, pinned to the unmodified reference by
tests/test_oracle.py) and the golden vectors.

Tolerances: hash tables, bucket indices and integer-valued
sketches bit-exact; fp64 values |g - c| <= 1e-10 (|c| + ||c||_inf) per entry;
fp32 inputs 1e-4 on the same rule.
"""
import os

import numpy as np
import pytest
import torch

from oracle import fcs_oracle as O
import paper_2106_13062_b200 as st
from paper_2106_13062_b200 import configs

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
RTOL64, RTOL32 = 1e-10, 1e-4


def rel_close(got, want, rtol):
    got = got.detach().cpu().numpy() if torch.is_tensor(got) else np.asarray(got)
    want = np.asarray(want)
    tol = rtol * (np.abs(want) + np.abs(want).max(initial=0.0))
    err = np.abs(got - want)
    assert got.shape == want.shape, (got.shape, want.shape)
    assert np.all(err <= tol), f"max err {err.max()} vs tol {tol.min()}"
    return True


@pytest.fixture
def spectral_path(monkeypatch):
    """Engines built under this fixture take the spectral (FFT correlation)
    estimator path: tests of the transform kernels must not be served by the
    direct time-domain path the cost rule would pick at their sizes."""
    monkeypatch.setenv("ST_ENGINE_PATH", "spectral")


def oracle_family(fam: st.HashFamily):
    return ([fam.pair(n).bucket_map() for n in range(fam.modes())],
            [fam.pair(n).sign_map() for n in range(fam.modes())], fam.hash_lens())


# ------------------------------------------------------------------ K0
@pytest.mark.parametrize("I,J,seed", [(100, 1000, 1), (1024, 16384, 0xDEADBEEF), (1, 1, 0),
                                      (512, 2048, 7), (4097, 3, 2 ** 63 + 5)])
def test_hash_pair_bitexact(cuda, I, J, seed):
    p = st.HashPair(I, J, seed)
    b, s = O.hash_pair(I, J, seed)
    assert (p.bucket_map() == b).all() and (p.sign_map() == s).all()


def test_family_tables_bitexact(cuda):
    cfg = st.EstimatorConfig(hash_len=3000, sketch_count=10, seed=3)
    fams = st.families_for([200, 200, 200], cfg)
    packed = st.packed_families(fams).cpu().numpy().view(np.uint32)
    want = []
    for fb, fs, _ in O.families_for([200, 200, 200], 3000, 10, 3):
        for b, s in zip(fb, fs):
            want.append(b.astype(np.uint64) | np.where(s < 0, 1 << 31, 0).astype(np.uint64))
    assert (packed == np.concatenate(want).astype(np.uint32)).all()
    # Appendix A: first entries of HashFamily({100,100,100},1000,family_seed(0,0))
    f = st.HashFamily([100, 100, 100], 1000, st.family_seed(0, 0))
    assert f.pair(0).bucket_map()[:6].tolist() == [652, 387, 787, 778, 375, 401]
    assert f.composed_len() == 2998


def test_hash_errors(cuda):
    with pytest.raises(ValueError):
        st.HashPair(0, 5, 1)
    with pytest.raises(ValueError):
        st.HashPair(bucket_map=[0, 5], sign_map=[1, 1], hash_len=5)
    with pytest.raises(ValueError):
        st.HashPair(bucket_map=[0, 1], sign_map=[1, 0], hash_len=5)


# ------------------------------------------------------------------ K1
def test_dense_kat_2x2(cuda):
    fam = st.HashFamily(pairs=[st.HashPair(bucket_map=[0, 1], sign_map=[1, 1], hash_len=2),
                               st.HashPair(bucket_map=[0, 0], sign_map=[1, 1], hash_len=2)])
    out = st.fcs_sketch(st.DenseTensor.from_array(np.outer([1.0, 2.0], [1.0, 1.0])), fam)
    assert out.values.cpu().tolist() == [2.0, 4.0, 0.0]


def test_dense_golden(cuda):
    x = GOLD["dense_small_x"]
    fam = st.HashFamily(x.shape, 7, st.family_seed(3, 0))
    rel_close(st.fcs_sketch(x, fam).values, GOLD["dense_small_sketch"], 1e-13)
    x4 = GOLD["dense_o4_x"]
    fam4 = st.HashFamily(x4.shape, 5, st.family_seed(9, 1))
    rel_close(st.fcs_sketch(x4, fam4).values, GOLD["dense_o4_sketch"], 1e-13)


@pytest.mark.parametrize("shape,J,D,dtype", [((37, 11, 23), 29, 3, np.float64),
                                             ((64, 48, 40), 500, 4, np.float32),
                                             ((5, 4, 3, 2, 3), 7, 2, np.float64),
                                             ((1000,), 77, 2, np.float64)])
def test_dense_integer_bitexact(cuda, shape, J, D, dtype):
    """Small-integer data: every partial sum is exact, so any bucket or sign
    error shows up as an exact mismatch (bucket indices bit-exact)."""
    rng = np.random.default_rng(11)
    x = rng.integers(-8, 9, size=shape).astype(dtype)
    fams = st.families_for(list(shape), st.EstimatorConfig(J, D, 99))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        assert (got[d] == O.fcs_dense(x.astype(np.float64), b, s, j)).all()


@pytest.mark.parametrize("i0", [4, 100, 128, 200, 256, 500, 512, 1000, 1024, 1028, 2048, 6])
@pytest.mark.parametrize("D", [1, 2, 3])
def test_dense_f32_kernel_variants(cuda, i0, D):
    """Every fp32 kernel variant by fiber length: guarded / full-vector fixed
    point with 1-8 vectors per lane, the bank-grouped order (D >= 2, full
    vectors), unaligned fibers (I_0 % 4 != 0) and fibers beyond 1024 elements
    (float-atomic kernel). Integer data: fixed point is exact, so bit-exact."""
    rng = np.random.default_rng(i0 + D)
    x = rng.integers(-8, 9, size=(i0, 6, 5)).astype(np.float32)
    fams = st.families_for([i0, 6, 5], st.EstimatorConfig(300, D, 5))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
    for d, f in enumerate(fams):
        b, s_, j = oracle_family(f)
        assert (got[d] == O.fcs_dense(x.astype(np.float64), b, s_, j)).all(), d


def test_dense_f32_deterministic(cuda):
    """The fp32 fixed-point path is run-to-run bit-identical: integer shared
    atomics, a fixed-order sample reduction for the scale and fixed-order
    partial sums (K1)."""
    rng = np.random.default_rng(21)
    x = rng.standard_normal((1024, 40, 24)).astype(np.float32)
    fams = st.families_for([1024, 40, 24], st.EstimatorConfig(4096, 4, 3))
    t = st.DenseTensor.from_array(x)
    first = st.fcs_dense_batched(t, fams)
    for _ in range(3):
        assert torch.equal(st.fcs_dense_batched(t, fams), first)


def test_dense_c1_full(cuda):
    """BASELINE config 1: 100^3 fp64, J=1000, D=1 -> 2998 buckets."""
    c = configs.C1
    x = configs.c1_tensor(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams)
    assert got.shape == (1, 2998)
    b, s, j = oracle_family(fams[0])
    rel_close(got[0], O.fcs_dense(x, b, s, j), RTOL64)


def test_dense_f32_wide_sketch(cuda):
    """c4 geometry on a slab: fp32, J=16384 per mode -> J~=49150 (one family per SM)."""
    rng = np.random.default_rng(4)
    x = rng.standard_normal((1024, 32, 16)).astype(np.float32)
    fams = st.families_for([1024, 32, 16], st.EstimatorConfig(16384, 4, 4))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams)
    assert got.shape == (4, 49150)
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        rel_close(got[d], O.fcs_dense(x.astype(np.float64), b, s, j), RTOL32)


def test_dense_c4_full_size(cuda):
    """BASELINE config 4 at full size (1024^3 fp32, J = 16384, D = 4), the bench
    workload, through size-independent checks: (i) every bucket against an
    independent kernel — the fp64 global-atomic path on the widened tensor
    (itself pinned to the oracle in test_dense_global_fallback) — at the fp32
    rule; (ii) the zeroth and first moments of each sketch against direct
    contractions of the tensor: sum_b sk[b] = <T, s0 (x) s1 (x) s2> and
    sum_b b sk[b] = sum_n <T, ... (h_n s_n) ...> (every element lands in bucket
    h0 + h1 + h2 with sign s0 s1 s2). Moment tolerance 1e-3 ||T||_F (x J~ for
    the first): the fixed-point rounding sums to ~2e-2 here, a dropped or
    doubled fiber chunk moves the sum by ~1e3."""
    import ctypes as C
    from paper_2106_13062_b200 import _lib as L
    c = configs.C4
    n = int(np.prod(c.dims))
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    L.check(L.lib().st_device_gaussian(L.ST_F32, c.seed, n, C.c_void_p(x.data_ptr()), None))
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_dense_batched(st.DenseTensor(list(c.dims), x), fams)
    x64 = x.double()
    del x
    ref = st.fcs_dense_batched(st.DenseTensor(list(c.dims), x64), fams)
    assert got.shape == ref.shape == (4, 49150)
    rel_close(got, ref.cpu().numpy(), RTOL32)
    X = x64.view(c.dims[2], c.dims[1], c.dims[0])  # column-major: [i2][i1][i0]
    norm = float(torch.linalg.vector_norm(x64))
    jt = got.shape[1]
    b = torch.arange(jt, dtype=torch.float64, device="cuda")
    for d, f in enumerate(fams):
        s = [torch.tensor(f.pair(k).sign_map(), dtype=torch.float64, device="cuda") for k in range(3)]
        h = [torch.tensor(f.pair(k).bucket_map().astype(np.int64), dtype=torch.float64,
                          device="cuda") for k in range(3)]

        def con(a0, a1, a2):
            return float(((X @ a0) @ a1) @ a2)
        m0 = con(s[0], s[1], s[2])
        m1 = con(h[0] * s[0], s[1], s[2]) + con(s[0], h[1] * s[1], s[2]) + \
            con(s[0], s[1], h[2] * s[2])
        assert abs(float(got[d].sum()) - m0) <= 1e-3 * norm, (d, float(got[d].sum()), m0)
        assert abs(float(got[d] @ b) - m1) <= 1e-3 * norm * jt, (d, float(got[d] @ b), m1)


def _c4_gpu_and_reference(x, report=False):
    """K1 on the device-resident config-4-geometry tensor x (fp32, flat) and
    the unmodified reference's fcs_sketch (oracle/_ref) on the same values
    widened to fp64: 64 slabs of 16 i_3-planes per family, each sketched by the
    reference with the family's last-mode table sliced to the slab (linearity,
    SPEC.md:224), summed in slab order; all host threads."""
    import concurrent.futures as cf
    import ctypes as C
    from oracle import ref
    from paper_2106_13062_b200 import _lib as L
    c = configs.C4
    dims = list(c.dims)
    fams = st.families_for(dims, st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    lib = L.lib()
    packed = st.packed_families(fams)
    dims_a, lens_a = L.size_array(dims), L.size_array([c.hash_len] * 3)
    ws_bytes = lib.st_fcs_dense_workspace(L.ST_F32, 3, dims_a, dims[2], c.sketch_count, lens_a)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    out = torch.empty((c.sketch_count, fams[0].composed_len()), dtype=torch.float64,
                      device="cuda")
    L.check(lib.st_fcs_dense(L.ST_F32, C.c_void_p(x.data_ptr()), 3, dims_a, 0, dims[2],
                             c.sketch_count, C.c_void_p(packed.data_ptr()), lens_a,
                             C.c_void_p(out.data_ptr()), 0, C.c_void_p(ws.data_ptr()), ws_bytes,
                             None))
    got = out.cpu().numpy()
    S, fb, ctas = C.c_int(0), C.c_size_t(0), C.c_size_t(0)
    L.check(lib.st_fcs_dense_report(L.ST_F32, 3, dims_a, dims[2], c.sketch_count, lens_a,
                                    C.c_void_p(ws.data_ptr()), ws_bytes, C.byref(S), C.byref(fb),
                                    C.byref(ctas)))
    host = x.cpu().numpy()
    per = dims[0] * dims[1]
    tabs = [ref.hash_family(dims, c.hash_len, ref.family_seed(c.seed, d)) for d in range(c.sketch_count)]
    slab = 16

    def one(task):
        s0, d = task
        b, sg, _ = tabs[d]
        t = host[s0 * per:(s0 + slab) * per].astype(np.float64).reshape(
            (dims[0], dims[1], slab), order="F")
        return ref.fcs_dense_tables(t, [b[0], b[1], b[2][s0:s0 + slab]],
                                    [sg[0], sg[1], sg[2][s0:s0 + slab]], [c.hash_len] * 3)
    tasks = [(s0, d) for d in range(c.sketch_count) for s0 in range(0, dims[2], slab)]
    with cf.ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        outs = list(ex.map(one, tasks))
    want = np.zeros_like(got)
    for (s0, d), o in zip(tasks, outs):  # slab order per family
        want[d] += o
    return got, want, {"S": S.value, "fallback_ctas": fb.value, "ctas": ctas.value}


def precision(got, want):
    """max |g-c| / ||c||_inf and the pure relative error on the buckets with
    |c| > 1e-3 ||c||_inf (per family)."""
    inf = np.abs(want).max(axis=-1, keepdims=True)
    big = np.abs(want) > 1e-3 * inf
    err = np.abs(got - want)
    return float((err / inf).max()), float((err[big] / np.abs(want[big])).max())


def test_dense_c4_full_vs_reference(cuda):
    """The bench workload itself (config 4: 1024^3 fp32 device fill, J = 16384,
    D = 4) against the unmodified reference; every bucket at the fp32 rule, and
    no CTA falling back. The pure relative error of the buckets above
    1e-3 ||c||_inf is bounded by the fixed-point quantum (2^-(S+1) per
    element, ~22k elements per bucket): < 1e-3."""
    import ctypes as C
    from paper_2106_13062_b200 import _lib as L
    c = configs.C4
    n = int(np.prod(c.dims))
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    L.check(L.lib().st_device_gaussian(L.ST_F32, c.seed, n, C.c_void_p(x.data_ptr()), None))
    got, want, rep = _c4_gpu_and_reference(x)
    del x
    rel_close(got, want, RTOL32)
    inf_err, rel_big = precision(got, want)
    assert rep["fallback_ctas"] == 0 and rel_big < 1e-3, (rep, inf_err, rel_big)


@pytest.mark.parametrize("kind", ["lognormal4", "sparse_outliers"])
def test_dense_c4_wide_range_vs_reference(cuda, kind):
    """Wide-dynamic-range fp32 data at config-4 geometry:
    lognormal sigma = 4 (values e^(4 N(0,1)), up to ~1e10), and N(0,1) with
    4096 outliers of magnitude 1e6..1e9 at random positions. Every bucket at
    the fp32 rule and the large buckets to 1e-4 relative."""
    import ctypes as C
    from paper_2106_13062_b200 import _lib as L
    c = configs.C4
    n = int(np.prod(c.dims))
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    L.check(L.lib().st_device_gaussian(L.ST_F32, c.seed + 11, n, C.c_void_p(x.data_ptr()), None))
    if kind == "lognormal4":
        x.mul_(4.0).exp_()
    else:
        g = torch.Generator(device="cuda").manual_seed(7)
        pos = torch.randint(0, n, (4096,), device="cuda", generator=g)
        mag = torch.pow(10.0, 6.0 + 3.0 * torch.rand(4096, device="cuda", generator=g))
        sgn = torch.where(torch.rand(4096, device="cuda", generator=g) < 0.5, -1.0, 1.0)
        x[pos] = (mag * sgn).float()
    got, want, rep = _c4_gpu_and_reference(x)
    del x
    rel_close(got, want, RTOL32)
    inf_err, rel_big = precision(got, want)
    # outliers go through the exact fp64 diversion; lognormal's mid-size mass
    # stays in fixed point at a coarse scale (its rms is set by the tail)
    assert rel_big < (1e-3 if kind == "lognormal4" else 1e-4), (rep, inf_err, rel_big)


def test_dense_beyond_2e32_elements(cuda):
    """64-bit indexing: a 1024 x 2048 x 2049 fp32 tensor (4.3e9 elements, 17 GB)
    through the fp32 fixed-point kernel, per bucket against the fp64 kernel on
    the widened tensor and by the zeroth moment (see test_dense_c4_full_size)."""
    import ctypes as C
    from paper_2106_13062_b200 import _lib as L
    dims = [1024, 2048, 2049]
    n = int(np.prod(dims))
    assert n > 2 ** 32
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    L.check(L.lib().st_device_gaussian(L.ST_F32, 77, n, C.c_void_p(x.data_ptr()), None))
    fams = st.families_for(dims, st.EstimatorConfig(4096, 2, 11))
    got = st.fcs_dense_batched(st.DenseTensor(dims, x), fams)
    x64 = x.double()
    del x
    ref = st.fcs_dense_batched(st.DenseTensor(dims, x64), fams)
    rel_close(got, ref.cpu().numpy(), RTOL32)
    X = x64.view(dims[2], dims[1], dims[0])
    norm = float(torch.linalg.vector_norm(x64))
    for d, f in enumerate(fams):
        s = [torch.tensor(f.pair(k).sign_map(), dtype=torch.float64, device="cuda") for k in range(3)]
        m0 = float(((X @ s[0]) @ s[1]) @ s[2])
        assert abs(float(got[d].sum()) - m0) <= 1e-3 * norm, (d, float(got[d].sum()), m0)
    del x64, X
    torch.cuda.empty_cache()


def test_dense_global_fallback(cuda):
    """fp64 sketch larger than shared memory (J~ = 29998 -> 240 KB): global path."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal((30, 20, 10))
    fams = st.families_for([30, 20, 10], st.EstimatorConfig(10000, 2, 8))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams)
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        rel_close(got[d], O.fcs_dense(x, b, s, j), RTOL64)


def test_dense_slabs_sum_to_full(cuda):
    """Element sharding by the last mode (the multi-GPU partition): partial
    sketches of the slabs add up to the full sketch (linearity)."""
    from paper_2106_13062_b200 import dist
    rng = np.random.default_rng(6)
    x = rng.integers(-4, 5, size=(40, 30, 24)).astype(np.float64)
    t = st.DenseTensor.from_array(x)
    fams = st.families_for([40, 30, 24], st.EstimatorConfig(50, 3, 1))
    full = st.fcs_dense_batched(t, fams)
    acc = torch.zeros_like(full)
    for rank in range(5):
        acc += dist.shard_sketch(t, fams, rank, 5)
    assert torch.equal(acc, full)


def test_dense_zero_and_empty_effects(cuda):
    x = np.zeros((8, 9, 10))
    fams = st.families_for([8, 9, 10], st.EstimatorConfig(5, 2, 1))
    assert (st.fcs_dense_batched(st.DenseTensor.from_array(x), fams) == 0).all()


def test_dense_errors(cuda):
    fam = st.HashFamily([4, 5], 3, 1)
    with pytest.raises(ValueError):
        st.fcs_sketch(np.ones((5, 4)), fam)
    with pytest.raises(ValueError):
        st.fcs_sketch(np.ones((4, 5, 1)), fam)
    with pytest.raises(ValueError):
        st.DenseTensor([3, 0])


# ------------------------------------------------------------- CS / CP
def test_cs_kat_and_columns(cuda):
    pair = st.HashPair(bucket_map=[0, 1, 0], sign_map=[1, -1, 1], hash_len=2)
    assert st.cs_sketch([1.0, 2.0, 3.0], pair).values.cpu().tolist() == [4.0, -2.0]
    p = st.HashPair(400, 4000, 12)
    u = np.random.default_rng(1).standard_normal((400, 7))
    got = st.cs_sketch_columns(u, p).cpu().numpy()
    want = O.cs_sketch_columns(u, p.bucket_map(), p.sign_map(), 4000)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-14)


def test_cp_golden(cuda):
    fs = [GOLD[f"cp_f{i}"] for i in range(3)]
    fam = st.HashFamily([10, 12, 14], 9, st.family_seed(4, 2))
    got = st.fcs_sketch(st.CpTensor(GOLD["cp_w"], fs), fam).values
    rel_close(got, GOLD["cp_sketch"], RTOL64)
    rel_close(got, GOLD["cp_dense_sketch"], 1e-9)  # path identity


def test_cp_c2_full(cuda):
    """BASELINE config 2: CP 400^3, R=50, J=4000 (J~=11998), D=10."""
    c = configs.C2
    w, fs = configs.c2_cp(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_cp_batched(st.CpTensor(w, fs), fams)
    assert got.shape == (10, 11998)
    for d in (0, 7):
        b, s, j = oracle_family(fams[d])
        rel_close(got[d], O.fcs_cp(w, fs, b, s, j), RTOL64)


def test_full_configs_vs_reference(cuda):
    """BASELINE configs 1, 2, 3 and 5 at full size against the unmodified reference
    (oracle/_ref, shim FFT): the dense sketch of config 1, the CP sketch of config 2 (all 10 families), the
    config-3 engine's T(I,u,u) / T(u,u,u) and deflation, and config 5's
    Kronecker composition (reference fcs_sketch of each operand with its two
    pairs, then the reference fft_convolve)."""
    from oracle import ref
    c = configs.C1
    x = configs.c1_tensor(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
    rel_close(got[0], ref.fcs_dense(x, c.hash_len, ref.family_seed(c.seed, 0)), RTOL64)
    c = configs.C2
    w, fs = configs.c2_cp(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_cp_batched(st.CpTensor(w, fs), fams).cpu().numpy()
    for d in range(c.sketch_count):
        rel_close(got[d], ref.fcs_cp(w, fs, c.hash_len, ref.family_seed(c.seed, d)), RTOL64)
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, c.sketch_count,
                                                                        c.seed))
    reng = ref.Engine(t, c.hash_len, c.sketch_count, c.seed)
    u = V[:, 0] + 0.2 * V[:, 3]
    rel_close(eng.iuu(u), reng.iuu(u), RTOL64)
    rel_close(eng.uuu(u), reng.uuu(u), RTOL64)
    eng.deflate(lam[0], V[:, 0], V[:, 0], V[:, 0])
    reng.deflate(lam[0], V[:, 0], V[:, 0], V[:, 0])
    rel_close(eng.iuu(u), reng.iuu(u), RTOL64)
    c = configs.C5
    A, B = configs.c5_matrices(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_kron(A, B, fams).cpu().numpy()
    for d in (0, 3, 7):
        b, sg, _ = ref.hash_family(list(c.dims), c.hash_len, ref.family_seed(c.seed, d))
        fa = ref.fcs_dense_tables(A, [b[0], b[1]], [sg[0], sg[1]], [c.hash_len] * 2)
        fb = ref.fcs_dense_tables(B, [b[2], b[3]], [sg[2], sg[3]], [c.hash_len] * 2)
        want = ref.fft_convolve([fa, fb], len(fa) + len(fb) - 1)
        rel_close(got[d], want, RTOL64)


def test_ts_hcs_full_size_vs_reference(cuda):
    """The (f1) sketches and engines at BASELINE sizes against the unmodified
    reference: TS and HCS of the config-1 tensor (100^3, J = 1000 / 8 per mode),
    the TS and Plain engines at the config-3 geometry (200^3, J = 3000, D = 10):
    T(I,u,u), T(u,u,u), and TS of the config-2 CP tensor."""
    from oracle import ref
    c = configs.C1
    x = configs.c1_tensor(c)
    fam = st.HashFamily(list(c.dims), c.hash_len, st.family_seed(c.seed, 0))
    b, sg, j = oracle_family(fam)
    rel_close(st.ts_sketch(x, fam).values, ref.ts_dense_tables(x, b, sg, j), RTOL64)
    fam8 = st.HashFamily(list(c.dims), 8, st.family_seed(c.seed, 1))
    b8, s8, j8 = oracle_family(fam8)
    rel_close(st.hcs_sketch(x, fam8).values, ref.hcs_dense_tables(x, b8, s8, j8), RTOL64)
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    eng = st.make_contraction_engine(st.DenseTensor.from_array(t), st.SketchBackend.TS,
                                     st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    reng = ref.Engine(t, c.hash_len, c.sketch_count, c.seed, backend=ref.BACKEND_TS)
    u = V[:, 1] - 0.3 * V[:, 2]
    rel_close(eng.iuu(u), reng.iuu(u), RTOL64)
    rel_close(eng.uuu(u), reng.uuu(u), RTOL64)
    # the Plain (exact, the reference factory's default) engine at the same size
    peng = st.make_contraction_engine(st.DenseTensor.from_array(t), st.SketchBackend.Plain,
                                      st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    rpeng = ref.Engine(t, c.hash_len, c.sketch_count, c.seed, backend=ref.BACKEND_PLAIN)
    rel_close(peng.iuu(u), rpeng.iuu(u), RTOL64)
    rel_close(peng.uuu(u), rpeng.uuu(u), RTOL64)
    # TS of the config-2 CP tensor (all ten families' first and last)
    c = configs.C2
    w, fs = configs.c2_cp(c)
    cp = st.CpTensor(w, fs)
    for d in (0, 9):
        fam = st.HashFamily(list(c.dims), c.hash_len, st.family_seed(c.seed, d))
        b, sg, j = oracle_family(fam)
        rel_close(st.ts_sketch(cp, fam).values, ref.ts_cp_tables(w, fs, b, sg, j), RTOL64)


def test_cp_vs_dense_path(cuda):
    """fcs_cp == fcs_dense(densify) on a random rank-5 10x12x14."""
    rng = np.random.default_rng(3)
    fs = [rng.standard_normal((d, 5)) for d in (10, 12, 14)]
    w = rng.standard_normal(5)
    fams = st.families_for([10, 12, 14], st.EstimatorConfig(33, 3, 8))
    cp = st.fcs_cp_batched(st.CpTensor(w, fs), fams)
    dense = st.fcs_dense_batched(st.DenseTensor.from_array(configs.densify(w, fs)), fams)
    rel_close(cp, dense.cpu().numpy(), 1e-9)


def test_convolve_pairs(cuda):
    rng = np.random.default_rng(2)
    a, b = rng.standard_normal((3, 4095)), rng.standard_normal((3, 4095))
    got = st.convolve_pairs(torch.from_numpy(a), torch.from_numpy(b)).cpu().numpy()
    for i in range(3):
        rel_close(got[i], np.convolve(a[i], b[i]), 1e-11)
    k = st.convolve_pairs(torch.tensor([[1.0, 2.0]]), torch.tensor([[2.0, 0.0]]))
    np.testing.assert_allclose(k.cpu().numpy()[0], [2, 4, 0], atol=1e-14)


# ------------------------------------------------------------ Kronecker
def test_kron_c5_and_slice(cuda):
    """BASELINE config 5: FCS(A (x) B) = conv(FCS(A), FCS(B)), J=2048, D=8; checked
    against the oracle composition and, on 64x64 slices, against the direct dense
    FCS of the explicit Kronecker product (shape (I3,I1,I4,I2), family (p2,p0,p3,p1))."""
    c = configs.C5
    A, B = configs.c5_matrices(c)
    fams = st.families_for(list(c.dims), st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed))
    got = st.fcs_kron(A, B, fams)
    assert got.shape == (8, 8189)
    for d in (0, 5):
        b, s, j = oracle_family(fams[d])
        fa = O.fcs_dense(A, b[:2], s[:2], j[:2])
        fb = O.fcs_dense(B, b[2:], s[2:], j[2:])
        rel_close(got[d], np.convolve(fa, fb), RTOL64)
    # slice check (prefix property: families over dims 64 are prefixes of the 512 ones)
    As, Bs = A[:64, :64], B[:64, :64]
    fams64 = st.families_for([64] * 4, st.EstimatorConfig(c.hash_len, 2, c.seed))
    got64 = st.fcs_kron(As, Bs, fams64)
    K = np.kron(As, Bs).reshape((64, 64, 64, 64), order="F")  # (i3, i1, i4, i2)
    for d in range(2):
        b, s, j = oracle_family(fams64[d])
        perm = [2, 0, 3, 1]
        direct = O.fcs_dense(K, [b[p] for p in perm], [s[p] for p in perm], [j[p] for p in perm])
        rel_close(got64[d], direct, 1e-9)


# ------------------------------------------------------------ estimators
def test_engine_golden(cuda):
    eng = st.FcsEngine(st.DenseTensor.from_array(GOLD["eng_t"]), st.EstimatorConfig(6, 3, 5))
    u, v, w = GOLD["eng_u"], GOLD["eng_v"], GOLD["eng_w"]
    rel_close(eng.iuu(u), GOLD["eng_iuu"], RTOL64)
    rel_close(eng.iuv(u, v, 1), GOLD["eng_iuv1"], RTOL64)
    rel_close(eng.iuv(u, v, 2), GOLD["eng_iuv2"], RTOL64)
    rel_close(eng.uvw(u, v, w), GOLD["eng_uvw"][0], RTOL64)
    eng.deflate(0.7, u, v, w)
    rel_close(eng.iuu(u), GOLD["eng_defl_iuu"], RTOL64)
    rel_close(eng.uvw(u, v, w), GOLD["eng_defl_uvw"][0], RTOL64)
    with pytest.raises(ValueError):
        eng.iuv(u, v, 3)
    with pytest.raises(ValueError):
        eng.iuv(u[:5], v, 0)


def test_engine_medium_batched(cuda):
    """Batched T(I,u,u) and T(u,u,u) for 15 vectors at once vs the oracle engine
    (60^3, J=300, D=10 — the c3 estimator with a smaller tensor)."""
    rng = np.random.default_rng(8)
    t = rng.standard_normal((60, 60, 60))
    cfg = st.EstimatorConfig(300, 10, 3)
    eng = st.FcsEngine(st.DenseTensor.from_array(t), cfg)
    oeng = O.FcsEngine(t, 300, 10, 3)
    U = rng.standard_normal((15, 60))
    got = eng.iuv_batch(U, U, 0).cpu().numpy()
    vals = eng.uvw_batch(U, U, U).cpu().numpy()
    for l in (0, 9, 14):
        rel_close(got[l], oeng.iuu(U[l]), RTOL64)
        rel_close(vals[l], oeng.uuu(U[l]), RTOL64)
    # sketches survive the round trip through the cached spectra
    rel_close(eng.sketches()[2], oeng.pres[2].values, 1e-12)


def test_engine_c3_size(cuda):
    """BASELINE config 3 estimator geometry: 200^3, J=3000 (J~=8998), D=10."""
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(c.hash_len, 10, c.seed))
    oeng = O.FcsEngine(t, c.hash_len, 10, c.seed)
    u = V[:, 0] + 0.1 * V[:, 1]
    rel_close(eng.iuu(u), oeng.iuu(u), RTOL64)
    rel_close(eng.uuu(u), oeng.uuu(u), RTOL64)


def test_rtpm_golden(cuda):
    cfg = st.RtpmConfig(target_rank=2, num_inits=3, num_power_iters=5, backend=st.SketchBackend.FCS,
                        estimator=st.EstimatorConfig(12, 3, 21))
    cp = st.rtpm(st.DenseTensor.from_array(GOLD["rtpm_t"]), cfg)
    rel_close(cp.weights, GOLD["rtpm_weights"], 1e-8)
    f = cp._factors_cm[0].t()
    rel_close(f, GOLD["rtpm_factor"], 1e-8)


def test_device_gaussian_distribution(cuda):
    import ctypes as C
    from paper_2106_13062_b200 import _lib
    x = torch.empty(1 << 22, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().st_device_gaussian(_lib.ST_F32, 4, x.numel(), C.c_void_p(x.data_ptr()),
                                             None))
    torch.cuda.synchronize()
    assert abs(float(x.mean())) < 3e-3 and abs(float(x.std()) - 1) < 3e-3
    h = configs.host_gaussian(4, 1000)
    np.testing.assert_allclose(x[:1000].cpu().numpy(), h.astype(np.float32), rtol=1e-6, atol=1e-6)


# ---------------------------------------------------- fp32 fixed-point path
def _f32_case(x, J=300, D=3, seed=5):
    fams = st.families_for(list(x.shape), st.EstimatorConfig(J, D, seed))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
    want = []
    for f in fams:
        b, s, j = oracle_family(f)
        want.append(O.fcs_dense(x.astype(np.float64), b, s, j))
    return got, np.stack(want)


def test_dense_f32_outlier_fallback(cuda):
    """An outlier the scale sample misses overflows the int32 fixed point; the
    CTA must detect it and redo its chunk with float accumulation."""
    rng = np.random.default_rng(21)
    x = rng.standard_normal((256, 64, 48)).astype(np.float32)
    x[17, 33, 40] = 3.0e9
    x[200, 5, 1] = -7.5e8
    got, want = _f32_case(x)
    rel_close(got, want, RTOL32)
    # the buckets that receive no outlier, against their own scale (the
    # outliers' buckets would otherwise set the ||c||_inf pad for all of them)
    fams = st.families_for(list(x.shape), st.EstimatorConfig(300, 3, 5))
    mask = np.ones_like(want, bool)
    for d, f in enumerate(fams):
        for idx in ((17, 33, 40), (200, 5, 1)):
            mask[d, sum(int(f.pair(n).bucket_map()[i]) for n, i in enumerate(idx))] = False
    rel_close(got[mask], want[mask], RTOL32)


@pytest.mark.parametrize("sigma", [1e-6, 1e-10, 1e-30])
def test_dense_f32_small_magnitude(cuda, sigma):
    """Small-magnitude fp32 data keeps its relative accuracy: the sampled
    fixed-point exponent grows with 1/sigma (up to 2^120) instead of being
    capped, so elements are not rounded away (advisor round 1)."""
    rng = np.random.default_rng(31)
    x = (sigma * rng.standard_normal((256, 64, 48))).astype(np.float32)
    got, want = _f32_case(x.astype(np.float32))
    rel_close(got, want, RTOL32)


def test_dense_f32_scale_invariant(cuda):
    """Scaling the input by 2^-k (exact in fp32) shifts the fixed-point
    exponent by exactly k: the sketch of 2^-k x is bit-identical to 2^-k times
    the sketch of x, down to 2^-90 (S = 109)."""
    rng = np.random.default_rng(33)
    x = rng.standard_normal((512, 64, 40)).astype(np.float32)
    base, _ = _f32_case(x)
    for k in (20, 33, 90):
        got, _ = _f32_case((x * np.float32(2.0 ** -k)).astype(np.float32))
        assert np.array_equal(got, base * 2.0 ** -k), k


@pytest.mark.parametrize("sigma", [1.0, 1e-30])
def test_dense_f32_sample_misses_data(cuda, sigma):
    """Every sampled fiber is zero (the scale sample reads fibers k * F / 2048,
    here every 16th fiber): the exponent defaults to the top (2^120), so data
    of ordinary magnitude trips the exact range check and each CTA redoes its
    chunk with float atomics; tiny data is represented at full resolution."""
    rng = np.random.default_rng(32)
    x = (sigma * rng.standard_normal((128, 512, 64))).astype(np.float32)
    fib = x.reshape(128, -1, order="F")
    fib[:, ::16] = 0.0  # the sampled fibers (32768 fibers, 2048 samples)
    x = fib.reshape(x.shape, order="F")
    got, want = _f32_case(x, J=200)
    rel_close(got, want, RTOL32)


def test_dense_f32_biased_data(cuda):
    """All-positive data (mean 100): the sampled scale must keep partials in range."""
    rng = np.random.default_rng(22)
    x = (100.0 + rng.standard_normal((512, 32, 40))).astype(np.float32)
    got, want = _f32_case(x, J=64)
    rel_close(got, want, RTOL32)


def test_dense_f32_nan_propagates(cuda):
    x = np.ones((128, 8, 8), np.float32)
    x[3, 4, 5] = np.nan
    got, want = _f32_case(x, J=50, D=2)
    assert (np.isnan(got) == np.isnan(want)).all()
    rel_close(np.nan_to_num(got), np.nan_to_num(want), RTOL32)


def test_dense_f32_unaligned_pointer(cuda):
    """An fp32 tensor that is not 16-byte aligned takes the generic kernel."""
    rng = np.random.default_rng(23)
    base = torch.from_numpy(rng.standard_normal(64 * 16 * 8 + 1).astype(np.float32)).cuda()
    flat = base[1:]
    t = st.DenseTensor([64, 16, 8], flat)
    fams = st.families_for([64, 16, 8], st.EstimatorConfig(40, 2, 3))
    got = st.fcs_dense_batched(t, fams).cpu().numpy()
    x = flat.cpu().numpy().astype(np.float64).reshape((64, 16, 8), order="F")
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        rel_close(got[d], O.fcs_dense(x, b, s, j), RTOL32)


def test_rtpm_c3_per_call(cuda):
    """BASELINE config 3 (200^3, J=3000, D=10, 15 restarts x 20 iterations, R=10).
    At this size the sketch noise dominates the signal (||noise||_F ~ 28 vs
    lambda in [1, 2]), so RTPM trajectories are chaotic: two exact-arithmetic-
    equivalent oracle runs (FFT length J~ vs a padded length) already end in
    different components. Parity is therefore checked per call
    on the actual batched iterates, and the full run must complete finitely."""
    import math
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    est = st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed)
    cp = st.rtpm(st.DenseTensor.from_array(t),
                 st.RtpmConfig(c.rank, configs.C3_INITS, configs.C3_ITERS,
                                backend=st.SketchBackend.FCS, estimator=est))
    assert np.isfinite(cp.weights.cpu().numpy()).all()
    eng = st.FcsEngine(st.DenseTensor.from_array(t), est)
    oeng = O.FcsEngine(t, c.hash_len, c.sketch_count, c.seed)
    rng = O.SplitMix64(O.mix(c.seed ^ 0x7274706D))
    U = np.stack([O.random_unit(rng, 200) for _ in range(configs.C3_INITS)])
    for it in range(3):  # the first power iterations of all 15 restarts, batched
        Y = eng.iuv_batch(U, U, 0).cpu().numpy()
        vals = eng.uvw_batch(U, U, U).cpu().numpy()
        for l in (0, 7, 14):
            rel_close(Y[l], oeng.iuu(U[l]), RTOL64)
            rel_close(vals[l], oeng.uuu(U[l]), RTOL64)
        U = Y / np.linalg.norm(Y, axis=1, keepdims=True)


def test_rtpm_well_conditioned_vs_oracle(cuda):
    """End-to-end rtpm parity where the sketch resolves the components."""
    rng = np.random.default_rng(31)
    q, _ = np.linalg.qr(rng.standard_normal((40, 3)))
    t = configs.densify([3.0, 2.0, 1.5], [q, q, q]) + 1e-4 * rng.standard_normal((40, 40, 40))
    est = st.EstimatorConfig(1000, 5, 17)
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(3, 5, 10, st.SketchBackend.FCS, est))
    w, f = O.rtpm(O.FcsEngine(t, 1000, 5, 17), 40, 3, 5, 10, 17)
    rel_close(cp.weights, w, 1e-8)
    rel_close(cp._factors_cm[0].t(), f, 1e-8)
    assert np.allclose(np.sort(w)[::-1], [3.0, 2.0, 1.5], atol=0.15)


def test_dense_host_entry_slabs(cuda):
    """st_fcs_dense_host (host buffers, chunked H2D/compute pipeline) on a slab
    [lo, hi) of the last mode equals the device path's partial for that slab."""
    import ctypes as C
    from paper_2106_13062_b200 import _lib as L
    from paper_2106_13062_b200 import dist
    rng = np.random.default_rng(41)
    dims = [128, 24, 40]
    x = rng.standard_normal(dims).astype(np.float32)
    fams = st.families_for(dims, st.EstimatorConfig(300, 3, 12))
    t = st.DenseTensor.from_array(x)
    lens = L.size_array([300] * 3)
    seeds = L.u64_array([f.master_seed() for f in fams])
    for rank, world in ((0, 1), (1, 3), (2, 3)):
        lo, hi = dist.shard_range(dims[-1], rank, world)
        host = np.ascontiguousarray(x[:, :, lo:hi].ravel(order="F"))
        out = np.empty((3, 898), np.float64)
        L.check(L.lib().st_fcs_dense_host(L.ST_F32, host.ctypes.data_as(C.c_void_p), 3,
                                          L.size_array(dims), lo, hi - lo, 3, seeds, lens,
                                          out.ctypes.data_as(C.c_void_p)))
        xs = np.zeros_like(x, dtype=np.float64)
        xs[:, :, lo:hi] = x[:, :, lo:hi]
        want = np.stack([O.fcs_dense(xs, *oracle_family(f)) for f in fams])
        rel_close(out, want, RTOL32)


# ------------------------------------------------------------ TS / HCS (§8(f))
def test_ts_hcs_golden(cuda):
    x = GOLD["dense_small_x"]
    fam = st.HashFamily([6, 5, 4], 7, st.family_seed(6, 0))
    rel_close(st.ts_sketch(x, fam).values, GOLD["ts_dense"], RTOL64)
    rel_close(st.hcs_sketch(x, fam).values, GOLD["hcs_dense"], RTOL64)
    fs = [GOLD[f"tscp_f{i}"] for i in range(3)]
    cp = st.CpTensor(GOLD["tscp_w"], fs)
    rel_close(st.ts_sketch(cp, fam).values, GOLD["ts_cp"], RTOL64)
    rel_close(st.hcs_sketch(cp, fam).values, GOLD["hcs_cp"], RTOL64)
    with pytest.raises(ValueError):
        st.ts_sketch(x, st.HashFamily([6, 5, 4], [7, 7, 8], 3))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ts_hcs_dense_vs_oracle(cuda, dtype):
    rng = np.random.default_rng(51)
    x = rng.standard_normal((96, 40, 30)).astype(dtype)
    fam = st.HashFamily([96, 40, 30], 25, st.family_seed(8, 2))
    b, s, j = oracle_family(fam)
    tol = RTOL64 if dtype == np.float64 else RTOL32
    xd = x.astype(np.float64)
    rel_close(st.ts_sketch(x, fam).values, O.ts_sketch(xd, b, s, j), tol)
    rel_close(st.hcs_sketch(x, fam).values, O.hcs_sketch(xd, b, s, j), tol)


def test_ts_hcs_cp_vs_oracle(cuda):
    rng = np.random.default_rng(52)
    fs = [rng.standard_normal((d, 6)) for d in (50, 40, 30)]
    w = rng.standard_normal(6)
    w[2] = 0.0
    fam = st.HashFamily([50, 40, 30], 20, st.family_seed(9, 0))
    b, s, j = oracle_family(fam)
    cp = st.CpTensor(w, fs)
    rel_close(st.ts_sketch(cp, fam).values, O.ts_cp(w, fs, b, s, j), RTOL64)
    rel_close(st.hcs_sketch(cp, fam).values, O.hcs_cp(w, fs, b, s, j), RTOL64)
    # path identities: TS/HCS of CP == TS/HCS of the densified tensor
    dense = configs.densify(w, fs)
    rel_close(st.ts_sketch(cp, fam).values, st.ts_sketch(dense, fam).values.cpu().numpy(), 1e-9)
    rel_close(st.hcs_sketch(cp, fam).values, st.hcs_sketch(dense, fam).values.cpu().numpy(), 1e-9)


# ------------------------------------------------- K1 fp64 fixed point (fx64)
def _f64_case(x, J, D, seed=5):
    fams = st.families_for(list(x.shape), st.EstimatorConfig(J, D, seed))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
    want = []
    for f in fams:
        b, s, j = oracle_family(f)
        want.append(O.fcs_dense(x, b, s, j))
    return got, np.stack(want)


@pytest.mark.parametrize("shape,J,D", [((1024, 64, 128), 3000, 1),  # NV = 32, full fibers
                                       ((100, 300, 300), 1000, 1),  # NV = 4, partial
                                       ((37, 500, 500), 800, 1),    # NV = 2, partial
                                       ((512, 40, 40), 2048, 8),    # NV = 16, D = 8
                                       ((300, 120, 60, 4), 500, 2)])  # order 4, NV = 16 partial
def test_dense_f64_fixed_point_integer_bitexact(cuda, shape, J, D):
    """fp64 fixed point (64-bit partials as two int32 words with exact carries,
    >= 8M element-updates per call): integer data sums exactly, so the result
    equals the reference's serial fp64 sum bit for bit."""
    rng = np.random.default_rng(sum(shape) + J)
    x = rng.integers(-1000, 1001, size=shape).astype(np.float64)
    got, want = _f64_case(x, J, D)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("shape,J,D", [((2048, 70, 60), 3000, 1),   # 2 full segments of 1024
                                       ((3000, 50, 60), 2000, 1),   # 4 segments of 768, last 696
                                       ((1100, 90, 90), 1500, 1),   # 2 segments of 576 / 524
                                       ((16384, 24, 24), 4096, 1)])  # 16 segments (the limit)
def test_dense_f64_fixed_point_long_fibers(cuda, shape, J, D):
    """I_0 > 1024: each fiber split into 2^l segments, one warp per segment
    (fx_segments): integer data bit-exact against the reference's serial sum,
    Gaussian data at the fp64 rule."""
    rng = np.random.default_rng(sum(shape))
    x = rng.integers(-1000, 1001, size=shape).astype(np.float64)
    got, want = _f64_case(x, J, D)
    assert np.array_equal(got, want)
    x = rng.standard_normal(shape)
    got, want = _f64_case(x, J, D)
    rel_close(got, want, RTOL64)


@pytest.mark.parametrize("shape,J,D", [((256, 200, 200), 10000, 1),   # J~ = 29,998: 2 ranges
                                       ((300, 150, 190), 20000, 2),   # J~ = 59,998: 3 ranges
                                       ((2048, 80, 64), 12000, 1),    # ranges x segments
                                       ((64, 200, 700), 22000, 1)])   # J~ = 65,998 >= 2^16: global
def test_dense_f64_fixed_point_bucket_ranges(cuda, shape, J, D):
    """fp64 with J~ beyond shared memory: the fixed point over R bucket
    ranges, one CTA per (chunk, family, range) (formerly fp64 global
    atomics). Integer data bit-exact, Gaussian data at the fp64 rule, and an
    outlier that sends one range's CTA to its fp64-atomic redo."""
    rng = np.random.default_rng(sum(shape) + J)
    x = rng.integers(-1000, 1001, size=shape).astype(np.float64)
    got, want = _f64_case(x, J, D)
    assert np.array_equal(got, want)
    x = rng.standard_normal(shape)
    x[5, 7, 9] = 4.0e22
    got, want = _f64_case(x, J, D)
    rel_close(got, want, RTOL64)


@pytest.mark.parametrize("shape,J,D", [((512, 128, 128), 25000, 1),   # J~ = 74,998: 2 ranges
                                       ((1024, 96, 96), 40000, 2)])   # J~ = 119,998: 3 ranges
def test_dense_f32_fixed_point_bucket_ranges(cuda, shape, J, D):
    """fp32 with J~ beyond shared memory (int32 buckets): the scalar-load
    fixed point over bucket ranges (formerly fp64 global atomics). Integer
    data bit-exact; Gaussian data at the fp32 rule; an outlier sends its
    range CTA to the float redo."""
    rng = np.random.default_rng(sum(shape) + J)
    fams = st.families_for(list(shape), st.EstimatorConfig(J, D, 8))
    for kind in ("int", "gauss"):
        x = (rng.integers(-8, 9, size=shape) if kind == "int"
             else rng.standard_normal(shape)).astype(np.float32)
        if kind == "gauss":
            x[3, 5, 7] = 2.0e9
        got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
        for d, f in enumerate(fams):
            b, s_, j = oracle_family(f)
            want = O.fcs_dense(x.astype(np.float64), b, s_, j)
            if kind == "int":
                assert np.array_equal(got[d], want), d
            else:
                rel_close(got[d], want, RTOL32)


@pytest.mark.parametrize("shape", [(2048, 64, 66), (1100, 90, 90), (3001, 50, 60)])
def test_dense_f32_fixed_point_long_fibers(cuda, shape):
    """fp32 with I_0 > 1024 (formerly fp32 shared atomics): the scalar-load
    int32 fixed point over fiber segments, at the fp32 rule against the oracle
    and bit-identical across runs."""
    rng = np.random.default_rng(sum(shape) + 1)
    x = rng.standard_normal(shape).astype(np.float32)
    fams = st.families_for(list(shape), st.EstimatorConfig(2500, 2, 3))
    t = st.DenseTensor.from_array(x)
    got = st.fcs_dense_batched(t, fams)
    assert torch.equal(st.fcs_dense_batched(t, fams), got)
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        rel_close(got[d], O.fcs_dense(x.astype(np.float64), b, s, j), RTOL32)


def test_dense_f64_fixed_point_gaussian(cuda):
    """Gaussian fp64 data through the fixed point at the fp64 rule, and the
    large buckets to 1e-12 relative (quantum 2^-(S+1) per element, S ~ 48)."""
    rng = np.random.default_rng(41)
    x = rng.standard_normal((1024, 96, 96))
    got, want = _f64_case(x, 4096, 1)
    rel_close(got, want, RTOL64)
    big = np.abs(want) > 1e-3 * np.abs(want).max()
    assert np.all(np.abs(got - want)[big] <= 1e-12 * np.abs(want)[big])


def test_dense_f64_fixed_point_deterministic(cuda):
    rng = np.random.default_rng(42)
    x = rng.standard_normal((256, 200, 200))
    fams = st.families_for([256, 200, 200], st.EstimatorConfig(2000, 2, 9))
    t = st.DenseTensor.from_array(x)
    first = st.fcs_dense_batched(t, fams)
    for _ in range(2):
        assert torch.equal(st.fcs_dense_batched(t, fams), first)


def test_dense_f64_fixed_point_outliers_and_nan(cuda):
    """Outliers beyond the fixed-point range (2^51 quanta) and NaN: the CTA
    that sees one redoes its chunk with fp64 atomics; results at the rule,
    NaN propagated to the buckets that receive it."""
    rng = np.random.default_rng(43)
    x = rng.standard_normal((200, 200, 200))
    x[17, 33, 40] = 3.0e25
    x[150, 5, 190] = -7.5e18
    got, want = _f64_case(x, 3000, 1)
    rel_close(got, want, RTOL64)
    x[3, 4, 5] = np.nan
    got, want = _f64_case(x, 3000, 1)
    assert (np.isnan(got) == np.isnan(want)).all()
    rel_close(np.nan_to_num(got), np.nan_to_num(want), RTOL64)


@pytest.mark.parametrize("sigma", [1e-150, 1e150])
def test_dense_f64_fixed_point_extreme_magnitude(cuda, sigma):
    rng = np.random.default_rng(44)
    x = sigma * rng.standard_normal((128, 250, 256))
    got, want = _f64_case(x, 1500, 1)
    rel_close(got, want, RTOL64)


# -------------------------------------------------------- sparse (COO) FCS
def _coo(shape, density, seed, dtype=np.float64):
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    nnz = max(1, int(n * density))
    flat = rng.choice(n, size=nnz, replace=False)
    coords = np.stack(np.unravel_index(flat, shape, order="F"), axis=1).astype(np.int64)
    vals = rng.standard_normal(nnz).astype(dtype)
    dense = np.zeros(shape, dtype=np.float64)
    dense[tuple(coords.T)] = vals
    return vals, coords, dense


@pytest.mark.parametrize("density", [0.01, 0.001])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sparse_coo_vs_reference(cuda, density, dtype):
    """FCS from a COO list equals the unmodified reference's fcs_sketch of the
    densified tensor (1 % and 0.1 % density; fp64 at the fp64 rule, fp32 values
    widened exactly)."""
    from oracle import ref
    shape = (120, 90, 70)
    vals, coords, dense = _coo(shape, density, 50 + int(1e4 * density), dtype)
    fams = st.families_for(list(shape), st.EstimatorConfig(400, 3, 8))
    got = st.fcs_coo_batched(vals, coords, shape, fams).cpu().numpy()
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        rel_close(got[d], ref.fcs_dense_tables(dense, b, s, j), RTOL64)


def test_sparse_coo_duplicates_zeros_errors(cuda):
    shape = (7, 5, 4)
    fams = st.families_for(list(shape), st.EstimatorConfig(9, 2, 3))
    coords = np.array([[1, 2, 3], [1, 2, 3], [6, 4, 0], [0, 0, 0]])
    vals = np.array([1.5, -0.25, 2.0, 0.0])
    dense = np.zeros(shape)
    dense[1, 2, 3] = 1.25
    dense[6, 4, 0] = 2.0
    got = st.fcs_coo_batched(vals, coords, shape, fams).cpu().numpy()
    for d, f in enumerate(fams):
        b, s, j = oracle_family(f)
        np.testing.assert_array_equal(got[d], O.fcs_dense(dense, b, s, j))
    empty = st.fcs_coo_batched(np.zeros(0), np.zeros((0, 3)), shape, fams)
    assert torch.count_nonzero(empty) == 0
    with pytest.raises(ValueError, match="compose: index out of range"):
        st.fcs_coo_batched([1.0], [[7, 0, 0]], shape, fams)


def test_sparse_coo_c4_geometry(cuda):
    """Config-4 geometry (1024^3, J = 16384, D = 4) at 0.1 % density (1.07M
    nonzeros): the COO sketch equals K1 (fp64, itself pinned to the
    reference) on the densified tensor."""
    shape = (1024, 1024, 1024)
    rng = np.random.default_rng(77)
    nnz = (1 << 30) // 1000
    flat = np.unique(rng.integers(0, 1 << 30, size=nnz, dtype=np.int64))
    coords = np.stack(np.unravel_index(flat, shape, order="F"), axis=1)
    vals = rng.standard_normal(flat.size)
    fams = st.families_for(list(shape), st.EstimatorConfig(16384, 4, 4))
    got = st.fcs_coo_batched(vals, coords, shape, fams)
    dense = torch.zeros(1 << 30, dtype=torch.float64, device="cuda")
    dense[torch.from_numpy(flat).cuda()] = torch.from_numpy(vals).cuda()
    want = st.fcs_dense_batched(st.DenseTensor(list(shape), dense), fams)
    rel_close(got, want.cpu().numpy(), RTOL64)


@pytest.mark.parametrize("shape,J,D", [((1022, 96, 90), 2000, 1), ((333, 200, 130), 1500, 1)])
def test_dense_f32_odd_fiber_fixed_point(cuda, shape, J, D):
    """fp32 tensors whose fibers the float4 kernel cannot take (I_0 % 4 != 0)
    go through the same int32 fixed point with scalar loads: integer data
    bit-exact, Gaussian data at the fp32 rule."""
    rng = np.random.default_rng(sum(shape))
    xi = rng.integers(-50, 51, size=shape).astype(np.float32)
    fams = st.families_for(list(shape), st.EstimatorConfig(J, D, 6))
    got = st.fcs_dense_batched(st.DenseTensor.from_array(xi), fams).cpu().numpy()
    for d, f in enumerate(fams):
        b, s_, j = oracle_family(f)
        assert np.array_equal(got[d], O.fcs_dense(xi.astype(np.float64), b, s_, j))
    xg = rng.standard_normal(shape).astype(np.float32)
    got = st.fcs_dense_batched(st.DenseTensor.from_array(xg), fams).cpu().numpy()
    for d, f in enumerate(fams):
        b, s_, j = oracle_family(f)
        rel_close(got[d], O.fcs_dense(xg.astype(np.float64), b, s_, j), RTOL32)


# ------------------------------------------- cluster (8-CTA, DSMEM) estimator
@pytest.mark.parametrize("dims,J,D,seed", [((30, 24, 18), 2500, 5, 7),   # M = 8192 instantiation
                                           ((20, 26, 31), 3000, 4, 8),   # M = 9216 (config-3 J)
                                           ((22, 19, 27), 1800, 3, 9),   # M = 6144 (radix-6 pass)
                                           ((17, 23, 21), 4000, 3, 10),  # M = 12288 (radix 12)
                                           ((25, 20, 16), 1000, 4, 11),  # M = 3072
                                           ((16, 18, 20), 650, 3, 12)])  # M = 2048
def test_cluster_estimator_vs_oracle(cuda, spectral_path, dims, J, D, seed):
    """The cluster estimator (spectral_cluster.cu) on both of its transform
    lengths, every free mode (non-cubic, so the contracted-mode tables differ),
    with the median fused in (batch 1 and 3: one wave of clusters) and without
    it (per-family estimates), against the oracle engine; a batch beyond one
    wave takes the one-CTA kernel and must agree too."""
    rng = np.random.default_rng(seed)
    t = rng.standard_normal(dims)
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, D, seed))
    oeng = O.FcsEngine(t, J, D, seed)
    for f in range(3):
        c1 = 1 if f == 0 else 0
        c2 = 1 if f == 2 else 2
        for n in (1, 3, 16):
            A = rng.standard_normal((n, dims[c1]))
            B = rng.standard_normal((n, dims[c2]))
            got = eng.iuv_batch(A, B, f).cpu().numpy()
            per = eng.iuv_batch(A, B, f, median=False).cpu().numpy()
            for b in (0, n - 1):
                rel_close(got[b], oeng.iuv(A[b], B[b], f), RTOL64)
                for d in (0, D - 1):
                    want = O.iuv_spectral(oeng.pres[d], A[b], B[b], f)
                    rel_close(per[b, d], want, RTOL64)
    # T(u, v, w) as <w, T(u, v, I)> per family on the cluster estimator (median fused)
    for n in (1, 4):
        U, V, W = (rng.standard_normal((n, dims[m])) for m in range(3))
        got = eng.uvw_batch(U, V, W).cpu().numpy()
        for b in range(n):
            want = oeng.uvw(U[b], V[b], W[b])
            assert abs(got[b] - want) <= RTOL64 * 2 * abs(want) + 1e-300, (got[b], want)


def test_rtpm_cluster_tail_vs_oracle(cuda, spectral_path):
    """rtpm where both phases take the fused cluster tail (J = 2500 -> M = 8192;
    5 restarts x 5 families and the batch-1 refinement fit one wave): the
    median + row normalisation (restarts) and the refinement update with its
    sticky underflow stop equal the oracle's rtpm; a zero tensor exercises the
    underflow branches (rows become 0, the refinement stops at once)."""
    rng = np.random.default_rng(37)
    q, _ = np.linalg.qr(rng.standard_normal((36, 3)))
    t = configs.densify([3.0, 2.0, 1.5], [q, q, q]) + 1e-4 * rng.standard_normal((36, 36, 36))
    est = st.EstimatorConfig(2500, 5, 19)
    cp = st.rtpm(st.DenseTensor.from_array(t), st.RtpmConfig(3, 5, 8, st.SketchBackend.FCS, est))
    w, f = O.rtpm(O.FcsEngine(t, 2500, 5, 19), 36, 3, 5, 8, 19)
    rel_close(cp.weights, w, 1e-8)
    rel_close(cp._factors_cm[0].t(), f, 1e-8)
    assert np.allclose(np.sort(w)[::-1], [3.0, 2.0, 1.5], atol=0.15)
    z = np.zeros((12, 12, 12))
    cpz = st.rtpm(st.DenseTensor.from_array(z), st.RtpmConfig(2, 3, 4, st.SketchBackend.FCS,
                                                             st.EstimatorConfig(2500, 3, 5)))
    wz, fz = O.rtpm(O.FcsEngine(z, 2500, 3, 5), 12, 2, 3, 4, 5)
    np.testing.assert_array_equal(cpz.weights.cpu().numpy(), wz)
    np.testing.assert_array_equal(cpz._factors_cm[0].t().cpu().numpy(), fz)


def test_cluster_estimator_edges_vs_oracle(cuda, spectral_path):
    """Cluster estimator edges: a free mode longer than the early-gather
    registers (nf = 300 > 256), D = 17 (the fused median's general branch),
    the TS engine (the FCS kernels on the J-periodic extension, J = 2500 ->
    M = 8192), a NaN in a vector (non-finite median branch) and zero vectors."""
    rng = np.random.default_rng(53)
    dims = (300, 22, 18)
    t = rng.standard_normal(dims)
    J = 2500
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, 17, 4))
    oeng = O.FcsEngine(t, J, 17, 4)
    A = rng.standard_normal((2, dims[1]))
    B = rng.standard_normal((2, dims[2]))
    got = eng.iuv_batch(A, B, 0).cpu().numpy()
    for b in range(2):
        rel_close(got[b], oeng.iuv(A[b], B[b], 0), RTOL64)
    A[1, 3] = np.nan
    got = eng.iuv_batch(A, B, 0).cpu().numpy()
    want = oeng.iuv(A[1], B[1], 0)
    assert (np.isnan(got[1]) == np.isnan(want)).all()
    rel_close(got[0], oeng.iuv(A[0], B[0], 0), RTOL64)
    z = eng.iuv_batch(np.zeros((1, dims[1])), np.zeros((1, dims[2])), 0).cpu().numpy()
    assert np.array_equal(z, np.zeros((1, dims[0])))
    ts = st.TsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(J, 5, 6))
    ots = O.TsEngine(t, J, 5, 6)
    for f in range(3):
        c1 = 1 if f == 0 else 0
        c2 = 1 if f == 2 else 2
        a, b = rng.standard_normal(dims[c1]), rng.standard_normal(dims[c2])
        rel_close(ts.iuv(a, b, f), ots.iuv(a, b, f), 1e-9)


def test_cluster_estimator_repeatable(cuda, spectral_path):
    """Race check for the DSMEM exchanges, cluster barriers and the fused tail:
    100 rounds of back-to-back calls (T(I,u,v) at batch 1 and 4 with the fused
    median, and T(u,v,w)) must all agree with the first result to fp64
    round-off (compute-sanitizer is unavailable on this pool)."""
    rng = np.random.default_rng(61)
    t = rng.standard_normal((20, 18, 16))
    eng = st.FcsEngine(st.DenseTensor.from_array(t), st.EstimatorConfig(2500, 5, 13))
    A = torch.as_tensor(rng.standard_normal((4, 18)), device="cuda")
    B = torch.as_tensor(rng.standard_normal((4, 16)), device="cuda")
    V = torch.as_tensor(rng.standard_normal((4, 18)), device="cuda")
    U = torch.as_tensor(rng.standard_normal((4, 20)), device="cuda")
    first = [x.cpu().numpy() for x in
             [eng.iuv_batch(A[:n], B[:n], 0) for n in (1, 4)] + [eng.uvw_batch(U, V, B)]]
    outs = []
    for _ in range(100):
        outs.append([eng.iuv_batch(A[:n], B[:n], 0) for n in (1, 4)] + [eng.uvw_batch(U, V, B)])
    torch.cuda.synchronize()
    for o in outs:
        for g, f in zip(o, first):
            rel_close(g, f, 1e-12)


def test_dense_fuzz_paths_vs_oracle(cuda):
    """Seeded random shapes through every K1 path (shared-memory atomics,
    fp32 float4 / scalar-load fixed point, fp64 fixed point, fiber segments,
    bucket ranges, global atomics): integer data must match the reference's
    serial sum bit for bit, whatever path the planner picks."""
    rng = np.random.default_rng(2024)
    cases = []
    for _ in range(6):   # small calls: shared-memory atomic kernels
        cases.append((tuple(int(v) for v in rng.integers(3, 40, size=3)), int(rng.integers(20, 400)),
                      int(rng.integers(1, 5)), rng.choice([np.float32, np.float64])))
    cases += [((1024, 96, 88), 700, 1, np.float32),     # float4 fixed point
              ((1021, 97, 86), 900, 2, np.float32),     # scalar-load fixed point (I0 % 4 != 0)
              ((2500, 60, 56), 1100, 1, np.float32),    # fiber segments (fp32)
              ((700, 120, 100), 1300, 1, np.float64),   # fp64 fixed point
              ((1500, 80, 70), 2000, 1, np.float64),    # fp64 fiber segments
              ((300, 160, 180), 11000, 1, np.float64),  # fp64 bucket ranges
              ((300, 160, 180), 21000, 1, np.float32),  # fp32 bucket ranges
              ((40, 50, 60), 30000, 1, np.float64)]     # beyond shared memory, small: global
    for shape, J, D, dt in cases:
        x = rng.integers(-6, 7, size=shape).astype(dt)
        fams = st.families_for(list(shape), st.EstimatorConfig(J, D, int(rng.integers(1, 1 << 30))))
        got = st.fcs_dense_batched(st.DenseTensor.from_array(x), fams).cpu().numpy()
        for d, f in enumerate(fams):
            b, s_, j = oracle_family(f)
            want = O.fcs_dense(x.astype(np.float64), b, s_, j)
            assert np.array_equal(got[d], want), (shape, J, D, dt, d)
