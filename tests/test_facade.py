"""The reference's free-function API defined over the GPU (libsketchtensor_b200.so,
integration/sketchtensor_b200.cpp) and linked with the reference's OWN cpd.cpp,
tensor.cpp, hashing.cpp and rng.cpp in place of sketch.cpp, estimators.cpp and
fft.cpp (integration/_build/test_facade, built by `make -C integration`).
Every output is compared with the unmodified reference (oracle/_ref) on the
same inputs: the config-1 dense FCS, the config-2 CP FCS (D = 10), the
config-5 Kronecker composition (D = 8), rtpm through the reference's own
driver, every engine backend of the reference factory, the exact-length
dft / idft_real / fft_convolve and precompute_z, the TS / HCS / CS sketches,
and the reference's error types and messages."""
import os
import subprocess

import numpy as np
import pytest

from oracle import ref
from paper_2106_13062_b200 import configs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "test_facade")


def rel_close(got, want, rtol):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, (got.shape, want.shape)
    tol = rtol * (np.abs(want) + np.abs(want).max(initial=0.0))
    err = np.abs(got - want)
    assert np.all(err <= tol), f"max err {err.max()} (rel {np.max(err / (tol / rtol + 1e-300))})"


def run(tmp_path, *args):
    assert os.path.exists(BIN), "integration/_build/test_facade missing: make -C integration"
    r = subprocess.run([BIN] + [str(a) for a in args], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr + r.stdout
    return r.stdout


def put(tmp_path, name, arr):
    p = os.path.join(tmp_path, name)
    np.ascontiguousarray(np.asarray(arr, np.float64)).tofile(p)
    return p


def get(tmp_path, name):
    return np.fromfile(os.path.join(tmp_path, name), dtype=np.float64)


def test_facade_fcs_dense_c1(cuda, tmp_path):
    c = configs.C1
    x = configs.c1_tensor(c)
    tp = put(tmp_path, "t.bin", x.ravel(order="F"))
    run(tmp_path, "fcs_dense", tp, c.hash_len, 2, c.seed, os.path.join(tmp_path, "o.bin"),
        *c.dims)
    got = get(tmp_path, "o.bin").reshape(2, -1)
    for d in range(2):
        rel_close(got[d], ref.fcs_dense(x, c.hash_len, ref.family_seed(c.seed, d)), 1e-10)


def test_facade_fcs_cp_c2(cuda, tmp_path):
    c = configs.C2
    w, fs = configs.c2_cp(c)
    wp = put(tmp_path, "w.bin", w)
    fp = put(tmp_path, "f.bin", np.concatenate([np.asarray(f).ravel(order="F") for f in fs]))
    run(tmp_path, "fcs_cp", wp, fp, len(w), c.hash_len, c.sketch_count, c.seed,
        os.path.join(tmp_path, "o.bin"), *c.dims)
    got = get(tmp_path, "o.bin").reshape(c.sketch_count, -1)
    for d in (0, 4, 9):
        rel_close(got[d], ref.fcs_cp(w, fs, c.hash_len, ref.family_seed(c.seed, d)), 1e-10)


def test_facade_kron_c5(cuda, tmp_path):
    c = configs.C5
    A, B = configs.c5_matrices(c)
    ap = put(tmp_path, "a.bin", np.asarray(A).ravel(order="F"))
    bp = put(tmp_path, "b.bin", np.asarray(B).ravel(order="F"))
    run(tmp_path, "kron", ap, bp, 512, 512, 512, 512, c.hash_len, c.sketch_count, c.seed,
        os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin").reshape(c.sketch_count, -1)
    for d in (0, 5):
        b, sg, _ = ref.hash_family(list(c.dims), c.hash_len, ref.family_seed(c.seed, d))
        fa = ref.fcs_dense_tables(A, [b[0], b[1]], [sg[0], sg[1]], [c.hash_len] * 2)
        fb = ref.fcs_dense_tables(B, [b[2], b[3]], [sg[2], sg[3]], [c.hash_len] * 2)
        rel_close(got[d], ref.fft_convolve([fa, fb], len(fa) + len(fb) - 1), 1e-10)


@pytest.mark.parametrize("backend", [ref.BACKEND_FCS, 2])  # FCS, TS
def test_facade_rtpm_reference_driver(cuda, tmp_path, backend):
    """The reference's rtpm (cpd.cpp:234-277), unmodified, on the facade:
    weights and factors equal the reference's on a well-conditioned tensor."""
    q = np.linalg.qr(np.random.default_rng(71).standard_normal((40, 3)))[0]
    t = configs.densify([3.0, 2.0, 1.5], [q, q, q])
    tp = put(tmp_path, "t.bin", t.ravel(order="F"))
    run(tmp_path, "rtpm", tp, 40, 3, 5, 10, backend, 1000, 5, 17, os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin")
    w, f = ref.rtpm(t, 3, 5, 10, 1000, 5, 17, backend=backend)
    rel_close(got[:3], w, 1e-8)
    rel_close(got[3:].reshape((40, 3), order="F"), f, 1e-8)


def test_facade_engine_c3(cuda, tmp_path):
    """The reference's FcsEngine (cpd.cpp:61-94) over the facade at config 3
    (200^3, J = 3000, D = 10): T(u,v,w) and T(I,.,.) at every free mode, then a
    deflation and again, against the reference engine."""
    c = configs.C3
    t, lam, V = configs.c3_tensor(c)
    rng = np.random.default_rng(3)
    vecs = [rng.standard_normal(600) for _ in range(2)]
    _engine_case(tmp_path, t, ref.BACKEND_FCS, c.hash_len, c.sketch_count, c.seed, vecs, 1e-9)


@pytest.mark.parametrize("backend", [0, 1, 2, 3])  # Plain, CS, TS, HCS
def test_facade_engine_backends(cuda, tmp_path, backend):
    rng = np.random.default_rng(80 + backend)
    t = rng.standard_normal((14, 12, 10))
    vecs = [rng.standard_normal(36) for _ in range(2)]
    _engine_case(tmp_path, t, backend, 9, 3, 21, vecs, 1e-9)


def _engine_case(tmp_path, t, backend, J, D, seed, vecs, rtol):
    dims = t.shape
    tp = put(tmp_path, "t.bin", t.ravel(order="F"))
    up = put(tmp_path, "u.bin", np.concatenate(vecs))
    run(tmp_path, "engine", tp, *dims, backend, J, D, seed, up, len(vecs),
        os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin")
    eng = ref.Engine(t, J, D, seed, backend=backend)
    want = []

    def calls():
        for v in vecs:
            v0, v1, v2 = v[:dims[0]], v[dims[0]:dims[0] + dims[1]], v[dims[0] + dims[1]:]
            want.append([eng.uvw(v0, v1, v2)])
            want.append(eng.iuv(v1, v2, 0))
            want.append(eng.iuv(v0, v2, 1))
            want.append(eng.iuv(v0, v1, 2))
    calls()
    v = vecs[0]
    eng.deflate(0.75, v[:dims[0]], v[dims[0]:dims[0] + dims[1]], v[dims[0] + dims[1]:])
    calls()
    off = 0
    for wv in want:
        wv = np.asarray(wv, np.float64)
        rel_close(got[off:off + wv.size], wv, rtol)
        off += wv.size
    assert off == got.size


@pytest.mark.parametrize("n", [7, 2998, 8998, 11998, 49150])
def test_facade_exact_transforms(cuda, tmp_path, n):
    """dft / idft_real / fft_convolve at exactly n points (any n: 8998 =
    2 * 11 * 409, 49150 through the two-level FFT), against the reference."""
    rng = np.random.default_rng(n)
    ln = min(n, 9000) if n > 7 else 12  # n < len exercises the truncation
    x = rng.standard_normal(ln)
    xp = put(tmp_path, "x.bin", x)
    run(tmp_path, "fft", xp, ln, n, os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin")
    spec = got[:2 * n:2] + 1j * got[1:2 * n:2]
    want = ref.dft(x, n)
    assert np.max(np.abs(spec - want)) <= 1e-11 * np.max(np.abs(want))
    rel_close(got[2 * n:3 * n], ref.idft_real(want), 1e-10)
    rel_close(got[3 * n:], ref.fft_convolve([x, x[:ln // 2]], n), 1e-10)


@pytest.mark.parametrize("free_mode", [0, 1, 2])
def test_facade_precompute_z(cuda, tmp_path, free_mode):
    """precompute_z (estimators.cpp:151-167): the WHOLE length-n z vector,
    circular wrap included, against the reference."""
    rng = np.random.default_rng(90 + free_mode)
    t = rng.standard_normal((30, 30, 30))
    a, b = rng.standard_normal(30), rng.standard_normal(30)
    tp = put(tmp_path, "t.bin", t.ravel(order="F"))
    run(tmp_path, "z", tp, 30, 101, 7, put(tmp_path, "a.bin", a), put(tmp_path, "b.bin", b),
        free_mode, os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin")
    n = 3 * 101 - 2
    spec, z = ref.precompute_z(t, 101, ref.family_seed(7, 0), a, b, free_mode)
    g = got[:2 * n:2] + 1j * got[1:2 * n:2]
    assert np.max(np.abs(g - spec)) <= 1e-11 * np.max(np.abs(spec))
    rel_close(got[2 * n:], z, 1e-10)


def test_facade_ts_hcs_cs_sketches(cuda, tmp_path):
    rng = np.random.default_rng(95)
    dims = (20, 16, 12)
    t = rng.standard_normal(dims)
    tv = t.ravel(order="F")
    J, seed = 11, 4
    run(tmp_path, "sketches", put(tmp_path, "t.bin", tv), *dims, J, seed,
        os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin")
    b, s, _ = ref.hash_family(dims, J, ref.family_seed(seed, 0))
    off = 0

    def take(n):
        nonlocal off
        v = got[off:off + n]
        off += n
        return v
    rel_close(take(J), ref.ts_dense_tables(t, b, s, [J] * 3), 1e-10)
    rel_close(take(J ** 3), ref.hcs_dense_tables(t, b, s, [J] * 3).ravel(order="F"), 1e-10)
    rel_close(take(J), ref.cs_sketch(tv[:dims[0]], b[0], s[0], J), 1e-10)
    fs, o = [], 0
    for d in dims:
        fs.append(tv[o:o + 3 * d].reshape((d, 3), order="F"))
        o += 3 * d
    w = np.array([1.0, -0.5, 2.0])
    rel_close(take(J), ref.ts_cp_tables(w, fs, b, s, [J] * 3), 1e-10)
    rel_close(take(J ** 3), ref.hcs_cp_tables(w, fs, b, s, [J] * 3).ravel(order="F"), 1e-10)
    rel_close(take(3 * J - 2), ref.fcs_cp_tables(w, fs, b, s, [J] * 3), 1e-10)
    rel_close(take(3 * J).reshape((J, 3), order="F"),
              ref.cs_sketch_columns(fs[0], b[0], s[0], J), 1e-10)
    assert off == got.size


def test_facade_errors(cuda, tmp_path):
    """The reference's exception types and messages through the facade."""
    out = run(tmp_path, "errors")
    lines = out.strip().splitlines()
    bad = [ln for ln in lines if not (ln.startswith("ok ") or ln.startswith("median "))]
    assert not bad, out
    assert "median 2 2.5" in out
    for msg in ("dft: zero length", "idft_real: inverse transform is not real",
                "fcs_sketch: shape mismatch", "fcs_sketch: family order mismatch",
                "ts_sketch: all hash lengths must be equal", "cs_sketch: input length mismatch",
                "EstimatorConfig: hash_len and sketch_count must be >= 1",
                "median_reduce: empty input", "PrecomputedFcs: FCS sketch required",
                "estimator: no sketches"):
        assert msg in out, msg


@pytest.mark.parametrize("free_mode", [0, 2])
def test_facade_estimators_unequal_hash_lengths(cuda, tmp_path, free_mode):
    """estimate_uvw / estimate_iuv over PrecomputedFcs whose families have
    unequal hash lengths per mode (outside families_for): the facade's
    per-family exact path (st_fft_convolve / st_precompute_z + read-out)
    against the reference."""
    rng = np.random.default_rng(60 + free_mode)
    dims, lens = (18, 14, 11), (37, 29, 23)
    t = rng.standard_normal(dims)
    v = rng.standard_normal(sum(dims))
    run(tmp_path, "mixed", put(tmp_path, "t.bin", t.ravel(order="F")), *dims, *lens, 3, 9,
        put(tmp_path, "v.bin", v), free_mode, os.path.join(tmp_path, "o.bin"))
    got = get(tmp_path, "o.bin")
    u0, u1, u2 = v[:dims[0]], v[dims[0]:dims[0] + dims[1]], v[dims[0] + dims[1]:]
    uvw, iuv = ref.estimate_mixed(t, lens, 3, 9, u0, u1, u2, free_mode)
    rel_close(got[:1], [uvw], 1e-10)
    rel_close(got[1:], iuv, 1e-10)
