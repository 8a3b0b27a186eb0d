"""ORACLE TEST INFRASTRUCTURE — not product code.

A numpy restatement of the reference's fast-count-sketch (FCS) path, one
function per reference function, each citing the file:line it follows
(paths relative to /root/reference/proj). It is the CPU checker for the
CUDA product in ``paper_2106_13062_b200``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg may use it.

Pinning: this restatement is checked against (a) the spec's hand-derived
known-answer tests, (b) golden vectors in ``tests/golden/`` produced by the
UNMODIFIED reference sources compiled in ``oracle/_ref`` (see
``tests/golden/make_golden.py``), and (c) the reference library itself
through ``oracle/ref.py`` wherever it is buildable.

Numerics: integer hash work is bit-exact by construction. The dense scatter
uses ``np.bincount`` which adds weights sequentially in input order, i.e.
in the reference's flat column-major order (sketch.cpp:48-61,187-201), so
dense FCS values are bit-identical to the reference. FFT paths use numpy's
pocketfft at the reference's exact length n (FFTW in the reference), so they
agree to fp64 round-off, not bit-for-bit.
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK64 = (1 << 64) - 1


# --------------------------------------------------------------------- L0 RNG
def fmix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 output mix (rng.hpp:18-20), vectorised over uint64."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix_draw(seed: int, k) -> np.ndarray:
    """k-th draw (1-based) of SplitMix64(seed): state advances by GAMMA before
    mixing (rng.hpp:16-21), so draw k = fmix64(seed + k*GAMMA)."""
    k = np.asarray(k, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return fmix64(np.uint64(seed & _MASK64) + k * GAMMA)


def mix(v: int) -> int:
    """SplitMix64::mix (rng.hpp:42): first draw of a generator seeded with v."""
    return int(splitmix_draw(v, 1))


def mulhi64(a: np.ndarray, b: int) -> np.ndarray:
    """(uint128(a) * b) >> 64, the Lemire reduction of next_below (rng.hpp:25-28)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.uint64(b)
    lo32 = np.uint64(0xFFFFFFFF)
    a_lo, a_hi = a & lo32, a >> np.uint64(32)
    b_lo, b_hi = b & lo32, b >> np.uint64(32)
    with np.errstate(over="ignore"):
        ll = a_lo * b_lo
        lh = a_lo * b_hi
        hl = a_hi * b_lo
        hh = a_hi * b_hi
        mid = (ll >> np.uint64(32)) + (lh & lo32) + (hl & lo32)
        return hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))


class SplitMix64:
    """Sequential SplitMix64 with the Box–Muller spare (rng.hpp:12-48, rng.cpp:8-21).
    Pure-Python (math.log/sin/cos = the host libm the reference links), used
    only for the small RTPM initialisation streams."""

    def __init__(self, seed: int):
        self.state = seed & _MASK64
        self.spare = 0.0
        self.has_spare = False

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        return z ^ (z >> 31)

    def next_gaussian(self) -> float:
        if self.has_spare:
            self.has_spare = False
            return self.spare
        u1 = float((self.next() >> 11) + 1) * 2.0 ** -53
        u2 = float(self.next() >> 11) * 2.0 ** -53
        radius = math.sqrt(-2.0 * math.log(u1))
        angle = 2.0 * math.pi * u2
        self.spare = radius * math.sin(angle)
        self.has_spare = True
        return radius * math.cos(angle)


# ----------------------------------------------------------------- L1 hashing
def hash_pair(input_dim: int, hash_len: int, seed: int):
    """HashPair(I, J, seed) (hashing.cpp:10-22): for each i in order, bucket
    from draw 2i+1 via next_below, sign from the top bit of draw 2i+2."""
    if input_dim == 0 or hash_len == 0:
        raise ValueError("HashPair: dimensions must be positive")
    i = np.arange(input_dim, dtype=np.uint64)
    bucket = mulhi64(splitmix_draw(seed, 2 * i + 1), hash_len).astype(np.uint32)
    top = splitmix_draw(seed, 2 * i + 2) >> np.uint64(63)
    sign = np.where(top != 0, -1, 1).astype(np.int8)
    return bucket, sign


def family_seed(base_seed: int, d: int) -> int:
    """family_seed (hashing.cpp:123-125)."""
    return mix((base_seed + d) & _MASK64)


def hash_family(dims, hash_lens, master_seed: int):
    """HashFamily ctor (hashing.cpp:42-59): pair n seeded master ^ n."""
    if isinstance(hash_lens, int):
        hash_lens = [hash_lens] * len(dims)
    if len(dims) == 0 or len(dims) != len(hash_lens):
        raise ValueError("HashFamily: need one hash length per mode")
    pairs = [hash_pair(int(d), int(j), master_seed ^ n) for n, (d, j) in
             enumerate(zip(dims, hash_lens))]
    return [p[0] for p in pairs], [p[1] for p in pairs], [int(j) for j in hash_lens]


def composed_len(hash_lens) -> int:
    """HashFamily::composed_len (hashing.cpp:77-81)."""
    return int(sum(hash_lens)) - len(hash_lens) + 1


def families_for(dims, hash_len: int, sketch_count: int, seed: int):
    """families_for (estimators.cpp:104-115)."""
    if hash_len == 0 or sketch_count == 0:
        raise ValueError("EstimatorConfig: hash_len and sketch_count must be >= 1")
    return [hash_family(dims, hash_len, family_seed(seed, d)) for d in range(sketch_count)]


def composed_tables(buckets, signs, dims=None):
    """Composed bucket/sign for every flat index, first mode fastest
    (materialize_composed_pair, hashing.cpp:100-121)."""
    b = np.zeros(1, np.int64)
    s = np.ones(1, np.int64)
    for bn, sn in zip(buckets, signs):  # mode n varies slower than modes < n
        b = (b[None, :] + np.asarray(bn, np.int64)[:, None]).ravel()
        s = (s[None, :] * np.asarray(sn, np.int64)[:, None]).ravel()
    return b, s


# ---------------------------------------------------------------- L2 sketches
def _check_family(shape, buckets, op):
    """require_family_matches (sketch.cpp:12-22)."""
    if len(shape) != len(buckets):
        raise ValueError(f"{op}: family order mismatch")
    for n, bn in enumerate(buckets):
        if shape[n] != len(bn):
            raise ValueError(f"{op}: shape mismatch")


def fcs_dense(t: np.ndarray, buckets, signs, hash_lens, chunk: int = 1 << 24) -> np.ndarray:
    """fcs_sketch(DenseTensor, HashFamily) (sketch.cpp:187-201): serial
    scatter in flat column-major order (odometer, sketch.cpp:48-61), zeros
    skipped. ``t`` is an ndarray whose Fortran order is the reference layout
    (or a flat vector when dims are taken from the tables)."""
    t = np.asarray(t)
    shape = t.shape if t.ndim > 1 else tuple(len(b) for b in buckets)
    _check_family(shape, buckets, "fcs_sketch")
    n_out = composed_len(hash_lens)
    flat = t.ravel(order="F") if t.ndim > 1 else t
    out = np.zeros(n_out, np.float64)
    # Mode-0 tables broadcast against the composed tables of modes >= 1.
    b0 = np.asarray(buckets[0], np.int64)
    s0 = np.asarray(signs[0], np.float64)
    rest_b, rest_s = composed_tables(buckets[1:], signs[1:]) if len(buckets) > 1 else (
        np.zeros(1, np.int64), np.ones(1, np.int64))
    i0 = len(b0)
    fibers_per_chunk = max(1, chunk // i0)
    for f0 in range(0, len(rest_b), fibers_per_chunk):
        f1 = min(len(rest_b), f0 + fibers_per_chunk)
        v = np.asarray(flat[f0 * i0:f1 * i0], np.float64)
        bk = (rest_b[f0:f1, None] + b0[None, :]).ravel()
        sg = (rest_s[f0:f1, None].astype(np.float64) * s0[None, :]).ravel()
        nz = v != 0.0
        # np.add.at is unbuffered and applied in index order: the serial
        # reference sum values[bucket] += sign * value, chunk after chunk.
        np.add.at(out, bk[nz], sg[nz] * v[nz])
    return out


def cs_sketch(x, bucket, sign, hash_len: int) -> np.ndarray:
    """cs_sketch (sketch.cpp:105-116)."""
    x = np.asarray(x, np.float64)
    if len(x) != len(bucket):
        raise ValueError("cs_sketch: input length mismatch")
    nz = x != 0.0
    return np.bincount(np.asarray(bucket, np.int64)[nz],
                       weights=np.asarray(sign, np.float64)[nz] * x[nz], minlength=hash_len)


def cs_sketch_columns(u, bucket, sign, hash_len: int) -> np.ndarray:
    """cs_sketch_columns (sketch.cpp:118-133): I x R -> J x R."""
    u = np.asarray(u, np.float64)
    if u.shape[0] != len(bucket):
        raise ValueError("cs_sketch_columns: input length mismatch")
    out = np.zeros((hash_len, u.shape[1]), np.float64)
    for r in range(u.shape[1]):
        out[:, r] = cs_sketch(u[:, r], bucket, sign, hash_len)
    return out


# -------------------------------------------------------------------- L1 FFT
def dft(x, n: int) -> np.ndarray:
    """dft (fft.cpp:42-51): zero-pad or truncate to n, forward e^{-i}."""
    if n == 0:
        raise ValueError("dft: zero length")
    buf = np.zeros(n, np.complex128)
    x = np.asarray(x, np.float64)
    m = min(n, len(x))
    buf[:m] = x[:m]
    return np.fft.fft(buf)


def idft_real(spec) -> np.ndarray:
    """idft_real (fft.cpp:53-73): backward e^{+i}, x 1/n, real part, residue check."""
    spec = np.asarray(spec, np.complex128)
    n = len(spec)
    if n == 0:
        raise ValueError("idft_real: zero length")
    out = np.fft.ifft(spec)
    re, im = out.real, out.imag
    if math.sqrt(float(im @ im)) > 1e-9 * math.sqrt(float(re @ re)) + 1e-12:
        raise RuntimeError("idft_real: inverse transform is not real")
    return re.copy()


def fft_convolve(inputs, n: int) -> np.ndarray:
    """fft_convolve (fft.cpp:75-84)."""
    if len(inputs) == 0:
        raise ValueError("fft_convolve: no inputs")
    acc = dft(inputs[0], n)
    for x in inputs[1:]:
        acc = acc * dft(x, n)
    return idft_real(acc)


def convolved_cp_sketch(weights, factors, buckets, signs, hash_lens, n: int) -> np.ndarray:
    """convolved_cp_sketch (sketch.cpp:65-86): per-rank FFT convolution of the
    per-mode column count sketches, weighted sum over r (zero weights skipped)."""
    cs = [cs_sketch_columns(f, b, s, j) for f, b, s, j in zip(factors, buckets, signs, hash_lens)]
    out = np.zeros(n, np.float64)
    for r, w in enumerate(np.asarray(weights, np.float64)):
        if w == 0.0:
            continue
        out += w * fft_convolve([c[:, r] for c in cs], n)
    return out


def fcs_cp(weights, factors, buckets, signs, hash_lens) -> np.ndarray:
    """fcs_sketch(CpTensor, HashFamily) (sketch.cpp:203-207)."""
    _check_family(tuple(f.shape[0] for f in factors), buckets, "fcs_sketch")
    return convolved_cp_sketch(weights, factors, buckets, signs, hash_lens,
                               composed_len(hash_lens))


def ts_sketch(t: np.ndarray, buckets, signs, hash_lens) -> np.ndarray:
    """ts_sketch(DenseTensor) (sketch.cpp:135-149): buckets mod J, equal J."""
    if len(set(hash_lens)) != 1:
        raise ValueError("ts_sketch: all hash lengths must be equal")
    _check_family(t.shape, buckets, "ts_sketch")
    b, s = composed_tables(buckets, signs)
    v = t.ravel(order="F")
    nz = v != 0.0
    return np.bincount(b[nz] % hash_lens[0], weights=s[nz] * v[nz], minlength=hash_lens[0])


def hcs_sketch(t: np.ndarray, buckets, signs, hash_lens) -> np.ndarray:
    """hcs_sketch(DenseTensor) (sketch.cpp:157-173): per-mode buckets into a
    J_1 x ... x J_N tensor (returned with Fortran-order layout)."""
    _check_family(t.shape, buckets, "hcs_sketch")
    flat = np.zeros(1, np.int64)
    sg = np.ones(1, np.int64)
    stride = 1
    for bn, sn, j in zip(buckets, signs, hash_lens):
        flat = (flat[None, :] + stride * np.asarray(bn, np.int64)[:, None]).ravel()
        sg = (sg[None, :] * np.asarray(sn, np.int64)[:, None]).ravel()
        stride *= j
    v = t.ravel(order="F")
    nz = v != 0.0
    out = np.bincount(flat[nz], weights=sg[nz] * v[nz], minlength=stride)
    return out.reshape(tuple(hash_lens), order="F")


# ------------------------------------------------------------- L3 estimators
def median_reduce(values):
    """median_reduce (estimators.cpp:117-138): even count -> mean of the two
    middle order statistics; vectors reduce elementwise."""
    v = np.asarray(values, np.float64)
    if v.size == 0:
        raise ValueError("median_reduce: empty input")
    s = np.sort(v, axis=0)
    n = s.shape[0]
    if n % 2 == 1:
        return s[n // 2]
    return 0.5 * (s[n // 2 - 1] + s[n // 2])


class PrecomputedFcs:
    """PrecomputedFcs (estimators.cpp:140-149): sketch + cached n-point DFT."""

    def __init__(self, values, buckets, signs, hash_lens):
        self.values = np.asarray(values, np.float64)
        self.buckets, self.signs, self.hash_lens = buckets, signs, hash_lens
        self.n = composed_len(hash_lens)
        if len(self.values) != self.n:
            raise ValueError("SketchVec: length contract violated")
        self.spectrum = dft(self.values, self.n)


def _contracted_modes(free_mode: int, op: str):
    """contracted_modes (estimators.cpp:23-29)."""
    if free_mode > 2:
        raise ValueError(f"{op}: mode out of range")
    return (1 if free_mode == 0 else 0), (1 if free_mode == 2 else 2)


def uvw_spectral(pre: PrecomputedFcs, u, v, w) -> float:
    """uvw_spectral + spectral_dot (estimators.cpp:38-64)."""
    if len(pre.buckets) != 3:
        raise ValueError("estimate_uvw: order-3 family required")
    for x, m in ((u, 0), (v, 1), (w, 2)):
        if len(x) != len(pre.buckets[m]):
            raise ValueError("estimate_uvw: vector length mismatch")
    n = pre.n
    g = dft(cs_sketch(u, pre.buckets[0], pre.signs[0], pre.hash_lens[0]), n)
    fv = dft(cs_sketch(v, pre.buckets[1], pre.signs[1], pre.hash_lens[1]), n)
    fw = dft(cs_sketch(w, pre.buckets[2], pre.signs[2], pre.hash_lens[2]), n)
    g = g * (fv * fw)
    return float(np.sum((pre.spectrum * np.conj(g)).real) / n)


def precompute_z(pre: PrecomputedFcs, a, b, free_mode: int) -> np.ndarray:
    """precompute_z (estimators.cpp:151-167)."""
    c1, c2 = _contracted_modes(free_mode, "precompute_z")
    n = pre.n
    fa = dft(cs_sketch(a, pre.buckets[c1], pre.signs[c1], pre.hash_lens[c1]), n)
    fb = dft(cs_sketch(b, pre.buckets[c2], pre.signs[c2], pre.hash_lens[c2]), n)
    return idft_real(pre.spectrum * np.conj(fa) * np.conj(fb))


def iuv_spectral(pre: PrecomputedFcs, a, b, free_mode: int) -> np.ndarray:
    """iuv_spectral (estimators.cpp:66-90): out_i = s_f(i) z[h_f(i)]."""
    if len(pre.buckets) != 3:
        raise ValueError("estimate_iuv: order-3 family required")
    c1, c2 = _contracted_modes(free_mode, "estimate_iuv")
    if len(a) != len(pre.buckets[c1]) or len(b) != len(pre.buckets[c2]):
        raise ValueError("estimate_iuv: vector length mismatch")
    z = precompute_z(pre, a, b, free_mode)
    return np.asarray(pre.signs[free_mode], np.float64) * z[np.asarray(pre.buckets[free_mode],
                                                                       np.int64)]


def estimate_uvw(pres, u, v, w) -> float:
    """estimate_uvw (estimators.cpp:169-174) via median_over (:92-100)."""
    if len(pres) == 0:
        raise ValueError("estimator: no sketches")
    return float(median_reduce([uvw_spectral(p, u, v, w) for p in pres]))


def estimate_iuv(pres, a, b, free_mode: int) -> np.ndarray:
    """estimate_iuv (estimators.cpp:180-186)."""
    if len(pres) == 0:
        raise ValueError("estimator: no sketches")
    return median_reduce([iuv_spectral(p, a, b, free_mode) for p in pres])


def precompute_fcs(t, fam) -> PrecomputedFcs:
    """precompute_fcs (estimators.cpp:147-149)."""
    b, s, j = fam
    return PrecomputedFcs(fcs_dense(t, b, s, j), b, s, j)


# -------------------------------------------------------------------- L4 CPD
class FcsEngine:
    """FcsEngine (cpd.cpp:61-94)."""

    def __init__(self, t: np.ndarray, hash_len: int, sketch_count: int, seed: int):
        self.shape = t.shape
        self.pres = [precompute_fcs(t, fam) for fam in
                     families_for(t.shape, hash_len, sketch_count, seed)]

    def uvw(self, u, v, w) -> float:
        return estimate_uvw(self.pres, u, v, w)

    def iuv(self, a, b, free_mode: int) -> np.ndarray:
        return estimate_iuv(self.pres, a, b, free_mode)

    def uuu(self, u) -> float:
        return self.uvw(u, u, u)

    def iuu(self, u) -> np.ndarray:
        return self.iuv(u, u, 0)

    def deflate(self, weight: float, u, v, w):
        """cpd.cpp:79-87: values -= fcs_sketch(rank_one(weight, {u,v,w}))."""
        facs = [np.asarray(x, np.float64).reshape(-1, 1) for x in (u, v, w)]
        for i, p in enumerate(self.pres):
            comp = fcs_cp([weight], facs, p.buckets, p.signs, p.hash_lens)
            self.pres[i] = PrecomputedFcs(p.values - comp, p.buckets, p.signs, p.hash_lens)


def random_unit(rng: SplitMix64, dim: int) -> np.ndarray:
    """random_unit (cpd.cpp:199-204)."""
    v = np.array([rng.next_gaussian() for _ in range(dim)], np.float64)
    norm = math.sqrt(float(v @ v))
    return v / norm if norm > 0 else v


def normalize_or_zero(v: np.ndarray):
    """normalize_or_zero (cpd.cpp:208-216); returns (vector, ok)."""
    norm = math.sqrt(float(v @ v))
    if norm < 1e-150:
        return np.zeros_like(v), False
    return v / norm, True


def rtpm(engine, dim: int, rank: int, num_inits: int, num_iters: int, seed: int):
    """rtpm (cpd.cpp:234-277) over any engine with iuu/uuu/deflate."""
    if rank == 0 or num_inits == 0 or num_iters == 0:
        raise ValueError("rtpm: rank, inits, and iterations must be >= 1")
    init_rng = SplitMix64(mix(seed ^ 0x7274706D))
    weights = np.zeros(rank)
    factor = np.zeros((dim, rank))
    for r in range(rank):
        best, best_value = None, -math.inf
        for _ in range(num_inits):
            u = random_unit(init_rng, dim)
            for _ in range(num_iters):
                u, ok = normalize_or_zero(engine.iuu(u))
                if not ok:
                    break
            value = engine.uuu(u)
            if value > best_value:
                best_value, best = value, u
        for _ in range(num_iters):
            nxt, ok = normalize_or_zero(engine.iuu(best))
            if not ok:
                break
            best = nxt
        weight = engine.uuu(best)
        weights[r] = weight
        factor[:, r] = best
        engine.deflate(weight, best, best, best)
    return weights, factor


# ------------------------------------------------------------ synthetic data
def gaussian_stream(seed: int, n: int) -> np.ndarray:  # noqa: D401
    """n draws of SplitMix64(seed).next_gaussian() (rng.cpp:8-21), vectorised
    via the counter identity (draw k = fmix64(seed + k*GAMMA)): pair p uses
    draws 2p+1 (u1) and 2p+2 (u2) and yields (r cos, r sin). numpy's SIMD
    log/cos can differ from glibc by 1 ulp on ~0.1% of draws; the sequential
    ``SplitMix64.next_gaussian`` above is the bit-exact form."""
    pairs = (n + 1) // 2
    p = np.arange(pairs, dtype=np.uint64)
    d1 = splitmix_draw(seed, 2 * p + 1)
    d2 = splitmix_draw(seed, 2 * p + 2)
    u1 = ((d1 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (d2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    radius = np.sqrt(-2.0 * np.log(u1))
    angle = 2.0 * math.pi * u2
    out = np.empty(2 * pairs, np.float64)
    out[0::2] = radius * np.cos(angle)
    out[1::2] = radius * np.sin(angle)
    return out[:n]


def ts_cp(weights, factors, buckets, signs, hash_lens) -> np.ndarray:
    """ts_sketch(CpTensor) (sketch.cpp:151-155): circular convolution at length J."""
    if len(set(hash_lens)) != 1:
        raise ValueError("ts_sketch: all hash lengths must be equal")
    _check_family(tuple(f.shape[0] for f in factors), buckets, "ts_sketch")
    return convolved_cp_sketch(weights, factors, buckets, signs, hash_lens, hash_lens[0])


def hcs_cp(weights, factors, buckets, signs, hash_lens) -> np.ndarray:
    """hcs_sketch(CpTensor) (sketch.cpp:175-185): densify of the count-sketched
    factors (tensor.cpp:86-115, zero weights skipped); returns J_0 x ... array."""
    _check_family(tuple(f.shape[0] for f in factors), buckets, "hcs_sketch")
    cs = [cs_sketch_columns(f, b, s, j) for f, b, s, j in zip(factors, buckets, signs, hash_lens)]
    out = np.zeros(tuple(hash_lens))
    for r, w in enumerate(np.asarray(weights, np.float64)):
        if w == 0.0:
            continue
        term = np.asarray(w, np.float64)
        for c in cs:
            term = np.multiply.outer(term, c[:, r])
        out += term
    return out


# ------------------------------------------------ TS engine, CPD drivers (§8(f))
class PrecomputedTs(PrecomputedFcs):
    """PrecomputedTs (estimators.cpp:209-215): TS sketch + its J-point DFT."""

    def __init__(self, values, buckets, signs, hash_lens):
        self.values = np.asarray(values, np.float64)
        self.buckets, self.signs, self.hash_lens = buckets, signs, hash_lens
        self.n = hash_lens[0]
        if len(self.values) != self.n:
            raise ValueError("PrecomputedTs: TS sketch required")
        self.spectrum = dft(self.values, self.n)


class TsEngine(FcsEngine):
    """TsEngine (cpd.cpp:96-126): estimates by circular correlation at length J
    (estimate_uvw / estimate_iuv over PrecomputedTs, estimators.cpp:221-233)."""

    def __init__(self, t: np.ndarray, hash_len: int, sketch_count: int, seed: int):
        self.shape = t.shape
        self.pres = []
        for b, s, j in families_for(t.shape, hash_len, sketch_count, seed):
            self.pres.append(PrecomputedTs(ts_sketch(t, b, s, j), b, s, j))

    def deflate(self, weight: float, u, v, w):
        """cpd.cpp:115-122: values -= ts_sketch(rank_one(weight, {u,v,w}))."""
        facs = [np.asarray(x, np.float64).reshape(-1, 1) for x in (u, v, w)]
        for i, p in enumerate(self.pres):
            comp = ts_cp([weight], facs, p.buckets, p.signs, p.hash_lens)
            self.pres[i] = PrecomputedTs(p.values - comp, p.buckets, p.signs, p.hash_lens)


def rtpm_asym(engine, dims, rank: int, num_inits: int, num_iters: int, seed: int):
    """rtpm_asym (cpd.cpp:279-335) over any engine with iuv/uvw/deflate."""
    if rank == 0 or num_inits == 0 or num_iters == 0:
        raise ValueError("rtpm_asym: rank, inits, and iterations must be >= 1")
    init_rng = SplitMix64(mix(seed ^ 0x72743161))
    weights = np.zeros(rank)
    factors = [np.zeros((n, rank)) for n in dims]

    def sweep(vecs):
        for m in range(3):
            c1, c2 = _contracted_modes(m, "estimate_iuv")
            vecs[m], _ = normalize_or_zero(engine.iuv(vecs[c1], vecs[c2], m))

    for r in range(rank):
        best, best_value = None, -math.inf
        for _ in range(num_inits):
            vecs = [random_unit(init_rng, n) for n in dims]
            for _ in range(num_iters):
                sweep(vecs)
            value = abs(engine.uvw(*vecs))
            if value > best_value:
                best_value, best = value, list(vecs)
        for _ in range(num_iters):
            sweep(best)
        weight = engine.uvw(*best)
        if weight < 0:
            best[0], weight = -best[0], -weight
        weights[r] = weight
        for n in range(3):
            factors[n][:, r] = best[n]
        engine.deflate(weight, *best)
    return weights, factors


def min_norm_solve(G: np.ndarray, B: np.ndarray) -> np.ndarray:
    """completeOrthogonalDecomposition().solve (Eigen semantics, cpd.cpp:369-370):
    column-pivoted QR, numerical rank #{|r_ii| > eps n max|r_kk|}, then the
    minimum-norm solution of the rank-r trapezoidal system."""
    import scipy.linalg
    n = G.shape[0]
    Q, R, P = scipy.linalg.qr(G, pivoting=True)
    d = np.abs(np.diag(R))
    r = int(np.sum(d > np.finfo(np.float64).eps * n * d.max(initial=0.0)))
    X = np.zeros((n, B.shape[1]))
    if r == 0:
        return X
    c = (Q.T @ B)[:r]
    y = np.linalg.lstsq(R[:r], c, rcond=None)[0]  # minimum-norm for the full-row-rank r x n
    X[P] = y
    return X


def residual_norm(t: np.ndarray, weights, factors) -> float:
    """residual_norm (cpd.cpp:385-392)."""
    a, b, c = factors
    diff = np.einsum("r,ir,jr,kr->ijk", np.asarray(weights, np.float64), a, b, c) - t
    den = float(np.sqrt(np.sum(t * t)))
    num = float(np.sqrt(np.sum(diff * diff)))
    if den == 0.0:
        return 0.0 if num == 0.0 else math.inf
    return num / den


def als(engine, t: np.ndarray, rank: int, max_iters: int, tol: float, seed: int):
    """als (cpd.cpp:337-383); returns (weights, factors, sweeps)."""
    if rank == 0 or max_iters == 0:
        raise ValueError("als: rank and iterations must be >= 1")
    dims = t.shape
    init_rng = SplitMix64(mix(seed ^ 0x616C73))
    factors = [np.stack([random_unit(init_rng, n) for _ in range(rank)], axis=1) for n in dims]
    weights = np.ones(rank)
    prev, sweeps = math.inf, 0
    for sweep in range(max_iters):
        for mode in range(3):
            o1, o2 = _contracted_modes(mode, "als")
            mttkrp = np.stack([engine.iuv(factors[o1][:, r], factors[o2][:, r], mode)
                               for r in range(rank)], axis=1)
            gram = (factors[o1].T @ factors[o1]) * (factors[o2].T @ factors[o2])
            f = min_norm_solve(gram, mttkrp.T).T
            for r in range(rank):
                norm = math.sqrt(float(f[:, r] @ f[:, r]))
                weights[r] = norm
                if norm > 1e-150:
                    f[:, r] /= norm
            factors[mode] = f
        residual = residual_norm(t, weights, factors)
        sweeps = sweep + 1
        if abs(prev - residual) < tol:
            break
        prev = residual
    return weights.copy(), factors, sweeps


# ------------------------------------------ inner products, regression, codecs
def inner_once(a, b, buckets, signs, hash_lens) -> float:
    """inner_once (estimators.cpp:193-196)."""
    if a.shape != b.shape:
        raise ValueError("inner_once: shape mismatch")
    return float(fcs_dense(a, buckets, signs, hash_lens) @ fcs_dense(b, buckets, signs, hash_lens))


def inner_once_ts(a, b, buckets, signs, hash_lens) -> float:
    """inner_once_ts (estimators.cpp:235-239)."""
    if a.shape != b.shape:
        raise ValueError("inner_once_ts: shape mismatch")
    return float(ts_sketch(a, buckets, signs, hash_lens) @ ts_sketch(b, buckets, signs, hash_lens))


def estimate_inner(a, b, hash_len: int, sketch_count: int, seed: int) -> float:
    """estimate_inner (estimators.cpp:198-207)."""
    if a.shape != b.shape:
        raise ValueError("estimate_inner: shape mismatch")
    return float(median_reduce([inner_once(a, b, *f) for f in
                                families_for(a.shape, hash_len, sketch_count, seed)]))


def regression_forward(x_rows, w_rows, bias, dims, hash_len: int, sketch_count: int,
                       seed: int) -> np.ndarray:
    """Y = median_d FCS_d(X rows) FCS_d(W rows)^T + b (PAPER.md
    Eq. 20); rows are column-major order-N tensors of shape dims."""
    dims = tuple(int(d) for d in dims)
    X = np.asarray(x_rows, np.float64).reshape(-1, int(np.prod(dims)))
    W = np.asarray(w_rows, np.float64).reshape(-1, int(np.prod(dims)))
    ests = []
    for f in families_for(dims, hash_len, sketch_count, seed):
        sx = np.stack([fcs_dense(x.reshape(dims, order="F"), *f) for x in X])
        sw = np.stack([fcs_dense(w.reshape(dims, order="F"), *f) for w in W])
        ests.append(sx @ sw.T)
    y = median_reduce(ests)
    return y + (0.0 if bias is None else np.asarray(bias, np.float64)[None, :])


def kron_tensor(a, b) -> np.ndarray:
    """A (x) B as the order-4 tensor K[i1, i2, i3, i4] = A[i1, i2] B[i3, i4]
    (the Kronecker matrix entry at row I3 i1 + i3, col I4 i2 + i4)."""
    return np.einsum("ij,kl->ijkl", np.asarray(a, np.float64), np.asarray(b, np.float64))


def contraction_tensor(a, b) -> np.ndarray:
    """A (x)_{3,1} B: C[i1, i2, i3, i4] = sum_l A[i1, i2, l] B[l, i3, i4]."""
    return np.einsum("ijl,lkm->ijkm", np.asarray(a, np.float64), np.asarray(b, np.float64))


def compress_tensor4(t4, hash_len: int, sketch_count: int, seed: int) -> np.ndarray:
    """The defining identity of compress_kron / compress_contraction
    (SPEC.md:403-404): fcs_dense of the materialised order-4 tensor per family."""
    return np.stack([fcs_dense(t4, *f) for f in
                     families_for(t4.shape, hash_len, sketch_count, seed)])


def decompress4(sk, fams, i1, i2, i3, i4) -> float:
    """median_d s1 s2 s3 s4 sk_d[(h1+h2+h3+h4) mod len]."""
    vals = []
    for d, (bk, sg, _) in enumerate(fams):
        h = sum(int(bk[n][i]) for n, i in enumerate((i1, i2, i3, i4)))
        s = int(np.prod([int(sg[n][i]) for n, i in enumerate((i1, i2, i3, i4))]))
        vals.append(s * sk[d][h % sk.shape[1]])
    return float(median_reduce(vals))
