"""ORACLE TEST INFRASTRUCTURE — not product code.

ctypes view of the UNMODIFIED reference library built by ``oracle/Makefile``
into ``oracle/_ref/libsketchtensor_ref.so`` (reference sources compiled in
place against the from-scratch Eigen/FFTW shims). Only ``tests/`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module; it is the checker, never the thing measured as the product.

Every wrapper mirrors one reference entry point and cites it. Errors map back
to the reference's exception types: ``std::invalid_argument`` -> ValueError,
``std::runtime_error`` -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libsketchtensor_ref.so")
REFERENCE_ROOT = "/root/reference/proj"

_lib = None

_p = C.c_void_p
_sz = C.c_size_t
_u64 = C.c_uint64
_d = C.c_double


def build() -> bool:
    """Compile oracle/_ref from the reference sources when they are present."""
    if not os.path.isdir(REFERENCE_ROOT):
        return os.path.exists(LIB_PATH)
    subprocess.run(["make", "-s", "-C", _HERE, "-j8"], check=True)
    return True


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_family_seed.restype = _u64
        L.ref_family_seed.argtypes = [_u64, _sz]
        L.ref_splitmix_draws.argtypes = [_u64, _sz, _p]
        L.ref_gaussian.argtypes = [_u64, _sz, _p]
        L.ref_engine_create.restype = _p
        L.ref_engine_create.argtypes = [_p, _p, _sz, _sz, _u64, C.c_int]
        L.ref_engine_destroy.argtypes = [_p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise RuntimeError(msg)
    raise Exception(msg)


def _dims(dims) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))


def splitmix_draws(seed: int, count: int) -> np.ndarray:
    """SplitMix64(seed).next() x count (rng.hpp:16-21)."""
    out = np.empty(count, dtype=np.uint64)
    lib().ref_splitmix_draws(_u64(seed), _sz(count), _ptr(out))
    return out


def family_seed(base: int, d: int) -> int:
    """family_seed (hashing.cpp:123-125)."""
    return int(lib().ref_family_seed(_u64(base), _sz(d)))


def gaussian(seed: int, n: int) -> np.ndarray:
    """n draws of SplitMix64(seed).next_gaussian() (rng.cpp:8-21)."""
    out = np.empty(n, dtype=np.float64)
    lib().ref_gaussian(_u64(seed), _sz(n), _ptr(out))
    return out


def hash_pair(seed: int, input_dim: int, hash_len: int):
    """HashPair(I, J, seed) tables (hashing.cpp:10-22)."""
    b = np.empty(max(input_dim, 1), dtype=np.uint32)
    s = np.empty(max(input_dim, 1), dtype=np.int8)
    _check(lib().ref_hash_pair(_u64(seed), _sz(input_dim), _sz(hash_len), _ptr(b), _ptr(s)))
    return b[:input_dim], s[:input_dim]


def hash_family(dims, hash_len: int, master: int):
    """HashFamily(dims, J, master) (hashing.cpp:42-59); returns (buckets, signs, J~)."""
    dims = _dims(dims)
    tot = int(dims.sum())
    b = np.empty(tot, dtype=np.uint32)
    s = np.empty(tot, dtype=np.int8)
    cl = _sz(0)
    _check(lib().ref_hash_family(_sz(len(dims)), _ptr(dims), _sz(hash_len), _u64(master),
                                 _ptr(b), _ptr(s), C.byref(cl)))
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(np.int64)
    return ([b[offs[n]:offs[n + 1]] for n in range(len(dims))],
            [s[offs[n]:offs[n + 1]] for n in range(len(dims))], int(cl.value))


def _pack_tables(buckets, signs):
    b = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint32) for x in buckets]))
    s = np.ascontiguousarray(np.concatenate([np.asarray(x, np.int8) for x in signs]))
    return b, s


def compose(buckets, signs, hash_lens, multi_index):
    """HashFamily::compose (hashing.cpp:83-98)."""
    dims = _dims([len(x) for x in buckets])
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    mi = _dims(multi_index)
    ob, os_ = _sz(0), C.c_int(0)
    _check(lib().ref_compose(_sz(len(dims)), _ptr(dims), _ptr(b), _ptr(s), _ptr(hl), _ptr(mi),
                             C.byref(ob), C.byref(os_)))
    return int(ob.value), int(os_.value)


def materialize(buckets, signs, hash_lens):
    """HashFamily::materialize_composed_pair (hashing.cpp:100-121)."""
    dims = _dims([len(x) for x in buckets])
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    tot = int(np.prod(dims))
    ob = np.empty(tot, np.uint32)
    os_ = np.empty(tot, np.int8)
    _check(lib().ref_materialize(_sz(len(dims)), _ptr(dims), _ptr(b), _ptr(s), _ptr(hl),
                                 _ptr(ob), _ptr(os_)))
    return ob, os_


def fcs_dense(t: np.ndarray, hash_len: int, master: int) -> np.ndarray:
    """fcs_sketch(DenseTensor, HashFamily(dims, J, master)) (sketch.cpp:187-201).

    ``t`` is given in the reference layout: a numpy array whose FORTRAN order is
    the column-major flat order (first index fastest)."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    out = np.empty(len(dims) * hash_len - len(dims) + 1, np.float64)
    _check(lib().ref_fcs_dense(_ptr(data), _sz(len(dims)), _ptr(dims), _sz(hash_len),
                               _u64(master), _ptr(out)))
    return out


def fcs_dense_tables(t: np.ndarray, buckets, signs, hash_lens) -> np.ndarray:
    """fcs_sketch(DenseTensor, HashFamily(explicit pairs)) (sketch.cpp:187-201)."""
    dims = _dims(t.shape)
    fdims = _dims([len(x) for x in buckets])
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = np.empty(max(int(hl.sum()) - len(hl) + 1, 1), np.float64)
    _check(lib().ref_fcs_dense_tables(_ptr(data), _sz(len(dims)), _ptr(dims), _sz(len(fdims)),
                                      _ptr(fdims), _ptr(b), _ptr(s), _ptr(hl), _ptr(out)))
    return out


def cs_sketch(x, bucket, sign, hash_len: int) -> np.ndarray:
    """cs_sketch (sketch.cpp:105-116)."""
    x = np.ascontiguousarray(np.asarray(x, np.float64))
    b = np.ascontiguousarray(np.asarray(bucket, np.uint32))
    s = np.ascontiguousarray(np.asarray(sign, np.int8))
    out = np.empty(hash_len, np.float64)
    _check(lib().ref_cs_sketch(_ptr(x), _sz(len(x)), _ptr(b), _ptr(s), _sz(len(b)),
                               _sz(hash_len), _ptr(out)))
    return out


def cs_sketch_columns(u, bucket, sign, hash_len: int) -> np.ndarray:
    """cs_sketch_columns (sketch.cpp:118-133); u is I x R, returns J x R."""
    u = np.asarray(u, np.float64)
    data = np.ascontiguousarray(u.ravel(order="F"))
    b = np.ascontiguousarray(np.asarray(bucket, np.uint32))
    s = np.ascontiguousarray(np.asarray(sign, np.int8))
    out = np.empty(hash_len * u.shape[1], np.float64)
    _check(lib().ref_cs_sketch_columns(_ptr(data), _sz(u.shape[0]), _sz(u.shape[1]), _ptr(b),
                                       _ptr(s), _sz(len(b)), _sz(hash_len), _ptr(out)))
    return out.reshape((hash_len, u.shape[1]), order="F")


def _pack_cp(weights, factors):
    w = np.ascontiguousarray(np.asarray(weights, np.float64))
    dims = _dims([f.shape[0] for f in factors])
    fs = np.ascontiguousarray(np.concatenate(
        [np.asarray(f, np.float64).ravel(order="F") for f in factors]))
    return w, dims, fs


def fcs_cp(weights, factors, hash_len: int, master: int) -> np.ndarray:
    """fcs_sketch(CpTensor, HashFamily(dims, J, master)) (sketch.cpp:203-207)."""
    w, dims, fs = _pack_cp(weights, factors)
    out = np.empty(len(dims) * hash_len - len(dims) + 1, np.float64)
    _check(lib().ref_fcs_cp(_ptr(w), _sz(len(w)), _sz(len(dims)), _ptr(dims), _ptr(fs),
                            _sz(hash_len), _u64(master), _ptr(out)))
    return out


def fcs_cp_tables(weights, factors, buckets, signs, hash_lens) -> np.ndarray:
    """fcs_sketch(CpTensor, HashFamily(explicit pairs)) (sketch.cpp:203-207)."""
    w, dims, fs = _pack_cp(weights, factors)
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = np.empty(int(hl.sum()) - len(hl) + 1, np.float64)
    _check(lib().ref_fcs_cp_tables(_ptr(w), _sz(len(w)), _sz(len(dims)), _ptr(dims), _ptr(fs),
                                   _ptr(b), _ptr(s), _ptr(hl), _ptr(out)))
    return out


def densify(weights, factors) -> np.ndarray:
    """densify (tensor.cpp:86-115); returns an array with Fortran-order layout."""
    w, dims, fs = _pack_cp(weights, factors)
    out = np.empty(int(np.prod(dims)), np.float64)
    _check(lib().ref_densify(_ptr(w), _sz(len(w)), _sz(len(dims)), _ptr(dims), _ptr(fs),
                             _ptr(out)))
    return out.reshape(tuple(int(x) for x in dims), order="F")


def kron(a, b) -> np.ndarray:
    """kron (tensor.cpp:228-236)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    da = np.ascontiguousarray(a.ravel(order="F"))
    db = np.ascontiguousarray(b.ravel(order="F"))
    out = np.empty(a.size * b.size, np.float64)
    _check(lib().ref_kron(_ptr(da), _sz(a.shape[0]), _sz(a.shape[1]), _ptr(db), _sz(b.shape[0]),
                          _sz(b.shape[1]), _ptr(out)))
    return out.reshape((a.shape[0] * b.shape[0], a.shape[1] * b.shape[1]), order="F")


def dft(x, n: int) -> np.ndarray:
    """dft (fft.cpp:42-51)."""
    x = np.ascontiguousarray(np.asarray(x, np.float64))
    out = np.empty(2 * max(n, 1), np.float64)
    _check(lib().ref_dft(_ptr(x), _sz(len(x)), _sz(n), _ptr(out)))
    return out[0::2] + 1j * out[1::2]


def idft_real(spec) -> np.ndarray:
    """idft_real (fft.cpp:53-73)."""
    spec = np.asarray(spec, np.complex128)
    inter = np.ascontiguousarray(np.stack([spec.real, spec.imag], axis=1).ravel())
    out = np.empty(max(len(spec), 1), np.float64)
    _check(lib().ref_idft_real(_ptr(inter), _sz(len(spec)), _ptr(out)))
    return out[:len(spec)]


def fft_convolve(inputs, n: int) -> np.ndarray:
    """fft_convolve (fft.cpp:75-84)."""
    arrs = [np.ascontiguousarray(np.asarray(x, np.float64)) for x in inputs]
    ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
    lens = _dims([len(a) for a in arrs]) if arrs else _dims([0])
    out = np.empty(max(n, 1), np.float64)
    _check(lib().ref_fft_convolve(ptrs, _ptr(lens), _sz(len(arrs)), _sz(n), _ptr(out)))
    return out[:n]


def median(values) -> float:
    """median_reduce scalar (estimators.cpp:117-123)."""
    v = np.ascontiguousarray(np.asarray(values, np.float64))
    out = _d(0)
    _check(lib().ref_median(_ptr(v), _sz(len(v)), C.byref(out)))
    return out.value


def median_vec(values) -> np.ndarray:
    """median_reduce vector (estimators.cpp:125-138); values is D x len."""
    v = np.ascontiguousarray(np.asarray(values, np.float64))
    if v.ndim != 2:
        raise ValueError("median_vec: need a D x len array")
    out = np.empty(v.shape[1], np.float64)
    _check(lib().ref_median_vec(_ptr(v), _sz(v.shape[0]), _sz(v.shape[1]), _ptr(out)))
    return out


BACKEND_PLAIN = 0
BACKEND_FCS = 4


class Engine:
    """make_contraction_engine (cpd.cpp:220-232) -> ContractionEngine (cpd.hpp:21-41)."""

    def __init__(self, t: np.ndarray, hash_len: int, sketch_count: int, seed: int,
                 backend: int = BACKEND_FCS):
        dims = _dims(t.shape)
        data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
        self.shape = tuple(int(x) for x in dims)
        self._h = lib().ref_engine_create(_ptr(data), _ptr(dims), _sz(hash_len),
                                          _sz(sketch_count), _u64(seed), C.c_int(backend))
        if not self._h:
            raise ValueError(lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_engine_destroy(C.c_void_p(self._h))
            self._h = None

    def iuv(self, a, b, free_mode: int) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(a, np.float64))
        b = np.ascontiguousarray(np.asarray(b, np.float64))
        out = np.empty(self.shape[free_mode] if free_mode < 3 else 1, np.float64)
        _check(lib().ref_engine_iuv(C.c_void_p(self._h), _ptr(a), _sz(len(a)), _ptr(b),
                                    _sz(len(b)), _sz(free_mode), _ptr(out)))
        return out

    def iuu(self, u) -> np.ndarray:
        return self.iuv(u, u, 0)

    def uvw(self, u, v, w) -> float:
        u, v, w = (np.ascontiguousarray(np.asarray(x, np.float64)) for x in (u, v, w))
        out = _d(0)
        _check(lib().ref_engine_uvw(C.c_void_p(self._h), _ptr(u), _sz(len(u)), _ptr(v),
                                    _sz(len(v)), _ptr(w), _sz(len(w)), C.byref(out)))
        return out.value

    def uuu(self, u) -> float:
        return self.uvw(u, u, u)

    def deflate(self, weight: float, u, v, w):
        u, v, w = (np.ascontiguousarray(np.asarray(x, np.float64)) for x in (u, v, w))
        _check(lib().ref_engine_deflate(C.c_void_p(self._h), _d(weight), _ptr(u), _sz(len(u)),
                                        _ptr(v), _sz(len(v)), _ptr(w), _sz(len(w))))


def rtpm(t: np.ndarray, rank: int, num_inits: int, num_iters: int, hash_len: int,
         sketch_count: int, seed: int, backend: int = BACKEND_FCS):
    """rtpm (cpd.cpp:234-277) on a cubical order-3 tensor; returns (weights, factor)."""
    dim = t.shape[0]
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    w = np.empty(rank, np.float64)
    f = np.empty(dim * rank, np.float64)
    _check(lib().ref_rtpm(_ptr(data), _sz(dim), _sz(rank), _sz(num_inits), _sz(num_iters),
                          C.c_int(backend), _sz(hash_len), _sz(sketch_count), _u64(seed),
                          _ptr(w), _ptr(f)))
    return w, f.reshape((dim, rank), order="F")


def residual_norm_sym(t: np.ndarray, weights, factor) -> float:
    """residual_norm (cpd.cpp:385-392) for a symmetric CP (shared factor)."""
    dim = t.shape[0]
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    w = np.ascontiguousarray(np.asarray(weights, np.float64))
    f = np.ascontiguousarray(np.asarray(factor, np.float64).ravel(order="F"))
    out = _d(0)
    _check(lib().ref_residual_norm_sym(_ptr(data), _sz(dim), _ptr(w), _sz(len(w)), _ptr(f),
                                       C.byref(out)))
    return out.value


def ts_dense_tables(t: np.ndarray, buckets, signs, hash_lens) -> np.ndarray:
    """ts_sketch(DenseTensor, HashFamily) (sketch.cpp:135-149)."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = np.empty(int(hl[0]), np.float64)
    _check(lib().ref_ts_dense_tables(_ptr(data), _sz(len(dims)), _ptr(dims), _ptr(b), _ptr(s),
                                     _ptr(hl), _ptr(out)))
    return out


def ts_cp_tables(weights, factors, buckets, signs, hash_lens) -> np.ndarray:
    """ts_sketch(CpTensor, HashFamily) (sketch.cpp:151-155)."""
    w, dims, fs = _pack_cp(weights, factors)
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = np.empty(int(hl[0]), np.float64)
    _check(lib().ref_ts_cp_tables(_ptr(w), _sz(len(w)), _sz(len(dims)), _ptr(dims), _ptr(fs),
                                  _ptr(b), _ptr(s), _ptr(hl), _ptr(out)))
    return out


def hcs_dense_tables(t: np.ndarray, buckets, signs, hash_lens) -> np.ndarray:
    """hcs_sketch(DenseTensor, HashFamily) (sketch.cpp:157-173); J_0 x ... array."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = np.empty(int(np.prod(hl)), np.float64)
    _check(lib().ref_hcs_dense_tables(_ptr(data), _sz(len(dims)), _ptr(dims), _ptr(b), _ptr(s),
                                      _ptr(hl), _ptr(out)))
    return out.reshape(tuple(int(x) for x in hl), order="F")


def hcs_cp_tables(weights, factors, buckets, signs, hash_lens) -> np.ndarray:
    """hcs_sketch(CpTensor, HashFamily) (sketch.cpp:175-185)."""
    w, dims, fs = _pack_cp(weights, factors)
    b, s = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = np.empty(int(np.prod(hl)), np.float64)
    _check(lib().ref_hcs_cp_tables(_ptr(w), _sz(len(w)), _sz(len(dims)), _ptr(dims), _ptr(fs),
                                   _ptr(b), _ptr(s), _ptr(hl), _ptr(out)))
    return out.reshape(tuple(int(x) for x in hl), order="F")


BACKEND_TS = 2


def _pack_factors(factors):
    return np.ascontiguousarray(np.concatenate(
        [np.asarray(f, np.float64).ravel(order="F") for f in factors]))


def _unpack_factors(f, dims, rank):
    out, off = [], 0
    for n in dims:
        out.append(f[off:off + n * rank].reshape((n, rank), order="F"))
        off += n * rank
    return out


def rtpm_asym(t: np.ndarray, rank: int, num_inits: int, num_iters: int, hash_len: int,
              sketch_count: int, seed: int, backend: int = BACKEND_FCS):
    """rtpm_asym (cpd.cpp:279-335); returns (weights, [F0, F1, F2])."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    w = np.empty(rank, np.float64)
    f = np.empty(int(dims.sum()) * rank, np.float64)
    _check(lib().ref_rtpm_asym(_ptr(data), _ptr(dims), _sz(rank), _sz(num_inits), _sz(num_iters),
                               C.c_int(backend), _sz(hash_len), _sz(sketch_count), _u64(seed),
                               _ptr(w), _ptr(f)))
    return w, _unpack_factors(f, [int(x) for x in dims], rank)


def als(t: np.ndarray, rank: int, max_iters: int, tol: float, hash_len: int, sketch_count: int,
        seed: int, backend: int = BACKEND_FCS):
    """als (cpd.cpp:337-383); returns (weights, [F0, F1, F2])."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    w = np.empty(rank, np.float64)
    f = np.empty(int(dims.sum()) * rank, np.float64)
    _check(lib().ref_als(_ptr(data), _ptr(dims), _sz(rank), _sz(max_iters), _d(tol),
                         C.c_int(backend), _sz(hash_len), _sz(sketch_count), _u64(seed),
                         _ptr(w), _ptr(f)))
    return w, _unpack_factors(f, [int(x) for x in dims], rank)


def residual_norm(t: np.ndarray, weights, factors) -> float:
    """residual_norm (cpd.cpp:385-392) for an order-3 CP."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    w = np.ascontiguousarray(np.asarray(weights, np.float64))
    f = _pack_factors(factors)
    out = _d(0)
    _check(lib().ref_residual_norm(_ptr(data), _ptr(dims), _ptr(w), _sz(len(w)), _ptr(f),
                                   C.byref(out)))
    return out.value


def estimate_inner(a: np.ndarray, b: np.ndarray, hash_len: int, sketch_count: int,
                   seed: int) -> float:
    """estimate_inner (estimators.cpp:198-207)."""
    dims = _dims(a.shape)
    da = np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    db = np.ascontiguousarray(np.asarray(b, np.float64).ravel(order="F"))
    out = _d(0)
    _check(lib().ref_estimate_inner(_ptr(da), _ptr(db), _sz(len(dims)), _ptr(dims),
                                    _sz(hash_len), _sz(sketch_count), _u64(seed), C.byref(out)))
    return out.value


def inner_once_tables(a: np.ndarray, b: np.ndarray, buckets, signs, hash_lens,
                      ts: bool = False) -> float:
    """inner_once / inner_once_ts (estimators.cpp:193-196, 235-239)."""
    dims = _dims(a.shape)
    da = np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    db = np.ascontiguousarray(np.asarray(b, np.float64).ravel(order="F"))
    bk, sg = _pack_tables(buckets, signs)
    hl = _dims(hash_lens)
    out = _d(0)
    _check(lib().ref_inner_once_tables(C.c_int(1 if ts else 0), _ptr(da), _ptr(db),
                                       _sz(len(dims)), _ptr(dims), _ptr(bk), _ptr(sg), _ptr(hl),
                                       C.byref(out)))
    return out.value


def psnr(a: np.ndarray, b: np.ndarray) -> float:
    """psnr (cpd.cpp:394-403)."""
    dims = _dims(a.shape)
    da = np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    db = np.ascontiguousarray(np.asarray(b, np.float64).ravel(order="F"))
    out = _d(0)
    _check(lib().ref_psnr(_ptr(da), _ptr(db), _sz(len(dims)), _ptr(dims), C.byref(out)))
    return out.value


def mode_unfold(t: np.ndarray, mode: int) -> np.ndarray:
    """mode_unfold (tensor.cpp:117-136)."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    n = int(dims[mode])
    out = np.empty(t.size, np.float64)
    _check(lib().ref_mode_unfold(_ptr(data), _sz(len(dims)), _ptr(dims), _sz(mode), _ptr(out)))
    return out.reshape((n, t.size // n), order="F")


def contract_pair(a: np.ndarray, b: np.ndarray, ma: int, mb: int) -> np.ndarray:
    """contract_pair (tensor.cpp:238-261); returns the result as an N-d array."""
    da, db = _dims(a.shape), _dims(b.shape)
    xa = np.ascontiguousarray(np.asarray(a, np.float64).ravel(order="F"))
    xb = np.ascontiguousarray(np.asarray(b, np.float64).ravel(order="F"))
    shape = [int(x) for n, x in enumerate(da) if n != ma] + [int(x) for n, x in enumerate(db)
                                                               if n != mb]
    out = np.empty(int(np.prod(shape)), np.float64)
    _check(lib().ref_contract_pair(_ptr(xa), _sz(len(da)), _ptr(da), _ptr(xb), _sz(len(db)),
                                   _ptr(db), _sz(ma), _sz(mb), _ptr(out)))
    return out.reshape(shape, order="F")


class ResidentTensor:
    """A reference DenseTensor held in C++ (built once, outside any timed
    region): ``fcs(buckets, signs, hash_lens)`` is exactly
    fcs_sketch(const DenseTensor&, HashFamily(explicit pairs)), sketch.cpp:187-201.
    ``gaussian`` fills it with SplitMix64(seed).next_gaussian() draws
    (rng.cpp:8-21), rounded through float32 when ``round_f32``."""

    def __init__(self, handle, dims):
        if not handle:
            raise RuntimeError(lib().ref_last_error().decode())
        self._h = handle
        self.dims = tuple(int(x) for x in dims)

    @classmethod
    def gaussian(cls, seed: int, dims, round_f32: bool = False):
        L = lib()
        L.ref_dense_gaussian.restype = _p
        L.ref_dense_gaussian.argtypes = [_u64, _sz, _p, C.c_int]
        dd = _dims(dims)
        return cls(L.ref_dense_gaussian(_u64(seed), _sz(len(dd)), _ptr(dd), int(round_f32)), dims)

    @classmethod
    def from_array(cls, t: np.ndarray):
        L = lib()
        L.ref_dense_create.restype = _p
        L.ref_dense_create.argtypes = [_p, _sz, _p]
        dd = _dims(t.shape)
        data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
        return cls(L.ref_dense_create(_ptr(data), _sz(len(dd)), _ptr(dd)), t.shape)

    def fcs(self, buckets, signs, hash_lens, out: np.ndarray = None) -> np.ndarray:
        L = lib()
        fdims = _dims([len(x) for x in buckets])
        b, s = _pack_tables(buckets, signs)
        hl = _dims(hash_lens)
        if out is None:
            out = np.empty(max(int(hl.sum()) - len(hl) + 1, 1), np.float64)
        _check(L.ref_fcs_dense_handle(_p(self._h), _sz(len(fdims)), _ptr(fdims), _ptr(b),
                                      _ptr(s), _ptr(hl), _ptr(out)))
        return out

    def close(self):
        if self._h:
            lib().ref_dense_destroy(_p(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def precompute_z(t: np.ndarray, hash_len: int, master: int, a, b, free_mode: int):
    """precompute_fcs + precompute_z (estimators.cpp:147-167) on a cubical
    tensor, family HashFamily({I,I,I}, J, master): (exact spectrum, z)."""
    dim = t.shape[0]
    n = 3 * hash_len - 2
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    av = np.ascontiguousarray(np.asarray(a, np.float64))
    bv = np.ascontiguousarray(np.asarray(b, np.float64))
    spec = np.empty(2 * n, np.float64)
    z = np.empty(n, np.float64)
    L = lib()
    L.ref_precompute_z.argtypes = [_p, _sz, _sz, _u64, _p, _p, _sz, _p, _p]
    _check(L.ref_precompute_z(_ptr(data), _sz(dim), _sz(hash_len), _u64(master), _ptr(av),
                              _ptr(bv), _sz(free_mode), _ptr(spec), _ptr(z)))
    return spec[0::2] + 1j * spec[1::2], z


def estimate_mixed(t: np.ndarray, lens, count: int, seed: int, u, v, w, free_mode: int):
    """estimate_uvw / estimate_iuv over precompute_fcs of families with
    unequal hash lengths (estimators.cpp:169-186): (uvw, iuv)."""
    dims = _dims(t.shape)
    data = np.ascontiguousarray(np.asarray(t, np.float64).ravel(order="F"))
    ln = _dims(lens)
    u, v, w = (np.ascontiguousarray(np.asarray(x, np.float64)) for x in (u, v, w))
    out = np.empty(int(dims[free_mode]), np.float64)
    uvw = _d(0)
    L = lib()
    L.ref_estimate_mixed.argtypes = [_p, _p, _p, _sz, _u64, _p, _p, _p, _sz, _p, _p]
    _check(L.ref_estimate_mixed(_ptr(data), _ptr(dims), _ptr(ln), _sz(count), _u64(seed),
                                _ptr(u), _ptr(v), _ptr(w), _sz(free_mode), C.byref(uvw),
                                _ptr(out)))
    return uvw.value, out
