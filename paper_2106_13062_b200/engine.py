"""ContractionEngine plug-in and the sketched RTPM driver over the B200 C-ABI.

Mirrors ``cpd.hpp:12-84``: ``SketchBackend``, ``ContractionEngine``
(uvw / iuv / deflate / uuu / iuu / shape), ``make_contraction_engine``,
``rtpm``, ``rtpm_asym``, ``als`` and ``residual_norm``, with all five
backends of the reference factory (cpd.cpp:220-232): FCS (the north star) and
TS through the spectral kernels, Plain (exact), HCS and long-pair CS through
the batched contraction kernels of engines_exact.cu. As in the reference,
``RtpmConfig`` / ``AlsConfig`` default to the Plain backend.

The engine keeps the D sketches' spectra resident on the device
(``st_engine_*``); batched entry points (``iuv_batch`` / ``uvw_batch``) are
the GPU-native extension that lets ``rtpm`` run all restarts in lockstep.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import _lib as L
from .sketchtensor import (CpTensor, DenseTensor, EstimatorConfig, _check, _dev, _ptr,
                           _stream)


class SketchBackend(enum.Enum):
    """SketchBackend (cpd.hpp:12), names per cpd.cpp:10-28."""
    Plain = 0
    CS = 1
    TS = 2
    HCS = 3
    FCS = 4


def backend_name(b: SketchBackend) -> str:
    return {SketchBackend.Plain: "plain", SketchBackend.CS: "cs", SketchBackend.TS: "ts",
            SketchBackend.HCS: "hcs", SketchBackend.FCS: "fcs"}[b]


def backend_from_name(name: str) -> SketchBackend:
    for b in SketchBackend:
        if backend_name(b) == name:
            return b
    raise ValueError("unknown backend: " + name)


def _vec(x, n: int, op: str) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(x, np.float64) if not torch.is_tensor(x) else x,
                        dtype=torch.float64)
    if t.shape[-1] != n:
        raise ValueError(f"{op}: vector length mismatch")
    return t.to(_dev()).contiguous()


class ContractionEngine:
    """ContractionEngine (cpd.hpp:21-41)."""

    def uvw(self, u, v, w) -> float:
        raise NotImplementedError

    def iuv(self, a, b, free_mode: int):
        raise NotImplementedError

    def deflate(self, weight: float, u, v, w) -> None:
        raise NotImplementedError

    def uuu(self, u) -> float:
        return self.uvw(u, u, u)

    def iuu(self, u):
        return self.iuv(u, u, 0)

    def shape(self) -> List[int]:
        raise NotImplementedError


class _DeviceEngine(ContractionEngine):
    """A contraction engine on the device (st_engine_create_backend): for the
    sketch backends D = cfg.sketch_count families from families_for
    (estimators.cpp:104-115), sketches built once; Plain keeps the tensor."""

    BACKEND: SketchBackend = SketchBackend.FCS

    def __init__(self, t: DenseTensor, cfg: EstimatorConfig):
        if not isinstance(t, DenseTensor):
            t = DenseTensor.from_array(t)
        if t.order() != 3:
            raise ValueError("make_contraction_engine: order-3 tensor required")
        if self.BACKEND != SketchBackend.Plain and (cfg.hash_len == 0 or cfg.sketch_count == 0):
            raise ValueError("EstimatorConfig: hash_len and sketch_count must be >= 1")
        self._D = 1 if self.BACKEND == SketchBackend.Plain else cfg.sketch_count
        self._shape = t.shape()
        self.cfg = cfg
        h = C.c_void_p()
        _check(L.lib().st_engine_create_backend(
            C.byref(h), self.BACKEND.value, t.st_dtype, _ptr(t.flat), L.size_array(self._shape),
            cfg.hash_len, cfg.sketch_count, C.c_uint64(cfg.seed & ((1 << 64) - 1)), _stream()))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().st_engine_destroy(h)
            except (TypeError, AttributeError):  # interpreter teardown: module globals gone
                pass
            self._h = None

    def shape(self) -> List[int]:
        return list(self._shape)

    _PATHS = {"auto": 0, "spectral": 1, "direct": 2}

    def set_path(self, path: str) -> None:
        """Estimator path of the FCS / TS backends (st_engine_set_path):
        "spectral" (FFT correlation against the cached spectra), "direct"
        (the same correlation in the time domain, correlate.cu) or "auto"
        (the cheaper by the engine's cost rule)."""
        if path not in self._PATHS:
            raise ValueError("set_path: unknown path")
        _check(L.lib().st_engine_set_path(self._h, self._PATHS[path]))

    def composed_len(self) -> int:
        """Sketch length: J~ = 3J - 2 (FCS) or J (TS)."""
        return int(L.lib().st_engine_composed_len(self._h))

    def sketches(self) -> torch.Tensor:
        """Current D x composed_len() sketch values (after any deflations)."""
        out = torch.empty((self._D, self.composed_len()), dtype=torch.float64,
                          device=_dev())
        _check(L.lib().st_engine_sketches(self._h, _ptr(out), _stream()))
        return out

    # ---- batched (GPU-native) forms
    def iuv_batch(self, a, b, free_mode: int, median: bool = True) -> torch.Tensor:
        if free_mode > 2:
            raise ValueError("estimate_iuv: mode out of range")
        c1 = 1 if free_mode == 0 else 0
        c2 = 1 if free_mode == 2 else 2
        A = _vec(a, self._shape[c1], "estimate_iuv")
        B = _vec(b, self._shape[c2], "estimate_iuv")
        A2, B2 = A.reshape(-1, self._shape[c1]), B.reshape(-1, self._shape[c2])
        if A2.shape[0] != B2.shape[0]:
            raise ValueError("estimate_iuv: batch mismatch")
        n = A2.shape[0]
        shape = (n, self._shape[free_mode]) if median else (n, self._D,
                                                            self._shape[free_mode])
        out = torch.empty(shape, dtype=torch.float64, device=_dev())
        _check(L.lib().st_engine_iuv(self._h, n, _ptr(A2), _ptr(B2), free_mode, _ptr(out),
                                     1 if median else 0, _stream()))
        return out

    def uvw_batch(self, u, v, w, median: bool = True) -> torch.Tensor:
        U = _vec(u, self._shape[0], "estimate_uvw").reshape(-1, self._shape[0])
        V = _vec(v, self._shape[1], "estimate_uvw").reshape(-1, self._shape[1])
        W = _vec(w, self._shape[2], "estimate_uvw").reshape(-1, self._shape[2])
        n = U.shape[0]
        out = torch.empty((n,) if median else (n, self._D), dtype=torch.float64,
                          device=_dev())
        _check(L.lib().st_engine_uvw(self._h, n, _ptr(U), _ptr(V), _ptr(W), _ptr(out),
                                     1 if median else 0, _stream()))
        return out

    # ---- reference interface
    def uvw(self, u, v, w) -> float:
        return float(self.uvw_batch(u, v, w)[0].item())

    def iuv(self, a, b, free_mode: int) -> np.ndarray:
        return self.iuv_batch(a, b, free_mode)[0].cpu().numpy()

    def deflate(self, weight: float, u, v, w) -> None:
        U = _vec(u, self._shape[0], "deflate")
        V = _vec(v, self._shape[1], "deflate")
        W = _vec(w, self._shape[2], "deflate")
        _check(L.lib().st_engine_deflate(self._h, C.c_double(weight), _ptr(U), _ptr(V), _ptr(W),
                                         _stream()))


class FcsEngine(_DeviceEngine):
    """FcsEngine (cpd.cpp:61-94): spectra of the D fast count sketches
    (precompute_fcs, estimators.cpp:140-149)."""
    BACKEND = SketchBackend.FCS


class TsEngine(_DeviceEngine):
    """TsEngine (cpd.cpp:96-126): D tensor sketches of length J (ts_sketch,
    sketch.cpp:135-149) and the circular-correlation estimates of
    estimators.cpp:209-233, computed by the FCS kernels on the sketch's
    J-periodic extension."""
    BACKEND = SketchBackend.TS


class PlainEngine(_DeviceEngine):
    """PlainEngine (cpd.cpp:36-59): exact contractions of the device-resident
    tensor (contract3 / contract3_free, tensor.cpp:181-226), exact deflation."""
    BACKEND = SketchBackend.Plain


class HcsEngine(_DeviceEngine):
    """HcsEngine (cpd.cpp:128-158): D higher-order count sketches J x J x J,
    contracted with the count sketches of the vectors (estimators.cpp:241-275)."""
    BACKEND = SketchBackend.HCS


class CsEngine(_DeviceEngine):
    """CsEngine (cpd.cpp:160-197): D long-pair count sketches of vec(T), the
    pair over all prod I_n indices hashed on the device (estimators.cpp:277-350)."""
    BACKEND = SketchBackend.CS


_ENGINES = {SketchBackend.FCS: FcsEngine, SketchBackend.TS: TsEngine,
            SketchBackend.Plain: PlainEngine, SketchBackend.HCS: HcsEngine,
            SketchBackend.CS: CsEngine}


def _engine_backend(backend: SketchBackend) -> int:
    if backend not in _ENGINES:
        raise ValueError("make_contraction_engine: unknown backend")
    return backend.value


def make_contraction_engine(t, backend: SketchBackend, cfg: EstimatorConfig) -> ContractionEngine:
    """make_contraction_engine (cpd.cpp:220-232)."""
    if not isinstance(t, DenseTensor):
        t = DenseTensor.from_array(t)
    if t.order() != 3:
        raise ValueError("make_contraction_engine: order-3 tensor required")
    _engine_backend(backend)
    return _ENGINES[backend](t, cfg)


@dataclass
class RtpmConfig:
    """RtpmConfig (cpd.hpp:49-55)."""
    target_rank: int = 1
    num_inits: int = 15
    num_power_iters: int = 20
    backend: SketchBackend = SketchBackend.Plain
    estimator: EstimatorConfig = field(default_factory=EstimatorConfig)


@dataclass
class AlsConfig:
    """AlsConfig (cpd.hpp:57-63)."""
    target_rank: int = 1
    max_iters: int = 50
    backend: SketchBackend = SketchBackend.Plain
    estimator: EstimatorConfig = field(default_factory=EstimatorConfig)
    tol: float = 1e-8


def _order3(t, op: str) -> DenseTensor:
    if not isinstance(t, DenseTensor):
        t = DenseTensor.from_array(t)
    if t.order() != 3:
        raise ValueError(f"{op}: order-3 tensor required")
    return t


def _seed(e: EstimatorConfig):
    return C.c_uint64(e.seed & ((1 << 64) - 1))


def _unpack_factors(f: np.ndarray, dims, R: int):
    out, off = [], 0
    for n in dims:
        out.append(f[off:off + n * R].reshape((R, n)).T.copy())
        off += n * R
    return out


def rtpm(t, cfg: RtpmConfig) -> CpTensor:
    """rtpm (cpd.cpp:234-277): restarts batched on the device (st_rtpm_backend);
    same initial-vector stream, argmax rule and deflation."""
    t = _order3(t, "rtpm")
    dims = t.shape()
    if dims[0] != dims[1] or dims[1] != dims[2]:
        raise ValueError("rtpm: cubical tensor required")
    if cfg.target_rank == 0 or cfg.num_inits == 0 or cfg.num_power_iters == 0:
        raise ValueError("rtpm: rank, inits, and iterations must be >= 1")
    backend = _engine_backend(cfg.backend)
    dim, R = dims[0], cfg.target_rank
    w = np.empty(R, np.float64)
    f = np.empty(dim * R, np.float64)
    e = cfg.estimator
    _check(L.lib().st_rtpm_backend(backend, t.st_dtype, _ptr(t.flat), dim, R, cfg.num_inits,
                                   cfg.num_power_iters, e.hash_len, e.sketch_count, _seed(e),
                                   w.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p),
                                   _stream()))
    factor = f.reshape((R, dim)).T
    return CpTensor(w, [factor, factor, factor])


def rtpm_asym(t, cfg: RtpmConfig) -> CpTensor:
    """rtpm_asym (cpd.cpp:279-335) for a general order-3 tensor (st_rtpm_asym)."""
    t = _order3(t, "rtpm_asym")
    if cfg.target_rank == 0 or cfg.num_inits == 0 or cfg.num_power_iters == 0:
        raise ValueError("rtpm_asym: rank, inits, and iterations must be >= 1")
    backend = _engine_backend(cfg.backend)
    dims, R = t.shape(), cfg.target_rank
    w = np.empty(R, np.float64)
    f = np.empty(sum(dims) * R, np.float64)
    e = cfg.estimator
    _check(L.lib().st_rtpm_asym(backend, t.st_dtype, _ptr(t.flat), L.size_array(dims), R,
                                cfg.num_inits, cfg.num_power_iters, e.hash_len, e.sketch_count,
                                _seed(e), w.ctypes.data_as(C.c_void_p),
                                f.ctypes.data_as(C.c_void_p), _stream()))
    return CpTensor(w, _unpack_factors(f, dims, R))


def als(t, cfg: AlsConfig, return_sweeps: bool = False):
    """als (cpd.cpp:337-383): engine MTTKRP columns (one batched iuv per mode),
    exact Gram solves, device residual each sweep (st_als)."""
    t = _order3(t, "als")
    if cfg.target_rank == 0 or cfg.max_iters == 0:
        raise ValueError("als: rank and iterations must be >= 1")
    backend = _engine_backend(cfg.backend)
    dims, R = t.shape(), cfg.target_rank
    w = np.empty(R, np.float64)
    f = np.empty(sum(dims) * R, np.float64)
    sweeps = C.c_size_t(0)
    e = cfg.estimator
    _check(L.lib().st_als(backend, t.st_dtype, _ptr(t.flat), L.size_array(dims), R,
                          cfg.max_iters, C.c_double(cfg.tol), e.hash_len, e.sketch_count,
                          _seed(e), w.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p),
                          C.byref(sweeps), _stream()))
    cp = CpTensor(w, _unpack_factors(f, dims, R))
    return (cp, int(sweeps.value)) if return_sweeps else cp


def residual_norm(t, cp: CpTensor) -> float:
    """residual_norm (cpd.cpp:385-392): ||t - densify(cp)||_F / ||t||_F on the
    device (st_residual_norm), order-3."""
    t = _order3(t, "residual_norm")
    dims = t.shape()
    if cp.order() != 3 or cp.shape() != list(dims):
        raise ValueError("residual_norm: CP shape does not match the tensor")
    R = cp.rank()
    packed = torch.cat([f.reshape(-1) for f in cp._factors_cm])
    w = cp.weights.contiguous()
    out = C.c_double(0.0)
    _check(L.lib().st_residual_norm(t.st_dtype, _ptr(t.flat), L.size_array(dims), _ptr(w), R,
                                    _ptr(packed), C.byref(out), _stream()))
    return out.value


def psnr(reference, estimate) -> float:
    """psnr (cpd.cpp:394-403): 10 log10(peak^2 / MSE), peak = max|reference|,
    capped at 99 dB, on the device (st_psnr)."""
    if not isinstance(reference, DenseTensor):
        reference = DenseTensor.from_array(reference)
    if not isinstance(estimate, DenseTensor):
        estimate = DenseTensor.from_array(estimate)
    if reference.shape() != estimate.shape():
        raise ValueError("psnr: shape mismatch")
    est = estimate.flat.to(reference.flat.dtype).contiguous()
    out = C.c_double(0.0)
    _check(L.lib().st_psnr(reference.st_dtype, _ptr(reference.flat), _ptr(est),
                           reference.size(), C.byref(out), _stream()))
    return out.value


def densify(cp: CpTensor) -> DenseTensor:
    """densify (tensor.cpp:86-115) on the device (st_densify)."""
    dims = cp.shape()
    out = torch.empty(int(np.prod(dims)), dtype=torch.float64, device=_dev())
    fptrs = (C.c_void_p * len(dims))(*[f.data_ptr() for f in cp._factors_cm])
    _check(L.lib().st_densify(len(dims), L.size_array(dims), cp.rank(), _ptr(cp.weights), fptrs,
                              _ptr(out), _stream()))
    return DenseTensor(dims, out)


def rank_one(weight: float, vectors) -> CpTensor:
    """rank_one (tensor.hpp): weight * v_1 o ... o v_N as a CpTensor."""
    return CpTensor([weight], [np.asarray(v, np.float64).reshape(-1, 1) if not torch.is_tensor(v)
                               else v.reshape(-1, 1) for v in vectors])


def contract3(t, u, v, w) -> float:
    """contract3 (tensor.cpp:181-197): T(u, v, w), exact, on the device."""
    return PlainEngine(_order3(t, "contract3"), EstimatorConfig(0, 0, 0)).uvw(u, v, w)


def contract3_free(t, a, b, free_mode: int) -> np.ndarray:
    """contract3_free (tensor.cpp:199-226): exact T with the identity at free_mode."""
    return PlainEngine(_order3(t, "contract3_free"), EstimatorConfig(0, 0, 0)).iuv(a, b, free_mode)


def inner(a, b) -> float:
    """inner (tensor.hpp): vec(a)^T vec(b) on the device (fixed-order dot)."""
    if not isinstance(a, DenseTensor):
        a = DenseTensor.from_array(a)
    if not isinstance(b, DenseTensor):
        b = DenseTensor.from_array(b)
    if a.shape() != b.shape():
        raise ValueError("inner: shape mismatch")
    x = a.flat.to(torch.float64).reshape(1, -1).contiguous()
    y = b.flat.to(torch.float64).reshape(1, -1).contiguous()
    out = torch.empty(1, dtype=torch.float64, device=_dev())
    _check(L.lib().st_sketch_dots(1, x.shape[1], _ptr(x), _ptr(y), _ptr(out), _stream()))
    return float(out.item())


# ------------------------------------------------ tensor utilities (tensor.hpp)
def _dense_from(t) -> DenseTensor:
    return t if isinstance(t, DenseTensor) else DenseTensor.from_array(t)


def mode_unfold(t, mode: int) -> torch.Tensor:
    """mode_unfold (tensor.cpp:117-136): the I_mode x prod_{m != mode} I_m
    matricization, columns in the flat order with mode `mode` removed; a device
    tensor (row/column indices as in the reference's Eigen matrix)."""
    t = _dense_from(t)
    dims = t.shape()
    if mode >= len(dims):
        raise ValueError("mode_unfold: mode out of range")
    inner = int(np.prod(dims[:mode], dtype=np.int64))
    n = dims[mode]
    outer = t.size() // (inner * n)
    # flat = (o * n + i) * inner + k  ->  M[i, o * inner + k]
    return t.flat.to(torch.float64).reshape(outer, n, inner).permute(1, 0, 2).reshape(n, -1)


def mode_fold(m, shape, mode: int) -> DenseTensor:
    """mode_fold (tensor.cpp:138-160): inverse of mode_unfold for `shape`."""
    shape = [int(s) for s in shape]
    if mode >= len(shape):
        raise ValueError("mode_fold: mode out of range")
    m = torch.as_tensor(m if torch.is_tensor(m) else np.asarray(m, np.float64),
                        dtype=torch.float64).to(_dev())
    inner = int(np.prod(shape[:mode], dtype=np.int64))
    n = shape[mode]
    total = int(np.prod(shape, dtype=np.int64))
    if tuple(m.shape) != (n, total // n):
        raise ValueError("mode_fold: matrix does not match shape")
    outer = total // (inner * n)
    flat = m.reshape(n, outer, inner).permute(1, 0, 2).reshape(-1).contiguous()
    return DenseTensor(shape, flat)


def contract_pair(a, b, mode_a: int, mode_b: int) -> DenseTensor:
    """contract_pair (tensor.cpp:238-261): contraction of a's mode_a with b's
    mode_b, result modes a-rest then b-rest (one device GEMM)."""
    a, b = _dense_from(a), _dense_from(b)
    if mode_a >= a.order() or mode_b >= b.order():
        raise ValueError("contract_pair: mode out of range")
    if a.shape()[mode_a] != b.shape()[mode_b]:
        raise ValueError("contract_pair: contracted dimensions differ")
    if a.order() + b.order() < 3:
        raise ValueError("contract_pair: result would have no modes")
    prod = mode_unfold(a, mode_a).t() @ mode_unfold(b, mode_b)  # a-rest x b-rest
    shape = [d for n, d in enumerate(a.shape()) if n != mode_a] + \
        [d for n, d in enumerate(b.shape()) if n != mode_b]
    return DenseTensor(shape, prod.t().contiguous().reshape(-1))  # column-major flat


def kron(a, b) -> torch.Tensor:
    """kron (tensor.cpp:228-236): Kronecker product of two matrices (device)."""
    ta = torch.as_tensor(a if torch.is_tensor(a) else np.asarray(a, np.float64),
                         dtype=torch.float64).to(_dev())
    tb = torch.as_tensor(b if torch.is_tensor(b) else np.asarray(b, np.float64),
                         dtype=torch.float64).to(_dev())
    return torch.kron(ta, tb)


def tensor_from_matrix(m) -> DenseTensor:
    """tensor_from_matrix (tensor.hpp): order-2 tensor, column-major copy."""
    tm = torch.as_tensor(m if torch.is_tensor(m) else np.asarray(m, np.float64),
                         dtype=torch.float64)
    return DenseTensor(list(tm.shape), tm.t().contiguous().reshape(-1))
