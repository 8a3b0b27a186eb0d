"""Inner-product estimates, the sketched regression forward map and the
Kronecker / contraction compression codecs.

The reference implements ``inner_once`` / ``estimate_inner`` /
``inner_once_ts`` (estimators.cpp:193-239); the regression map and the codecs
exist only as its spec (§4.2-4.3), which is the
contract here. Every compute step runs through the C-ABI (codecs.cu, K1,
the shared-memory FFT); nothing here falls back to the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np
import torch

from . import _lib as L
from .sketchtensor import (DenseTensor, EstimatorConfig, HashFamily, SketchKind, _check, _dev,
                           _ptr, _require_family, _stream, families_for, fcs_sketch,
                           packed_families, ts_sketch)

ENTRY_BYTES = 5  # one hash-map entry: uint32 bucket + int8 sign (hashing.hpp:41-42)


def _dense(t) -> DenseTensor:
    return t if isinstance(t, DenseTensor) else DenseTensor.from_array(t)


def _matrix(x) -> torch.Tensor:
    return torch.as_tensor(np.asarray(x, np.float64) if not torch.is_tensor(x) else x,
                           dtype=torch.float64)


def _seed(cfg: EstimatorConfig):
    return C.c_uint64(cfg.seed & ((1 << 64) - 1))


# ------------------------------------------------------------ inner products
def _same_shape(a: DenseTensor, b: DenseTensor, op: str):
    if a.shape() != b.shape():
        raise ValueError(f"{op}: shape mismatch")
    if a.flat.dtype != b.flat.dtype:
        raise ValueError(f"{op}: dtype mismatch")


def inner_once(a, b, family: HashFamily) -> float:
    """inner_once (estimators.cpp:193-196): <FCS(a), FCS(b)> for one family."""
    a, b = _dense(a), _dense(b)
    _same_shape(a, b, "inner_once")
    sa, sb = fcs_sketch(a, family).values, fcs_sketch(b, family).values
    return _dot(sa, sb)


def inner_once_ts(a, b, family: HashFamily) -> float:
    """inner_once_ts (estimators.cpp:235-239): <TS(a), TS(b)> for one family."""
    a, b = _dense(a), _dense(b)
    _same_shape(a, b, "inner_once_ts")
    return _dot(ts_sketch(a, family).values, ts_sketch(b, family).values)


def _dot(x: torch.Tensor, y: torch.Tensor) -> float:
    x, y = x.reshape(1, -1).contiguous(), y.reshape(1, -1).contiguous()
    out = torch.empty(1, dtype=torch.float64, device=_dev())
    _check(L.lib().st_sketch_dots(1, x.shape[1], _ptr(x), _ptr(y), _ptr(out), _stream()))
    return float(out.item())


def estimate_inner(a, b, cfg: EstimatorConfig, kind: SketchKind = SketchKind.FCS,
                   return_estimates: bool = False):
    """estimate_inner (estimators.cpp:198-207): median over cfg.sketch_count
    families of inner_once (kind FCS) or inner_once_ts (kind TS), all families
    in one K1 launch per tensor (st_estimate_inner)."""
    a, b = _dense(a), _dense(b)
    _same_shape(a, b, "estimate_inner")
    if cfg.hash_len == 0 or cfg.sketch_count == 0:
        raise ValueError("EstimatorConfig: hash_len and sketch_count must be >= 1")
    k = {SketchKind.FCS: L.ST_SKETCH_FCS, SketchKind.TS: L.ST_SKETCH_TS}.get(kind)
    if k is None:
        raise ValueError("estimate_inner: FCS or TS sketches only")
    est = torch.empty(cfg.sketch_count, dtype=torch.float64, device=_dev())
    out = C.c_double(0.0)
    _check(L.lib().st_estimate_inner(k, a.st_dtype, _ptr(a.flat), _ptr(b.flat), a.order(),
                                     L.size_array(a.shape()), cfg.hash_len, cfg.sketch_count,
                                     _seed(cfg), _ptr(est), C.byref(out), _stream()))
    return (out.value, est) if return_estimates else out.value


# ------------------------------------------------------------ regression map
def sketched_regression_forward(x_rows, w_rows, bias, dims: Sequence[int],
                                cfg: EstimatorConfig) -> torch.Tensor:
    """Y = median_d FCS_d(X_(1)^T)^T FCS_d(W_(N+1)^T) + b (SPEC.md:408-411,
    PAPER.md Eq. 20). x_rows: B x prod(dims), w_rows: C x prod(dims), each row
    a column-major order-N tensor; bias: C or None. Returns B x C (device)."""
    dims = [int(d) for d in dims]
    n = int(np.prod(dims))
    X = torch.as_tensor(x_rows if torch.is_tensor(x_rows) else np.asarray(x_rows))
    W = torch.as_tensor(w_rows if torch.is_tensor(w_rows) else np.asarray(w_rows))
    dt = torch.float32 if X.dtype == torch.float32 and W.dtype == torch.float32 else torch.float64
    X, W = X.to(_dev(), dt).reshape(-1, n).contiguous(), W.to(_dev(), dt).reshape(-1, n).contiguous()
    if X.shape[1] != n or W.shape[1] != n:
        raise ValueError("sketched_regression_forward: shape mismatch")
    B, Cn = X.shape[0], W.shape[0]
    b = None
    if bias is not None:
        b = _matrix(bias).reshape(-1).to(_dev()).contiguous()
        if b.numel() != Cn:
            raise ValueError("sketched_regression_forward: bias length mismatch")
    y = torch.empty((B, Cn), dtype=torch.float64, device=_dev())
    _check(L.lib().st_regression_forward(L.ST_F32 if dt == torch.float32 else L.ST_F64, _ptr(X),
                                         B, _ptr(W), Cn, _ptr(b), len(dims), L.size_array(dims),
                                         cfg.hash_len, cfg.sketch_count, _seed(cfg), _ptr(y),
                                         _stream()))
    return y


# ------------------------------------------------------------------- codecs
@dataclass
class KronSketch:
    """KronSketch / ContractionSketch: D copies of length
    sum J_n - 3 (4J - 3) under D families of 4 pairs over (I1, I2, I3, I4)."""
    values: torch.Tensor          # D x (sum J - 3), device
    families: List[HashFamily]
    dims: List[int]               # I1, I2, I3, I4
    packed: torch.Tensor

    def sketch_count(self) -> int:
        return len(self.families)


def _four_pair_families(dims, cfg: EstimatorConfig):
    fams = families_for(list(dims), cfg)
    return fams, packed_families(fams)


def compress_kron(a, b, cfg: EstimatorConfig) -> KronSketch:
    """compress_kron: never materialises A (x) B; per copy the
    CS of vec(A) under pairs 0-1 composed, of vec(B) under pairs 2-3, and their
    zero-padded FFT convolution (st_fcs_contraction with L = 1)."""
    A, Bm = _matrix(a), _matrix(b)
    if A.dim() != 2 or Bm.dim() != 2:
        raise ValueError("compress_kron: matrices required")
    return _contraction(A.reshape(A.shape[0], A.shape[1], 1),
                        Bm.reshape(1, Bm.shape[0], Bm.shape[1]), cfg)


def compress_contraction(a, b, cfg: EstimatorConfig) -> KronSketch:
    """compress_contraction: FCS of A (x)_{3,1} B for A
    (I1, I2, L), B (L, I3, I4) as sum_l of slice-pair convolutions."""
    A, Bm = _matrix(a), _matrix(b)
    if A.dim() != 3 or Bm.dim() != 3:
        raise ValueError("compress_contraction: order-3 tensors required")
    if A.shape[2] != Bm.shape[0]:
        raise ValueError("compress_contraction: L mismatch")
    return _contraction(A, Bm, cfg)


def _contraction(A: torch.Tensor, Bm: torch.Tensor, cfg: EstimatorConfig) -> KronSketch:
    dims = [A.shape[0], A.shape[1], Bm.shape[1], Bm.shape[2]]
    fams, packed = _four_pair_families(dims, cfg)
    ta, tb = DenseTensor.from_array(A), DenseTensor.from_array(Bm)
    lens = fams[0].hash_lens()
    out = torch.empty((len(fams), sum(lens) - 3), dtype=torch.float64, device=_dev())
    _check(L.lib().st_fcs_contraction(L.ST_F64, _ptr(ta.flat), L.size_array(list(A.shape)),
                                      _ptr(tb.flat), L.size_array(list(Bm.shape)), len(fams),
                                      _ptr(packed), L.size_array(lens), _ptr(out), _stream()))
    return KronSketch(out, fams, dims, packed)


def _decompress(sk: KronSketch, idx: np.ndarray) -> torch.Tensor:
    idx = np.ascontiguousarray(np.asarray(idx, np.int64).reshape(-1, 4))
    for n in range(4):
        if (idx[:, n] < 0).any() or (idx[:, n] >= sk.dims[n]).any():
            raise ValueError("decompress: index out of range")
    dev_idx = torch.from_numpy(idx.astype(np.uint32)).to(_dev())
    out = torch.empty(idx.shape[0], dtype=torch.float64, device=_dev())
    _check(L.lib().st_sketch_decompress(_ptr(sk.values), sk.sketch_count(), sk.values.shape[1],
                                        _ptr(sk.packed), 4, L.size_array(sk.dims), idx.shape[0],
                                        _ptr(dev_idx), _ptr(out), _stream()))
    return out


def decompress_kron(sk: KronSketch, row, col):
    """decompress_kron: median over D of the signed bucket
    read for (A (x) B)[row, col], row = I3 i1 + i3, col = I4 i2 + i4 (0-based).
    Scalars give a float; arrays give a device tensor of estimates."""
    I1, I2, I3, I4 = sk.dims
    r, c = np.asarray(row, np.int64), np.asarray(col, np.int64)
    if (r < 0).any() or (r >= I1 * I3).any() or (c < 0).any() or (c >= I2 * I4).any():
        raise ValueError("decompress_kron: index out of range")
    idx = np.stack(np.broadcast_arrays(r // I3, c // I4, r % I3, c % I4), axis=-1)
    out = _decompress(sk, idx)
    return float(out.item()) if np.ndim(row) == 0 and np.ndim(col) == 0 else out


def reconstruct_kron(sk: KronSketch) -> torch.Tensor:
    """Full (I1 I3) x (I2 I4) reconstruction (decompress looped over
    every entry), one thread per entry on the device."""
    I1, I2, I3, I4 = sk.dims
    out = torch.empty(I1 * I3 * I2 * I4, dtype=torch.float64, device=_dev())
    _check(L.lib().st_kron_decompress_all(_ptr(sk.values), sk.sketch_count(),
                                          sk.values.shape[1], _ptr(sk.packed),
                                          L.size_array(sk.dims), _ptr(out), _stream()))
    return out.reshape(I2 * I4, I1 * I3).t()


def decompress_contraction(sk: KronSketch, i1, i2, i3, i4):
    """decompress_contraction: estimate of
    (A (x)_{3,1} B)[i1, i2, i3, i4] (0-based)."""
    idx = np.stack(np.broadcast_arrays(*(np.asarray(x, np.int64) for x in (i1, i2, i3, i4))),
                   axis=-1)
    out = _decompress(sk, idx)
    return float(out.item()) if idx.ndim == 1 else out


def compression_ratio(family: HashFamily) -> float:
    """CR = prod I_n / J~ (§4.2)."""
    dims = [family.pair(n).input_dim() for n in range(family.modes())]
    return float(np.prod(dims, dtype=np.float64)) / family.composed_len()


def hash_memory(family: HashFamily) -> int:
    """Bytes of stored hash-map entries: sum_n I_n entries for FCS."""
    return ENTRY_BYTES * sum(family.pair(n).input_dim() for n in range(family.modes()))


def hash_memory_long_pair(dims: Sequence[int]) -> int:
    """The CS baseline's full-length composed pair: prod I_n entries."""
    return ENTRY_BYTES * int(np.prod([int(d) for d in dims], dtype=np.int64))
