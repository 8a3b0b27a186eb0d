"""Host mirror of the reference's ``sketchtensor`` API over the B200 C-ABI.

Names, argument meaning and error behaviour follow
``/root/reference/proj/include/sketchtensor/*.hpp`` (cited per symbol);
every compute call goes through ``include/fcs_b200.h`` into the sm_100a
kernels — there is no CPU path. Device memory is held in torch CUDA tensors
(plumbing only). ``std::invalid_argument`` surfaces as ``ValueError`` and
``std::runtime_error`` as ``RuntimeError``, as in the reference.

Layout: dense tensors are column-major with the first index fastest
(tensor.hpp:10-13). A numpy/torch array passed as a tensor is read in
Fortran order (``np.asfortranarray`` semantics); ``DenseTensor`` can also be
built from a flat column-major vector plus a shape.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib as L

_MASK64 = (1 << 64) - 1


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("fcs_b200: no CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _check(rc: int) -> None:
    L.check(rc)


# -------------------------------------------------------------------- hashing
def family_seed(base_seed: int, d: int) -> int:
    """family_seed (hashing.hpp:94, hashing.cpp:123-125)."""
    return int(L.lib().st_family_seed(C.c_uint64(base_seed & _MASK64), C.c_size_t(d)))


class HashPair:
    """HashPair (hashing.hpp:17-45). Seeded pairs are tabulated on the GPU
    (K0, bit-exact with hashing.cpp:10-22); explicit maps are validated like
    hashing.cpp:24-40."""

    def __init__(self, input_dim=None, hash_len=None, seed=None, *, bucket_map=None,
                 sign_map=None):
        if bucket_map is not None:
            b = np.asarray(bucket_map, dtype=np.int64)
            s = np.asarray(sign_map, dtype=np.int64)
            hash_len = int(hash_len)
            if b.size == 0 or hash_len == 0:
                raise ValueError("HashPair: dimensions must be positive")
            if b.shape != s.shape:
                raise ValueError("HashPair: bucket and sign maps differ in length")
            if (b < 0).any() or (b >= hash_len).any():
                raise ValueError("HashPair: bucket out of range")
            if not np.isin(s, (-1, 1)).all():
                raise ValueError("HashPair: sign must be +/-1")
            self._bucket = b.astype(np.uint32)
            self._sign = s.astype(np.int8)
            self._hash_len = hash_len
            self._seed = None
            return
        input_dim, hash_len = int(input_dim), int(hash_len)
        if input_dim == 0 or hash_len == 0:
            raise ValueError("HashPair: dimensions must be positive")
        dev = _dev()
        bk = torch.empty(input_dim, dtype=torch.int32, device=dev)
        sg = torch.empty(input_dim, dtype=torch.int8, device=dev)
        _check(L.lib().st_hash_tabulate(C.c_uint64(seed & _MASK64), input_dim, hash_len,
                                        _ptr(bk), _ptr(sg), _stream()))
        self._bucket = bk.cpu().numpy().view(np.uint32)
        self._sign = sg.cpu().numpy()
        self._hash_len = hash_len
        self._seed = int(seed) & _MASK64

    def input_dim(self) -> int:
        return int(self._bucket.size)

    def hash_len(self) -> int:
        return self._hash_len

    def seed(self) -> Optional[int]:
        return self._seed

    def bucket(self, i: int) -> int:
        return int(self._bucket[i])

    def sign(self, i: int) -> int:
        return int(self._sign[i])

    def bucket_map(self) -> np.ndarray:
        return self._bucket

    def sign_map(self) -> np.ndarray:
        return self._sign

    def packed(self) -> torch.Tensor:
        """Device packed table (bucket | sign bit 31), see include/fcs_b200.h."""
        p = self._bucket.astype(np.uint64) | np.where(self._sign < 0, np.uint64(1 << 31),
                                                      np.uint64(0))
        return torch.from_numpy(p.astype(np.uint32).view(np.int32).copy()).to(_dev())


class HashFamily:
    """HashFamily (hashing.hpp:51-89): pair n seeded master ^ n."""

    def __init__(self, input_dims=None, hash_lens=None, master_seed=None, *, pairs=None):
        if pairs is not None:
            if len(pairs) == 0:
                raise ValueError("HashFamily: no pairs")
            self._pairs = list(pairs)
            self._master = None
            return
        dims = [int(x) for x in input_dims]
        if isinstance(hash_lens, (int, np.integer)):
            hash_lens = [int(hash_lens)] * len(dims)
        lens = [int(x) for x in hash_lens]
        if len(dims) == 0 or len(dims) != len(lens):
            raise ValueError("HashFamily: need one hash length per mode")
        self._pairs = [HashPair(d, j, (master_seed ^ n) & _MASK64) for n, (d, j) in
                       enumerate(zip(dims, lens))]
        self._master = int(master_seed) & _MASK64

    def modes(self) -> int:
        return len(self._pairs)

    def pair(self, n: int) -> HashPair:
        return self._pairs[n]

    def pairs(self) -> List[HashPair]:
        return self._pairs

    def master_seed(self) -> Optional[int]:
        return self._master

    def input_dims(self) -> List[int]:
        return [p.input_dim() for p in self._pairs]

    def hash_lens(self) -> List[int]:
        return [p.hash_len() for p in self._pairs]

    def composed_len(self) -> int:
        """sum(J_n) - N + 1 (hashing.cpp:77-81)."""
        return sum(self.hash_lens()) - self.modes() + 1

    def compose(self, multi_index) -> tuple:
        """Composed (bucket, sign) of one multi-index (hashing.cpp:83-98)."""
        if len(multi_index) != self.modes():
            raise ValueError("compose: index order does not match family")
        b, s = 0, 1
        for n, i in enumerate(multi_index):
            if i >= self._pairs[n].input_dim():
                raise ValueError("compose: index out of range")
            b += self._pairs[n].bucket(i)
            s *= self._pairs[n].sign(i)
        return b, s

    def packed(self) -> torch.Tensor:
        return torch.cat([p.packed() for p in self._pairs])


def packed_families(families: Sequence[HashFamily]) -> torch.Tensor:
    """Concatenated packed tables of D families over the same dims (C-ABI layout).
    Seeded families are re-tabulated on the device in one pass (K0)."""
    fams = list(families)
    if all(f.master_seed() is not None for f in fams) and len(
            {tuple(f.input_dims()) for f in fams}) == 1:
        dims = fams[0].input_dims()
        lens = fams[0].hash_lens()
        out = torch.empty(len(fams) * sum(dims), dtype=torch.int32, device=_dev())
        _check(L.lib().st_family_tables(len(dims), L.size_array(dims), L.size_array(lens),
                                        len(fams), L.u64_array([f.master_seed() for f in fams]),
                                        _ptr(out), _stream()))
        return out
    return torch.cat([f.packed() for f in fams])


@dataclass
class EstimatorConfig:
    """EstimatorConfig (estimators.hpp:18-23)."""
    hash_len: int = 16
    sketch_count: int = 1
    seed: int = 0


def families_for(dims, cfg: EstimatorConfig) -> List[HashFamily]:
    """families_for (estimators.cpp:104-115)."""
    if cfg.hash_len == 0 or cfg.sketch_count == 0:
        raise ValueError("EstimatorConfig: hash_len and sketch_count must be >= 1")
    return [HashFamily(dims, cfg.hash_len, family_seed(cfg.seed, d))
            for d in range(cfg.sketch_count)]


# -------------------------------------------------------------------- tensors
class DenseTensor:
    """DenseTensor (tensor.hpp:14-52): column-major, first index fastest.
    Holds a flat device tensor (fp64, or fp32 as an API extension)."""

    def __init__(self, shape, data=None, dtype=torch.float64):
        shape = [int(x) for x in shape]
        if len(shape) == 0:
            raise ValueError("DenseTensor: empty shape")
        if any(x == 0 for x in shape):
            raise ValueError("DenseTensor: zero dimension")
        n = int(np.prod(shape))
        if data is None:
            self.flat = torch.zeros(n, dtype=dtype, device=_dev())
        else:
            flat = torch.as_tensor(np.asarray(data) if not torch.is_tensor(data) else data)
            flat = flat.reshape(-1)
            if flat.numel() != n:
                raise ValueError("DenseTensor: data length does not match shape")
            if flat.dtype not in (torch.float32, torch.float64):
                flat = flat.to(dtype)
            self.flat = flat.to(_dev()).contiguous()
        self._shape = shape

    @classmethod
    def from_array(cls, a, dtype=None) -> "DenseTensor":
        """Wrap an N-d array indexed a[i_0, ..., i_{N-1}] (stored column-major)."""
        if torch.is_tensor(a):
            flat = a.permute(*reversed(range(a.dim()))).reshape(-1)
            t = cls(list(a.shape), flat)
        else:
            a = np.asarray(a)
            t = cls(list(a.shape), np.ascontiguousarray(a.ravel(order="F")))
        if dtype is not None:
            t.flat = t.flat.to(dtype)
        return t

    def order(self) -> int:
        return len(self._shape)

    def shape(self) -> List[int]:
        return list(self._shape)

    def size(self) -> int:
        return self.flat.numel()

    @property
    def st_dtype(self) -> int:
        return L.ST_F32 if self.flat.dtype == torch.float32 else L.ST_F64


class CpTensor:
    """CpTensor (tensor.hpp:55-65): weights and one I_n x R factor per mode."""

    def __init__(self, weights, factors):
        self.weights = torch.as_tensor(np.asarray(weights, np.float64) if not torch.is_tensor(
            weights) else weights, dtype=torch.float64).reshape(-1).to(_dev())
        if len(factors) == 0:
            raise ValueError("CpTensor: no factors")
        fs = []
        for f in factors:
            f = torch.as_tensor(np.asarray(f, np.float64) if not torch.is_tensor(f) else f,
                                dtype=torch.float64)
            if f.dim() == 1:
                f = f.reshape(-1, 1)
            if f.shape[1] != self.weights.numel() or f.shape[0] == 0:
                raise ValueError("CpTensor: factor shape mismatch")
            # column-major I_n x R on the device: store the transpose contiguous
            fs.append(f.t().contiguous().to(_dev()))
        self._factors_cm = fs

    def order(self) -> int:
        return len(self._factors_cm)

    def rank(self) -> int:
        return self.weights.numel()

    def shape(self) -> List[int]:
        return [f.shape[1] for f in self._factors_cm]

    @property
    def factors(self) -> List[torch.Tensor]:
        """The I_n x R factor matrices (views of the column-major device copies)."""
        return [f.t() for f in self._factors_cm]


# ------------------------------------------------------------------- sketches
class SketchKind(enum.Enum):
    CS = 0
    TS = 1
    FCS = 2


class SketchVec:
    """SketchVec (sketch.hpp:15-21; length contract sketch.cpp:90-96)."""

    def __init__(self, values, family: HashFamily, kind: SketchKind):
        self.values = values
        self.family = family
        self.kind = kind
        expected = family.composed_len() if kind == SketchKind.FCS else family.pair(0).hash_len()
        if int(values.numel()) != expected:
            raise ValueError("SketchVec: length contract violated")


def _require_family(shape, family: HashFamily, op: str):
    """require_family_matches (sketch.cpp:12-34)."""
    if len(shape) != family.modes():
        raise ValueError(f"{op}: family order mismatch")
    for n in range(family.modes()):
        if shape[n] != family.pair(n).input_dim():
            raise ValueError(f"{op}: shape mismatch")


def fcs_dense_batched(t: DenseTensor, families: Sequence[HashFamily],
                      packed: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                      workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """D dense FCSs in one launch (K1); returns a D x J~ fp64 device tensor."""
    fams = list(families)
    for f in fams:
        _require_family(t.shape(), f, "fcs_sketch")
    lens = fams[0].hash_lens()
    if any(f.hash_lens() != lens for f in fams):
        raise ValueError("fcs_sketch: families differ in hash lengths")
    dims = t.shape()
    jt = fams[0].composed_len()
    if packed is None:
        packed = packed_families(fams)
    if out is None:
        out = torch.empty((len(fams), jt), dtype=torch.float64, device=_dev())
    ws_bytes = L.lib().st_fcs_dense_workspace(t.st_dtype, len(dims), L.size_array(dims),
                                              dims[-1], len(fams), L.size_array(lens))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=_dev())
    _check(L.lib().st_fcs_dense(t.st_dtype, _ptr(t.flat), len(dims), L.size_array(dims), 0,
                                dims[-1], len(fams), _ptr(packed), L.size_array(lens), _ptr(out),
                                0, _ptr(workspace), ws_bytes, _stream()))
    return out


def fcs_coo_batched(values, coords, shape, families: Sequence[HashFamily],
                    packed: Optional[torch.Tensor] = None) -> torch.Tensor:
    """D FCSs of a sparse tensor given as COO (st_fcs_coo, O(nnz)): values
    (nnz, fp32 or fp64) at coords (nnz x order, integer), shape = the dense
    shape. Equals fcs_sketch of the densified tensor (duplicates add up);
    ValueError "compose: index out of range" (hashing.cpp:90-92) for a
    coordinate outside the shape. Returns D x J~ fp64 on the device."""
    fams = list(families)
    shape = [int(x) for x in shape]
    for f in fams:
        _require_family(shape, f, "fcs_sketch")
    lens = fams[0].hash_lens()
    if any(f.hash_lens() != lens for f in fams):
        raise ValueError("fcs_sketch: families differ in hash lengths")
    v = torch.as_tensor(values if torch.is_tensor(values) else np.asarray(values)).reshape(-1)
    if v.dtype not in (torch.float32, torch.float64):
        v = v.to(torch.float64)
    v = v.to(_dev()).contiguous()
    c = torch.as_tensor(coords if torch.is_tensor(coords) else np.asarray(coords))
    nnz = v.numel()
    c = c.reshape(nnz, len(shape))
    if c.numel() and (int(c.min()) < 0 or int(c.max()) >= 2 ** 32):
        raise ValueError("compose: index out of range")
    c = c.to(torch.int64).to(_dev()).to(torch.int32).contiguous()  # uint32 bit pattern
    if packed is None:
        packed = packed_families(fams)
    out = torch.empty((len(fams), fams[0].composed_len()), dtype=torch.float64, device=_dev())
    bad = torch.zeros(1, dtype=torch.int64, device=_dev())
    dt = L.ST_F32 if v.dtype == torch.float32 else L.ST_F64
    _check(L.lib().st_fcs_coo(dt, _ptr(v), _ptr(c), nnz, len(shape), L.size_array(shape),
                              len(fams), _ptr(packed), L.size_array(lens), _ptr(out), 0,
                              _ptr(bad), _stream()))
    if int(bad.item()):
        raise ValueError("compose: index out of range")
    return out


def fcs_cp_batched(cp: CpTensor, families: Sequence[HashFamily],
                   packed: Optional[torch.Tensor] = None) -> torch.Tensor:
    """D CP-form FCSs (K2-K5); returns a D x J~ fp64 device tensor."""
    fams = list(families)
    for f in fams:
        _require_family(cp.shape(), f, "fcs_sketch")
    lens = fams[0].hash_lens()
    dims = cp.shape()
    jt = fams[0].composed_len()
    if packed is None:
        packed = packed_families(fams)
    out = torch.empty((len(fams), jt), dtype=torch.float64, device=_dev())
    ws_bytes = L.lib().st_fcs_cp_workspace(len(dims), L.size_array(dims), cp.rank(), len(fams),
                                           L.size_array(lens))
    if ws_bytes == 0:  # plan refused (composed length beyond the smem FFT); message is set
        _check(L.ST_EINVAL)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=_dev())
    fptrs = (C.c_void_p * len(dims))(*[f.data_ptr() for f in cp._factors_cm])
    _check(L.lib().st_fcs_cp(_ptr(cp.weights), cp.rank(), len(dims), L.size_array(dims), fptrs, 0,
                             cp.rank(), len(fams), _ptr(packed), L.size_array(lens), _ptr(out), 0,
                             _ptr(ws), ws_bytes, _stream()))
    return out


def fcs_sketch(t, family: HashFamily) -> SketchVec:
    """fcs_sketch(DenseTensor|CpTensor, HashFamily) (sketch.hpp:56,60;
    sketch.cpp:187-207)."""
    if isinstance(t, CpTensor):
        vals = fcs_cp_batched(t, [family])[0]
    else:
        if not isinstance(t, DenseTensor):
            t = DenseTensor.from_array(t)
        vals = fcs_dense_batched(t, [family])[0]
    return SketchVec(vals, family, SketchKind.FCS)


def cs_sketch_columns(u, pair: HashPair) -> torch.Tensor:
    """cs_sketch_columns (sketch.hpp:36, sketch.cpp:118-133): I x R -> J x R."""
    u = torch.as_tensor(np.asarray(u, np.float64) if not torch.is_tensor(u) else u,
                        dtype=torch.float64)
    if u.dim() == 1:
        u = u.reshape(-1, 1)
    if u.shape[0] != pair.input_dim():
        raise ValueError("cs_sketch_columns: input length mismatch")
    ucm = u.t().contiguous().to(_dev())
    out = torch.empty((u.shape[1], pair.hash_len()), dtype=torch.float64, device=_dev())
    _check(L.lib().st_cs_columns(_ptr(ucm), u.shape[0], u.shape[1], _ptr(pair.packed()),
                                 pair.hash_len(), _ptr(out), _stream()))
    return out.t()


def cs_sketch(x, pair: HashPair) -> SketchVec:
    """cs_sketch (sketch.hpp:33, sketch.cpp:105-116)."""
    x = torch.as_tensor(np.asarray(x, np.float64) if not torch.is_tensor(x) else x,
                        dtype=torch.float64).reshape(-1)
    if x.numel() != pair.input_dim():
        raise ValueError("cs_sketch: input length mismatch")
    vals = cs_sketch_columns(x.reshape(-1, 1), pair)[:, 0].contiguous()
    return SketchVec(vals, HashFamily(pairs=[pair]), SketchKind.CS)


class SketchTensor:
    """SketchTensor (sketch.hpp:24-29; shape contract sketch.cpp:98-103): a
    J_0 x ... x J_{N-1} sketch (``values``: ndarray-indexable torch tensor)."""

    def __init__(self, values: torch.Tensor, family: HashFamily):
        if list(values.shape) != family.hash_lens():
            raise ValueError("SketchTensor: shape does not match hash lengths")
        self.values = values
        self.family = family


def _cp_call(fn_ws, fn, cp: CpTensor, fams, out_len, ranks=True):
    dims = cp.shape()
    lens = fams[0].hash_lens()
    packed = packed_families(fams)
    out = torch.empty((len(fams), out_len), dtype=torch.float64, device=_dev())
    ws_bytes = fn_ws(len(dims), L.size_array(dims), cp.rank(), len(fams), L.size_array(lens))
    if ws_bytes == 0:
        _check(L.ST_EINVAL)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=_dev())
    fptrs = (C.c_void_p * len(dims))(*[f.data_ptr() for f in cp._factors_cm])
    if ranks:
        _check(fn(_ptr(cp.weights), cp.rank(), len(dims), L.size_array(dims), fptrs, 0, cp.rank(),
                  len(fams), _ptr(packed), L.size_array(lens), _ptr(out), 0, _ptr(ws), ws_bytes,
                  _stream()))
    else:
        _check(fn(_ptr(cp.weights), cp.rank(), len(dims), L.size_array(dims), fptrs, len(fams),
                  _ptr(packed), L.size_array(lens), _ptr(out), 0, _ptr(ws), ws_bytes, _stream()))
    return out


def _dense_call(fn_ws, fn, t: DenseTensor, fams, out_len):
    dims = t.shape()
    lens = fams[0].hash_lens()
    packed = packed_families(fams)
    out = torch.empty((len(fams), out_len), dtype=torch.float64, device=_dev())
    ws_bytes = fn_ws(t.st_dtype, len(dims), L.size_array(dims), dims[-1], len(fams),
                     L.size_array(lens))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=_dev())
    _check(fn(t.st_dtype, _ptr(t.flat), len(dims), L.size_array(dims), 0, dims[-1], len(fams),
              _ptr(packed), L.size_array(lens), _ptr(out), 0, _ptr(ws), ws_bytes, _stream()))
    return out


def ts_sketch(t, family: HashFamily) -> SketchVec:
    """ts_sketch(DenseTensor|CpTensor, HashFamily) (sketch.hpp:40,44;
    sketch.cpp:135-155): buckets compose by modular sum; equal J required."""
    lens = family.hash_lens()
    if any(j != lens[0] for j in lens):
        raise ValueError("ts_sketch: all hash lengths must be equal")
    lib = L.lib()
    if isinstance(t, CpTensor):
        _require_family(t.shape(), family, "ts_sketch")
        vals = _cp_call(lib.st_ts_cp_workspace, lib.st_ts_cp, t, [family], lens[0])[0]
    else:
        if not isinstance(t, DenseTensor):
            t = DenseTensor.from_array(t)
        _require_family(t.shape(), family, "ts_sketch")
        vals = _dense_call(lib.st_ts_dense_workspace, lib.st_ts_dense, t, [family], lens[0])[0]
    return SketchVec(vals, family, SketchKind.TS)


def hcs_sketch(t, family: HashFamily) -> SketchTensor:
    """hcs_sketch(DenseTensor|CpTensor, HashFamily) (sketch.hpp:47,51;
    sketch.cpp:157-185): per-mode buckets into a J_0 x ... x J_{N-1} tensor."""
    lens = family.hash_lens()
    n_out = int(np.prod(lens))
    lib = L.lib()
    if isinstance(t, CpTensor):
        _require_family(t.shape(), family, "hcs_sketch")
        flat = _cp_call(lib.st_hcs_cp_workspace, lib.st_hcs_cp, t, [family], n_out,
                        ranks=False)[0]
    else:
        if not isinstance(t, DenseTensor):
            t = DenseTensor.from_array(t)
        _require_family(t.shape(), family, "hcs_sketch")
        flat = _dense_call(lib.st_hcs_dense_workspace, lib.st_hcs_dense, t, [family], n_out)[0]
    # column-major flat -> tensor indexed [j_0, ..., j_{N-1}]
    vals = flat.reshape(list(reversed(lens))).permute(*reversed(range(len(lens))))
    return SketchTensor(vals, family)


def convolve_pairs(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Row-wise linear convolution (fft_convolve with two inputs, fft.cpp:75-84)."""
    a = a.to(_dev(), torch.float64).contiguous()
    b = b.to(_dev(), torch.float64).contiguous()
    if a.dim() == 1:
        a, b = a.reshape(1, -1), b.reshape(1, -1)
    out = torch.empty((a.shape[0], a.shape[1] + b.shape[1] - 1), dtype=torch.float64,
                      device=_dev())
    _check(L.lib().st_convolve_pairs(_ptr(a), a.shape[1], _ptr(b), b.shape[1], a.shape[0],
                                     _ptr(out), _stream()))
    return out


def fcs_kron(A, B, families: Sequence[HashFamily]) -> torch.Tensor:
    """FCS of the outer-product tensor A o B (4-mode families p0..p3):
    conv(FCS_{p0,p1}(vec A), FCS_{p2,p3}(vec B)). D x J~."""
    fams = list(families)
    A = torch.as_tensor(np.asarray(A, np.float64) if not torch.is_tensor(A) else A,
                        dtype=torch.float64)
    B = torch.as_tensor(np.asarray(B, np.float64) if not torch.is_tensor(B) else B,
                        dtype=torch.float64)
    dims = [A.shape[0], A.shape[1], B.shape[0], B.shape[1]]
    for f in fams:
        _require_family(dims, f, "fcs_kron")
    lens = fams[0].hash_lens()
    packed = packed_families(fams)
    acm = A.t().contiguous().to(_dev())
    bcm = B.t().contiguous().to(_dev())
    out = torch.empty((len(fams), fams[0].composed_len()), dtype=torch.float64, device=_dev())
    _check(L.lib().st_fcs_kron(_ptr(acm), dims[0], dims[1], _ptr(bcm), dims[2], dims[3],
                               len(fams), _ptr(packed), L.size_array(lens), _ptr(out), _stream()))
    return out


def median_reduce(values):
    """median_reduce (estimators.cpp:117-138): host helper over small inputs."""
    v = np.asarray(values, np.float64)
    if v.size == 0:
        raise ValueError("median_reduce: empty input")
    s = np.sort(v, axis=0)
    n = s.shape[0]
    return s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])


# ------------------------------------------------------------------ fft.hpp
def _dvec(x) -> torch.Tensor:
    return torch.as_tensor(x if torch.is_tensor(x) else np.asarray(x, np.float64),
                           dtype=torch.float64).reshape(-1).to(_dev()).contiguous()


def dft(x, n: int) -> torch.Tensor:
    """dft (fft.cpp:42-51): the n-point complex DFT of x zero-padded (or
    truncated) to EXACTLY n points, e^{-i} and unnormalised — st_dft, a
    Bluestein chirp-z over the library's own FFTs (fft.cuh / the two-level
    transform). Returns a complex128 device tensor of n bins."""
    if n == 0:
        raise ValueError("dft: zero length")
    v = _dvec(x)
    out = torch.empty(2 * n, dtype=torch.float64, device=_dev())
    _check(L.lib().st_dft(_ptr(v), v.numel(), n, _ptr(out), _stream()))
    return torch.view_as_complex(out.view(n, 2))


def idft_real(spectrum) -> torch.Tensor:
    """idft_real (fft.cpp:53-73): real part of the normalised inverse DFT at
    the spectrum's length (st_idft_real); RuntimeError when the imaginary
    residue exceeds 1e-9 of the real norm (+1e-12), as the reference."""
    s = torch.as_tensor(spectrum if torch.is_tensor(spectrum) else np.asarray(spectrum),
                        dtype=torch.complex128).reshape(-1).to(_dev()).contiguous()
    n = s.numel()
    if n == 0:
        raise ValueError("idft_real: zero length")
    out = torch.empty(n, dtype=torch.float64, device=_dev())
    _check(L.lib().st_idft_real(_ptr(torch.view_as_real(s)), n, _ptr(out), 1, _stream()))
    return out


def fft_convolve(inputs, n: int) -> torch.Tensor:
    """fft_convolve (fft.cpp:75-84): F^-1(prod F(x_i, n)) at exactly n points
    (circular; linear when n >= sum(len) - k + 1) — st_fft_convolve."""
    if len(inputs) == 0:
        raise ValueError("fft_convolve: no inputs")
    if n == 0:
        raise ValueError("dft: zero length")
    vs = [_dvec(x) for x in inputs]
    ptrs = (C.c_void_p * len(vs))(*[v.data_ptr() for v in vs])
    out = torch.empty(n, dtype=torch.float64, device=_dev())
    _check(L.lib().st_fft_convolve(ptrs, L.size_array([v.numel() for v in vs]), len(vs), n,
                                   _ptr(out), _stream()))
    return out
