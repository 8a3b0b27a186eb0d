"""Multi-GPU partitioning of the FCS hot path (one process per GPU).

Dense FCS is linear in the tensor, so elements are sharded by
contiguous slabs of the LAST (slowest) mode — BASELINE's "leading mode" read
as the one that keeps shards contiguous in the column-major layout
(tensor.hpp:10-13). Each rank sketches its slab with the full replicated
tables (K1 with last_begin/last_count) and the D x J~ partials are summed with
ONE all-reduce (NCCL over NVLink on the GPU box; gloo in the CPU tests).
CP-form FCS shards the rank index r the same way (st_fcs_cp r_begin/r_count).
"""
from __future__ import annotations

from typing import Callable, Optional, Sequence

import torch
import torch.distributed as dist

from .sketchtensor import DenseTensor, HashFamily, fcs_dense_batched


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Balanced contiguous [lo, hi) of n items for `rank` of `world`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("shard_range: bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_sketch(t: DenseTensor, families: Sequence[HashFamily], rank: int, world: int,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Partial D x J~ sketch of this rank's last-mode slab of a full tensor."""
    import ctypes as C
    from . import _lib as L
    from .sketchtensor import _check, _dev, _ptr, _stream, packed_families
    fams = list(families)
    dims = t.shape()
    lo, hi = shard_range(dims[-1], rank, world)
    per_slab = t.size() // dims[-1]
    jt = fams[0].composed_len()
    lens = fams[0].hash_lens()
    if out is None:
        out = torch.empty((len(fams), jt), dtype=torch.float64, device=_dev())
    packed = packed_families(fams)
    ws = L.lib().st_fcs_dense_workspace(t.st_dtype, len(dims), L.size_array(dims), hi - lo,
                                        len(fams), L.size_array(lens))
    wbuf = torch.empty(max(ws, 1), dtype=torch.uint8, device=_dev())
    esz = t.flat.element_size()
    base = C.c_void_p(t.flat.data_ptr() + lo * per_slab * esz)
    _check(L.lib().st_fcs_dense(t.st_dtype, base, len(dims), L.size_array(dims), lo, hi - lo,
                                len(fams), _ptr(packed), L.size_array(lens), _ptr(out), 0,
                                _ptr(wbuf), ws, _stream()))
    return out


def allreduce_sketch(partial: torch.Tensor, group=None) -> torch.Tensor:
    """The single collective of the path: sum of the D x J~ partials."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return partial


def sharded_sketch(partial_fn: Callable[[int, int, int], torch.Tensor], last_dim: int,
                   group=None) -> torch.Tensor:
    """Generic driver: partial_fn(lo, hi, rank) -> partial sketch; all-reduced."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(last_dim, rank, world)
    return allreduce_sketch(partial_fn(lo, hi, rank), group)


# ------------------------------------------------------------ CP-form FCS
def shard_ranks(R: int, rank: int, world: int) -> tuple:
    """CP-form FCS (c2) shards the rank index: ranks [lo, hi) of R per process
    (st_fcs_cp r_begin/r_count; the per-rank frequency-domain sum is linear)."""
    return shard_range(R, rank, world)


def sharded_cp_sketch(cp, families: Sequence[HashFamily], group=None) -> torch.Tensor:
    """D x J~ FCS of a CP tensor with its rank terms split over the group:
    each process sums its r-range (st_fcs_cp) and one all-reduce adds them."""
    import ctypes as C
    from . import _lib as L
    from .sketchtensor import _check, _dev, _ptr, _stream, packed_families
    fams = list(families)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_ranks(cp.rank(), rank, world)
    dims, lens = cp.shape(), fams[0].hash_lens()
    out = torch.empty((len(fams), fams[0].composed_len()), dtype=torch.float64, device=_dev())
    ws = L.lib().st_fcs_cp_workspace(len(dims), L.size_array(dims), max(hi - lo, 1), len(fams),
                                     L.size_array(lens))
    wbuf = torch.empty(max(ws, 1), dtype=torch.uint8, device=_dev())
    fptrs = (C.c_void_p * len(dims))(*[f.data_ptr() for f in cp._factors_cm])
    _check(L.lib().st_fcs_cp(_ptr(cp.weights), cp.rank(), len(dims), L.size_array(dims), fptrs,
                             lo, hi - lo, len(fams), _ptr(packed_families(fams)),
                             L.size_array(lens), _ptr(out), 0, _ptr(wbuf), ws, _stream()))
    return allreduce_sketch(out, group)


# ---------------------------------------------------- per-family sharding (c5)
def sharded_families(partial_fn: Callable[[int, int], torch.Tensor], D: int,
                     group=None) -> torch.Tensor:
    """Families split over the group (c5: D = 8 Kronecker sketches, one per
    rank): partial_fn(d_lo, d_hi) -> (d_hi - d_lo) x J~ rows; all-gathered into
    D x J~ in family order (uneven splits padded for the collective)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(D, rank, world)
    mine = partial_fn(lo, hi)
    if world == 1:
        return mine
    width = mine.shape[1]
    per = -(-D // world)
    pad = torch.zeros((per, width), dtype=mine.dtype, device=mine.device)
    pad[: hi - lo] = mine
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    rows = [bufs[r][: shard_range(D, r, world)[1] - shard_range(D, r, world)[0]]
            for r in range(world)]
    return torch.cat(rows, dim=0)


# ------------------------------------------------------------- sharded RTPM
def _comm_device(group=None) -> torch.device:
    """Device for collective buffers: the current CUDA device under NCCL."""
    if dist.is_initialized() and dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _np(x):
    import numpy as np
    return x.detach().cpu().numpy() if torch.is_tensor(x) else np.asarray(x, np.float64)


def sharded_rtpm(engine, dim: int, target_rank: int, num_inits: int, num_iters: int, seed: int,
                 group=None):
    """rtpm (cpd.cpp:234-277) with the L restarts split over the group (SURVEY.md
    §8(e), config 3). Every process draws the SAME initial vectors — random_unit
    (cpd.cpp:199-204) consumes the SplitMix64(mix(seed ^ 0x7274706d)) Gaussian
    stream in order, so component r, restart l uses draws
    [(r L + l) dim, (r L + l + 1) dim) — and runs its restart slice through the
    engine's batched calls; the (value, u) pairs are all-gathered and the
    strict-`>` argmax in restart order (first wins) picks the candidate;
    refinement and deflation are replicated (every process holds the same
    sketches). `engine` provides iuv_batch(U, U, 0) -> n x dim and
    uvw_batch(U, U, U) -> n rows, iuu(u), uuu(u) and deflate(w, u, u, u).
    Returns (weights, factor dim x rank) as numpy arrays."""
    import math

    import numpy as np

    from .configs import host_gaussian
    from .sketchtensor import family_seed
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_range(num_inits, rank, world)
    init_seed = family_seed(seed ^ 0x7274706D, 0)  # SplitMix64::mix(seed ^ 0x7274706d)
    draws = host_gaussian(init_seed, target_rank * num_inits * dim).reshape(
        target_rank, num_inits, dim)

    def normalize(v):  # normalize_or_zero (cpd.cpp:208-216)
        n = math.sqrt(float(v @ v))
        return (np.zeros_like(v), False) if n < 1e-150 else (v / n, True)

    weights = np.zeros(target_rank)
    factor = np.zeros((dim, target_rank))
    per = -(-num_inits // world)
    for r in range(target_rank):
        mine = np.stack([normalize(draws[r, l])[0] if float(draws[r, l] @ draws[r, l]) > 0
                         else draws[r, l] for l in range(lo, hi)]) if hi > lo else \
            np.zeros((0, dim))
        alive = np.ones(hi - lo, bool)
        for _ in range(num_iters):
            if not alive.any():
                break
            Y = _np(engine.iuv_batch(mine, mine, 0))
            for l in np.nonzero(alive)[0]:  # a stopped restart broke out of its loop
                mine[l], alive[l] = normalize(Y[l])
        vals = _np(engine.uvw_batch(mine, mine, mine)) if hi > lo else np.zeros(0)
        # the exchange buffer lives where the process group's backend can
        # reach it: the rank's GPU under NCCL (which rejects host tensors),
        # host memory under gloo
        buf = torch.zeros((per, dim + 1), dtype=torch.float64, device=_comm_device(group))
        buf[: hi - lo, 0] = torch.from_numpy(np.asarray(vals, np.float64).reshape(-1))
        buf[: hi - lo, 1:] = torch.from_numpy(mine)
        bufs = [buf]
        if dist.is_initialized():  # (also at world 1, so a 1-GPU NCCL run exercises it)
            bufs = [torch.empty_like(buf) for _ in range(world)]
            dist.all_gather(bufs, buf, group=group)
        allv = torch.cat([bufs[q][: shard_range(num_inits, q, world)[1] -
                                  shard_range(num_inits, q, world)[0]]
                          for q in range(world)]).cpu().numpy()
        best, best_value = None, -math.inf
        for l in range(num_inits):  # strict >, first wins (cpd.cpp:260)
            if allv[l, 0] > best_value:
                best_value, best = allv[l, 0], allv[l, 1:].copy()
        if best is None:
            raise RuntimeError("rtpm: no candidate with a finite contraction value")
        for _ in range(num_iters):  # refinement, replicated (cpd.cpp:266-270)
            nxt, ok = normalize(_np(engine.iuu(best)).reshape(-1))
            if not ok:
                break
            best = nxt
        weight = float(_np(engine.uuu(best)))
        weights[r] = weight
        factor[:, r] = best
        engine.deflate(weight, best, best, best)
    return weights, factor
