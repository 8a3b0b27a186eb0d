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
