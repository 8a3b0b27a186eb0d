"""CPU multi-process tests (gloo, world_size 2) of the N>1 path: the slab
partition and the single all-reduce reproduce the single-process sketch.
Per-rank partial sketches come from the oracle (the CPU checker stands in for
the GPU kernel here); the partition and the collective are the product code
in paper_2106_13062_b200/dist.py."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fcs_oracle as O
from paper_2106_13062_b200 import dist as pdist


def _worker(rank, world, port, x, fams, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def partial(lo, hi, r):
            rows = []
            for b, s, j in fams:
                slab = x[..., lo:hi]
                bs = list(b[:-1]) + [b[-1][lo:hi]]
                ss = list(s[:-1]) + [s[-1][lo:hi]]
                rows.append(O.fcs_dense(slab, bs, ss, j) if hi > lo else
                            np.zeros(O.composed_len(j)))
            return torch.from_numpy(np.stack(rows))
        out = pdist.sharded_sketch(partial, x.shape[-1])
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,last", [(2, 9), (2, 1), (3, 7)])
def test_sharded_sketch_matches_single(world, last):
    rng = np.random.default_rng(world * 10 + last)
    x = rng.integers(-5, 6, size=(6, 5, last)).astype(np.float64)
    fams = O.families_for(x.shape, 4, 2, 17)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 17 + last
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, fams, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.stack([O.fcs_dense(x, b, s, j) for b, s, j in fams])
    for r in range(world):
        assert (res[r] == want).all()  # integer data: exact


def test_shard_range_partitions():
    for n in (0, 1, 7, 1024):
        for w in (1, 2, 3, 8):
            rs = [pdist.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
    with pytest.raises(ValueError):
        pdist.shard_range(4, 2, 2)


# ------------------------------------------------ restart-sharded RTPM (c3)
class _OracleBatchEngine:
    """The oracle FcsEngine behind the batched engine interface sharded_rtpm uses
    (the CPU checker stands in for the GPU engine; the driver is product code)."""

    def __init__(self, t, J, D, seed):
        self.e = O.FcsEngine(t, J, D, seed)

    def iuv_batch(self, A, B, f):
        return np.stack([self.e.iuv(a, b, f) for a, b in zip(A, B)])

    def uvw_batch(self, U, V, W):
        return np.array([self.e.uvw(u, v, w) for u, v, w in zip(U, V, W)])

    def iuu(self, u):
        return self.e.iuu(u)

    def uuu(self, u):
        return self.e.uuu(u)

    def deflate(self, w, u, v, x):
        self.e.deflate(w, u, v, x)


def _rtpm_worker(rank, world, port, t, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = _OracleBatchEngine(t, 12, 3, 21)
        w, f = pdist.sharded_rtpm(eng, t.shape[0], 2, 5, 4, 21)
        q.put((rank, w, f))
    finally:
        dist.destroy_process_group()


def _run(world, target, args, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        item = q.get(timeout=180)
        res[item[0]] = item[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_rtpm_matches_single(world):
    """Restarts split over ranks (5 restarts on 2 or 3 ranks, uneven) give the
    single-process rtpm result on every rank."""
    rng = np.random.default_rng(4)
    qm, _ = np.linalg.qr(rng.standard_normal((10, 2)))
    t = np.einsum("r,ir,jr,kr->ijk", [2.0, 1.0], qm, qm, qm) + 1e-3 * rng.standard_normal(
        (10, 10, 10))
    res = _run(world, _rtpm_worker, (t,), 29700 + world)
    w0, f0 = O.rtpm(O.FcsEngine(t, 12, 3, 21), 10, 2, 5, 4, 21)
    for r in range(world):
        w, f = res[r]
        np.testing.assert_allclose(w, w0, rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(f, f0, rtol=1e-12, atol=1e-14)


def _family_worker(rank, world, port, a, b, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fams = O.families_for((3, 4, 4, 5), 6, 5, 2)
        K = O.kron_tensor(a, b)
        out = pdist.sharded_families(
            lambda lo, hi: torch.from_numpy(np.stack([O.fcs_dense(K, *fams[d])
                                                      for d in range(lo, hi)])
                                            if hi > lo else np.zeros((0, 4 * 6 - 3))), 5)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_families_kron(world):
    """Config 5's family split (one sketch per rank; here 5 families over 2/3 ranks)."""
    rng = np.random.default_rng(7)
    a, b = rng.standard_normal((3, 4)), rng.standard_normal((4, 5))
    res = _run(world, _family_worker, (a, b), 29800 + world)
    fams = O.families_for((3, 4, 4, 5), 6, 5, 2)
    want = np.stack([O.fcs_dense(O.kron_tensor(a, b), *f) for f in fams])
    for r in range(world):
        np.testing.assert_array_equal(res[r][0], want)


def _cp_worker(rank, world, port, w, fs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fams = O.families_for(tuple(f.shape[0] for f in fs), 7, 2, 3)
        lo, hi = pdist.shard_ranks(len(w), rank, world)
        part = np.stack([O.fcs_cp(w[lo:hi], [f[:, lo:hi] for f in fs], *fam) if hi > lo else
                         np.zeros(3 * 7 - 2) for fam in fams])
        out = pdist.allreduce_sketch(torch.from_numpy(part))
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_sharded_cp(world):
    """Config 2's rank split: per-rank sums over r-slices, one all-reduce."""
    rng = np.random.default_rng(9)
    w = rng.standard_normal(5)
    fs = [rng.standard_normal((n, 5)) for n in (6, 5, 4)]
    res = _run(world, _cp_worker, (w, fs), 29900 + world)
    fams = O.families_for((6, 5, 4), 7, 2, 3)
    want = np.stack([O.fcs_cp(w, fs, *fam) for fam in fams])
    for r in range(world):
        np.testing.assert_allclose(res[r][0], want, rtol=1e-12, atol=1e-12)


def test_c_abi_shard_range_matches_python():
    """The C-ABI's slab / rank-range rule (st_shard_range, used by the NCCL
    entries) is the one dist.py shards with."""
    import ctypes as C
    from paper_2106_13062_b200 import _lib as L
    lib = L.lib()
    for n in (0, 1, 7, 1024, 1000):
        for world in (1, 2, 3, 8):
            for rank in range(world):
                lo, cnt = C.c_size_t(), C.c_size_t()
                L.check(lib.st_shard_range(n, rank, world, C.byref(lo), C.byref(cnt)))
                plo, phi = pdist.shard_range(n, rank, world)
                assert (lo.value, lo.value + cnt.value) == (plo, phi)
