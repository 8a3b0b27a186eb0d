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
