"""Offline quad grouping for the TMA-staged K1 probe (fcs_dense_fxt_kernel):
per family, partition the 256 16-byte quads of a 1024-element fiber into 8
groups of 32 (one LDS.128 + 4 ATOMS per lane each) so each ATOMS spreads over
as many banks as possible, keeping slot i on a quad with quad % 8 == i % 8
(conflict-free LDS.128). Writes quads[d][g][lane] (uint8) for ST_FXT_QUADS and
prints the mean max-bank load per ATOMS (identity vs searched)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import fcs_oracle as O  # noqa: E402

rng = np.random.default_rng(0)


def anneal(B, iters):
    nq = B.shape[0]
    G = nq // 32
    oh = np.zeros((nq, 4, 32), np.int32)
    for q in range(nq):
        for k in range(4):
            oh[q, k, B[q, k]] += 1
    groups = np.arange(nq).reshape(G, 32).copy()
    H = np.array([oh[groups[j]].sum(0) for j in range(G)])
    cf = lambda h: h.max(axis=1).sum() * 64 + (h * h).sum()  # noqa: E731
    cost = np.array([cf(H[j]) for j in range(G)])
    for it in range(iters):
        T = 64.0 * (1 - it / iters) + 1e-3
        j1, j2 = rng.integers(G, size=2)
        if j1 == j2:
            continue
        q1 = rng.integers(32)
        q2 = (q1 % 8) + 8 * rng.integers(4)
        a, b = groups[j1, q1], groups[j2, q2]
        h1 = H[j1] - oh[a] + oh[b]
        h2 = H[j2] - oh[b] + oh[a]
        c1, c2 = cf(h1), cf(h2)
        dl = c1 + c2 - cost[j1] - cost[j2]
        if dl <= 0 or rng.random() < np.exp(-dl / T):
            groups[j1, q1], groups[j2, q2] = b, a
            H[j1], H[j2], cost[j1], cost[j2] = h1, h2, c1, c2
    score = np.mean([H[j].max(axis=1) for j in range(G)])
    return groups, score


def main(out, D=4, seed=4, iters=200000):
    fams = O.families_for([1024, 1024, 1024], 16384, D, seed)
    gs = []
    for d, (b, s, j) in enumerate(fams):
        B = (np.asarray(b[0]) % 32).reshape(256, 4)
        ident = np.mean([np.bincount(B[32 * j:32 * j + 32, k], minlength=32).max()
                         for j in range(8) for k in range(4)])
        g, score = anneal(B, iters)
        assert sorted(g.ravel().tolist()) == list(range(256))
        assert all(g[j, i] % 8 == i % 8 for j in range(8) for i in range(32))
        print(f"family {d}: identity {ident:.3f} -> searched {score:.3f} wavefronts/ATOMS")
        gs.append(g.astype(np.uint8))
    np.stack(gs).tofile(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "quads_c4.bin")
