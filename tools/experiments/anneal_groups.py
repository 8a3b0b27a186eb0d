"""Offline line grouping for K1 (config 4 families) by simulated annealing over
step swaps: writes groups[d][j][q] (uint8, D x 8 x 4) for the
ST_FX_GROUPS_FILE probe, and prints the mean max-bank load per ATOMS of the
greedy-equivalent identity start vs the annealed grouping."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import fcs_oracle as O  # noqa: E402

rng = np.random.default_rng(0)


def anneal(L, iters=30000, T0=1.0):
    lh = np.zeros((32, 4, 32), np.int32)
    for w in range(32):
        for k in range(4):
            lh[w, k] = np.bincount(L[w, k::4], minlength=32)
    groups = np.arange(32).reshape(8, 4).copy()
    H = np.array([lh[groups[j]].sum(0) for j in range(8)])  # 8 x 4 x 32
    cost = H.max(axis=2).sum(axis=1)
    cur = cost.sum()
    best, best_g = cur, groups.copy()
    for it in range(iters):
        T = T0 * (1 - it / iters) + 1e-3
        j1, j2 = rng.integers(8, size=2)
        if j1 == j2:
            continue
        q1, q2 = rng.integers(4, size=2)
        a, b = groups[j1, q1], groups[j2, q2]
        h1 = H[j1] - lh[a] + lh[b]
        h2 = H[j2] - lh[b] + lh[a]
        c1, c2 = h1.max(axis=1).sum(), h2.max(axis=1).sum()
        d = c1 + c2 - cost[j1] - cost[j2]
        if d <= 0 or rng.random() < np.exp(-d / T):
            groups[j1, q1], groups[j2, q2] = b, a
            H[j1], H[j2], cost[j1], cost[j2] = h1, h2, c1, c2
            cur += d
            if cur < best:
                best, best_g = cur, groups.copy()
    return best_g, best / 32


def main(out, D=4, seed=4):
    fams = O.families_for([1024, 1024, 1024], 16384, D, seed)
    gs = []
    for d, (b, s, j) in enumerate(fams):
        L = (np.asarray(b[0]) % 32).reshape(32, 32)
        g, score = anneal(L)
        ident = np.mean([np.bincount(L[4 * j:4 * j + 4, k::4].ravel(), minlength=32).max()
                         for j in range(8) for k in range(4)])
        print(f"family {d}: identity {ident:.3f} -> annealed {score:.3f} wavefronts/ATOMS")
        assert sorted(g.ravel().tolist()) == list(range(32))
        gs.append(g.astype(np.uint8))
    np.stack(gs).tofile(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "groups_annealed.bin")
