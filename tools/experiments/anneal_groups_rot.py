"""Offline joint annealing of K1 line groups and per-(step, lane) component
rotations for the config-4 families: writes D x 32 group bytes followed by
D x 8 x 32 rotation bytes (ST_FX_GROUPS_FILE + ST_FX_ROT probe)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import fcs_oracle as O  # noqa: E402

rng = np.random.default_rng(0)


def anneal(L, choices, iters=40000, T0=1.0):
    groups = np.arange(32).reshape(8, 4).copy()
    rot = np.zeros((8, 32), int)

    def step_cost(j):
        cnt = np.zeros((4, 32), int)
        for l in range(32):
            vals = L[groups[j][l // 8], 4 * (l % 8):4 * (l % 8) + 4]
            for k in range(4):
                cnt[k, vals[(k + rot[j][l]) % 4]] += 1
        return cnt.max(axis=1).sum()
    costs = [step_cost(j) for j in range(8)]
    cur = sum(costs)
    best, bg, br = cur, groups.copy(), rot.copy()
    for it in range(iters):
        T = T0 * (1 - it / iters) + 1e-3
        if len(choices) > 1 and rng.random() < 0.6:
            j = rng.integers(8); l = rng.integers(32); old = rot[j][l]
            rot[j][l] = choices[rng.integers(len(choices))]
            nc = step_cost(j); dd = nc - costs[j]
            if dd <= 0 or rng.random() < np.exp(-dd / T):
                costs[j] = nc; cur += dd
            else:
                rot[j][l] = old
        else:
            j1, j2 = rng.integers(8, size=2); q1, q2 = rng.integers(4, size=2)
            if j1 == j2:
                continue
            groups[j1][q1], groups[j2][q2] = groups[j2][q2], groups[j1][q1]
            n1, n2 = step_cost(j1), step_cost(j2); dd = n1 + n2 - costs[j1] - costs[j2]
            if dd <= 0 or rng.random() < np.exp(-dd / T):
                costs[j1], costs[j2] = n1, n2; cur += dd
            else:
                groups[j1][q1], groups[j2][q2] = groups[j2][q2], groups[j1][q1]
        if cur < best:
            best, bg, br = cur, groups.copy(), rot.copy()
    return bg, br, best / 32


def main(out, choices):
    fams = O.families_for([1024, 1024, 1024], 16384, 4, 4)
    gs, rs = [], []
    for d, (b, s, j) in enumerate(fams):
        L = (np.asarray(b[0]) % 32).reshape(32, 32)
        g, r, score = anneal(L, choices)
        print(f"family {d}: {score:.3f} wavefronts/ATOMS")
        gs.append(g.astype(np.uint8).ravel())
        rs.append(r.astype(np.uint8).ravel())
    np.concatenate(gs + rs).tofile(out)


if __name__ == "__main__":
    main(sys.argv[1], [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3])
