"""CPU tests of bench.py's driver contract that need no GPU: `--gpus N`
relaunches itself as N ranks (gloo probe), and the reference arm runs the
unmodified reference (oracle/_ref) without importing the product package."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_n_spawns_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--probe"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["ranks_seen"] == 2


def test_reference_workload_does_not_import_package():
    code = ("import sys, bench\n"
            "w = bench.RefC4(4, 2, 2)\n"
            "w.run()\n"
            "w.close()\n"
            "bad = [m for m in sys.modules if m.startswith('paper_2106_13062_b200')]\n"
            "assert not bad, bad\n"
            "print('ok', w.elements)\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert "ok 4194304" in r.stdout


def test_reference_chunks_sum_to_whole_tensor_sketch():
    """The chunked reference pass equals one fcs_sketch of the whole sample."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from oracle import ref
    w = bench.RefC4(3, 3, 1)
    w.run()
    got = w.parts.reshape(len(w.chunks), bench.C4_D, w.jt).sum(axis=0)
    xs = []  # each chunk draws from its own seed: rebuild them explicitly
    for (s0, s1) in w.chunks:
        t = ref.gaussian(bench.C4_SEED * 1000003 + s0, 1024 * 1024 * (s1 - s0))
        xs.append(t.astype(np.float32).astype(np.float64))
    x = np.concatenate(xs).reshape((1024, 1024, 3), order="F")
    for d in range(bench.C4_D):
        b, s = w.fams[d]
        want = ref.fcs_dense_tables(x, [b[0], b[1], b[2][:3]], [s[0], s[1], s[2][:3]],
                                    [bench.C4_J] * 3)
        assert np.allclose(got[d], want, rtol=1e-12, atol=1e-9 * np.abs(want).max())
    w.close()
