"""The reference-side C++ binding (integration/gpu_fcs_engine.cpp, compiled
against the reference's own headers) behaves like the reference FcsEngine on
every ContractionEngine call and through a power-iteration driver written only
against that interface (integration/test_drop_in.cpp)."""
import json
import os
import subprocess

import pytest

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration",
                   "_build", "test_drop_in")


@pytest.mark.gpu
def test_cpp_drop_in_engine(cuda):
    assert os.path.exists(BIN), "integration/_build/test_drop_in not built (make -C integration)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1]
    res = json.loads(line)
    assert r.returncode == 0 and res["ok"], r.stdout + r.stderr
