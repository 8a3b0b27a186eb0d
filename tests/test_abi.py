"""CPU tests of the drop-in boundary: the C-ABI library builds for sm_100a,
loads without a GPU, and exports exactly the symbols include/fcs_b200.h declares."""
import os
import re
import subprocess

import pytest

from paper_2106_13062_b200 import _lib

HEADER = _lib.HEADER


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(st_\w+)\s*\(", text,
                                 re.M)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for must in ("st_hash_tabulate", "st_family_tables", "st_fcs_dense", "st_fcs_cp",
                 "st_engine_iuv", "st_engine_uvw", "st_engine_deflate", "st_rtpm", "st_fcs_kron"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2106_13062_b200 import build
        build.build()
    lib = _lib.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_host_calls_without_gpu():
    # st_family_seed is pure host arithmetic: family_seed(0, d) (Appendix A)
    lib = _lib.lib()
    assert lib.st_family_seed(0, 0) == 0xE220A8397B1DCDAF
    assert lib.st_family_seed(0, 1) == 0x910A2DEC89025CC1
    assert lib.st_abi_version() == 3


def test_host_gaussian_matches_reference_stream():
    import numpy as np
    from oracle import fcs_oracle as O
    from paper_2106_13062_b200 import configs
    from oracle import ref
    got = configs.host_gaussian(5, 200001)  # multi-threaded path
    # numpy's SIMD log/cos may differ from glibc by 1 ulp; the C-ABI uses libm
    np.testing.assert_allclose(got, O.gaussian_stream(5, 200001), rtol=0, atol=1e-14)
    if ref.available():  # bit-identical to the reference's serial next_gaussian
        assert (got == ref.gaussian(5, 200001)).all()


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2106_13062_b200 import HashPair
    with pytest.raises(RuntimeError):
        HashPair(10, 5, 1)
