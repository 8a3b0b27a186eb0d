"""ctypes binding of the C-ABI in ``include/fcs_b200.h`` (``_lib/libfcs_b200.so``).

There is no CPU fallback: if the library is missing or no sm_100 GPU is
usable, every compute call raises. Status codes map to the reference's
exception types (``ST_EINVAL`` -> ValueError like std::invalid_argument,
``ST_ENUMERIC`` -> RuntimeError like std::runtime_error).
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libfcs_b200.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "fcs_b200.h")

ST_OK, ST_EINVAL, ST_ENUMERIC, ST_ECUDA, ST_ENCCL, ST_ENOMEM = range(6)
ST_F32, ST_F64 = 0, 1
ST_BACKEND_PLAIN, ST_BACKEND_CS, ST_BACKEND_TS, ST_BACKEND_HCS, ST_BACKEND_FCS = range(5)
ST_SKETCH_CS, ST_SKETCH_TS, ST_SKETCH_FCS = range(3)
MAX_ORDER = 8

p, sz, u64, i32, dbl = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int, C.c_double

# name -> (restype, argtypes); every symbol declared in include/fcs_b200.h.
SIGNATURES = {
    "st_last_error": (C.c_char_p, []),
    "st_abi_version": (i32, []),
    "st_device_query": (i32, [p, p, p]),
    "st_family_seed": (u64, [u64, sz]),
    "st_hash_tabulate": (i32, [u64, sz, sz, p, p, p]),
    "st_family_tables": (i32, [sz, p, p, sz, p, p, p]),
    "st_pack_tables": (i32, [sz, p, p, p, p]),
    "st_fcs_dense_workspace": (sz, [i32, sz, p, sz, sz, p]),
    "st_fcs_dense": (i32, [i32, p, sz, p, sz, sz, sz, p, p, p, i32, p, sz, p]),
    "st_fcs_dense_host": (i32, [i32, p, sz, p, sz, sz, sz, p, p, p]),
    "st_fcs_dense_host_tables": (i32, [i32, p, sz, p, sz, sz, sz, p, p, p]),
    "st_fcs_dense_report": (i32, [i32, sz, p, sz, sz, p, p, sz, p, p, p]),
    "st_cs_columns": (i32, [p, sz, sz, p, sz, p, p]),
    "st_fcs_coo": (i32, [i32, p, p, sz, sz, p, sz, p, p, p, i32, p, p]),
    "st_cs_expand": (i32, [p, sz, p, sz, p, p]),
    "st_fcs_cp_workspace": (sz, [sz, p, sz, sz, p]),
    "st_fcs_cp": (i32, [p, sz, sz, p, p, sz, sz, sz, p, p, p, i32, p, sz, p]),
    "st_convolve_pairs": (i32, [p, sz, p, sz, sz, p, p]),
    "st_fcs_kron": (i32, [p, sz, sz, p, sz, sz, sz, p, p, p, p]),
    "st_dft": (i32, [p, sz, sz, p, p]),
    "st_idft_real": (i32, [p, sz, p, i32, p]),
    "st_fft_convolve": (i32, [p, p, sz, sz, p, p]),
    "st_precompute_z": (i32, [p, sz, p, sz, p, sz, p, sz, p, sz, p, p]),
    "st_ts_dense_workspace": (sz, [i32, sz, p, sz, sz, p]),
    "st_ts_dense": (i32, [i32, p, sz, p, sz, sz, sz, p, p, p, i32, p, sz, p]),
    "st_ts_cp_workspace": (sz, [sz, p, sz, sz, p]),
    "st_ts_cp": (i32, [p, sz, sz, p, p, sz, sz, sz, p, p, p, i32, p, sz, p]),
    "st_hcs_dense_workspace": (sz, [i32, sz, p, sz, sz, p]),
    "st_hcs_dense": (i32, [i32, p, sz, p, sz, sz, sz, p, p, p, i32, p, sz, p]),
    "st_hcs_cp_workspace": (sz, [sz, p, sz, sz, p]),
    "st_hcs_cp": (i32, [p, sz, sz, p, p, sz, p, p, p, i32, p, sz, p]),
    "st_engine_create": (i32, [p, i32, p, p, sz, sz, u64, p]),
    "st_engine_create_backend": (i32, [p, i32, i32, p, p, sz, sz, u64, p]),
    "st_engine_from_sketches": (i32, [p, i32, p, sz, p, sz, p, p]),
    "st_engine_destroy": (i32, [p]),
    "st_engine_backend": (i32, [p]),
    "st_engine_composed_len": (sz, [p]),
    "st_engine_sketches": (i32, [p, p, p]),
    "st_engine_iuv": (i32, [p, sz, p, p, sz, p, i32, p]),
    "st_engine_uvw": (i32, [p, sz, p, p, p, p, i32, p]),
    "st_engine_deflate": (i32, [p, dbl, p, p, p, p]),
    "st_engine_set_path": (i32, [p, i32]),
    "st_rtpm": (i32, [i32, p, sz, sz, sz, sz, sz, sz, u64, p, p, p]),
    "st_rtpm_backend": (i32, [i32, i32, p, sz, sz, sz, sz, sz, sz, u64, p, p, p]),
    "st_rtpm_asym": (i32, [i32, i32, p, p, sz, sz, sz, sz, sz, u64, p, p, p]),
    "st_als": (i32, [i32, i32, p, p, sz, sz, dbl, sz, sz, u64, p, p, p, p]),
    "st_residual_norm": (i32, [i32, p, p, p, sz, p, p, p]),
    "st_densify": (i32, [sz, p, sz, p, p, p, p]),
    "st_psnr": (i32, [i32, p, p, sz, p, p]),
    "st_estimate_inner": (i32, [i32, i32, p, p, sz, p, sz, sz, u64, p, p, p]),
    "st_sketch_dots": (i32, [sz, sz, p, p, p, p]),
    "st_regression_forward": (i32, [i32, p, sz, p, sz, p, sz, p, sz, sz, u64, p, p]),
    "st_fcs_contraction": (i32, [i32, p, p, p, p, sz, p, p, p, p]),
    "st_sketch_decompress": (i32, [p, sz, sz, p, sz, p, sz, p, p, p]),
    "st_kron_decompress_all": (i32, [p, sz, sz, p, p, p, p]),
    "st_nccl_unique_id_bytes": (sz, []),
    "st_nccl_get_unique_id": (i32, [p]),
    "st_nccl_comm_init_rank": (i32, [p, i32, p, i32]),
    "st_nccl_comm_destroy": (i32, [p]),
    "st_shard_range": (i32, [sz, i32, i32, p, p]),
    "st_fcs_dense_nccl": (i32, [i32, p, sz, p, sz, p, p, p, p, sz, p, p]),
    "st_fcs_cp_nccl": (i32, [p, sz, sz, p, p, sz, p, p, p, p, sz, p, p]),
    "st_host_gaussian": (i32, [u64, sz, p, i32]),
    "st_device_gaussian": (i32, [i32, u64, sz, p, p]),
}

_lib = None


class LibraryMissing(ImportError):
    pass


def lib():
    """Load the CUDA library (fails loudly; never falls back to CPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} not built: run `python -m paper_2106_13062_b200.build` "
            "(no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)  # AttributeError if an exported symbol is missing
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == ST_OK:
        return
    msg = lib().st_last_error().decode(errors="replace")
    if rc == ST_EINVAL:
        raise ValueError(msg)
    if rc == ST_ENUMERIC:
        raise RuntimeError(msg)
    if rc == ST_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"fcs_b200 error {rc}: {msg}")


def size_array(values):
    arr = (C.c_size_t * max(len(values), 1))(*[int(v) for v in values])
    return arr


def u64_array(values):
    return (C.c_uint64 * max(len(values), 1))(*[int(v) & ((1 << 64) - 1) for v in values])
