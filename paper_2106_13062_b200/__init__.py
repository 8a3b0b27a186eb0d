"""B200-native fast count sketch (FCS) — arXiv 2106.13062 hot path.

sm_100a CUDA kernels behind the C-ABI in ``include/fcs_b200.h``
(``_lib/libfcs_b200.so``), with a host mirror of the reference's
``sketchtensor`` API. Importing the package does not touch the GPU; the first
compute call loads the library and fails loudly if it or the GPU is missing.
"""
from .sketchtensor import (CpTensor, DenseTensor, EstimatorConfig, HashFamily, HashPair,  # noqa
                           SketchKind, SketchTensor, SketchVec, convolve_pairs, cs_sketch,
                           cs_sketch_columns,
                           families_for, family_seed, fcs_coo_batched, fcs_cp_batched,
                           fcs_dense_batched,
                           fcs_kron, fcs_sketch, hcs_sketch, median_reduce, packed_families,
                           ts_sketch, dft, idft_real, fft_convolve)
from .engine import (AlsConfig, ContractionEngine, CsEngine, FcsEngine, HcsEngine,  # noqa
                     PlainEngine, RtpmConfig, SketchBackend,
                     TsEngine, als, backend_from_name, backend_name, make_contraction_engine,
                     residual_norm, rtpm, rtpm_asym, psnr, densify, rank_one, contract3,
                     contract3_free, inner, mode_unfold, mode_fold, contract_pair, kron,
                     tensor_from_matrix)

from .codecs import (KronSketch, compress_contraction, compress_kron, compression_ratio,  # noqa
                     decompress_contraction, decompress_kron, estimate_inner, hash_memory,
                     hash_memory_long_pair, inner_once, inner_once_ts, reconstruct_kron,
                     sketched_regression_forward)

__all__ = [n for n in dir() if not n.startswith("_")]
