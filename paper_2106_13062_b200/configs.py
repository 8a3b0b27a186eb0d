"""Seeded synthetic inputs for the five BASELINE.json configurations.

BASELINE names no dataset: every input is drawn from the
reference's own generator, SplitMix64 + Box-Muller (rng.hpp:12-48,
rng.cpp:8-21), through ``st_host_gaussian`` (host libm, bit-identical to the
serial reference stream) — except the 4 GiB config-4 tensor, which is filled
on the device (``st_device_gaussian``: same draws, CUDA libm, same
distribution, not bit-identical). Layouts are column-major (tensor.hpp:10-13).

Recipes (draw order is part of the definition):
  c1  seed 1: 3 factors 100x10 (draws in factor order, each column-major),
      columns normalised, lambda = 1, dense sum + 0.01 * N(0,1) noise drawn
      in flat column-major order. J = 1000, D = 1, estimator seed 1.
  c2  seed 2: 3 factors 400x50, normalised columns, lambda = 1. J = 4000, D = 10.
  c3  seed 3: 200x10 Gaussian -> Householder QR -> V; lambda_r = 1 + U[0,1)
      (next_double of SplitMix64(seed ^ 0x6c616d)); symmetric noise sigma 0.01
      drawn for i <= j <= k in lexicographic order and mirrored.
      J = 3000, D = 10, L = 15, T = 20, R = 10.
  c4  seed 4: 2^30 iid N(0,1) float32 (device fill). J = 16384, D = 4.
  c5  seed 5: A then B, 512x512 each, iid N(0,1). J = 2048 (4 pairs), D = 8.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass(frozen=True)
class Config:
    name: str
    dims: tuple
    hash_len: int
    sketch_count: int
    seed: int
    rank: int = 0


C1 = Config("c1_dense_100^3_f64", (100, 100, 100), 1000, 1, 1, rank=10)
C2 = Config("c2_cp_400^3_R50", (400, 400, 400), 4000, 10, 2, rank=50)
C3 = Config("c3_rtpm_200^3", (200, 200, 200), 3000, 10, 3, rank=10)
C4 = Config("c4_dense_1024^3_f32", (1024, 1024, 1024), 16384, 4, 4)
C5 = Config("c5_kron_512^2", (512, 512, 512, 512), 2048, 8, 5)
CONFIGS = {c.name.split("_")[0]: c for c in (C1, C2, C3, C4, C5)}
C3_INITS, C3_ITERS = 15, 20


def host_gaussian(seed: int, n: int) -> np.ndarray:
    """n draws of SplitMix64(seed).next_gaussian(), multi-threaded (C-ABI host call)."""
    out = np.empty(n, np.float64)
    L.check(L.lib().st_host_gaussian(C.c_uint64(seed), n, out.ctypes.data_as(C.c_void_p), 0))
    return out


def _normalized_factors(draws: np.ndarray, dims, rank: int):
    fs, off = [], 0
    for d in dims:
        f = draws[off:off + d * rank].reshape((d, rank), order="F").copy()
        f /= np.sqrt((f * f).sum(axis=0))
        fs.append(f)
        off += d * rank
    return fs, off


def densify(weights, factors) -> np.ndarray:
    """sum_r w_r u_r o v_r o w_r as an ndarray indexed [i, j, k] (tensor.cpp:86-115)."""
    a, b, c = factors
    return np.einsum("r,ir,jr,kr->ijk", np.asarray(weights, np.float64), a, b, c, optimize=True)


def c1_tensor(cfg: Config = C1) -> np.ndarray:
    n = int(np.prod(cfg.dims))
    draws = host_gaussian(cfg.seed, sum(cfg.dims) * cfg.rank + n)
    fs, off = _normalized_factors(draws, cfg.dims, cfg.rank)
    t = densify(np.ones(cfg.rank), fs)
    noise = draws[off:off + n].reshape(cfg.dims, order="F")
    return t + 0.01 * noise


def c2_cp(cfg: Config = C2):
    draws = host_gaussian(cfg.seed, sum(cfg.dims) * cfg.rank)
    fs, _ = _normalized_factors(draws, cfg.dims, cfg.rank)
    return np.ones(cfg.rank), fs


def _uniform(seed: int, n: int) -> np.ndarray:
    """n draws of SplitMix64(seed).next_double() (rng.hpp:31), via the counter identity."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def c3_tensor(cfg: Config = C3, dim: int = None, rank: int = None, sigma: float = 0.01):
    """Symmetric sum_r lambda_r v_r^{o3} + symmetric noise; returns (T, lambdas, V)."""
    dim = dim or cfg.dims[0]
    rank = rank or cfg.rank
    g = host_gaussian(cfg.seed, dim * rank)
    q, _ = np.linalg.qr(g.reshape((dim, rank), order="F"))
    lam = 1.0 + _uniform(cfg.seed ^ 0x6C616D, rank)
    t = densify(lam, [q, q, q])
    i, j, k = np.meshgrid(np.arange(dim), np.arange(dim), np.arange(dim), indexing="ij")
    mask = (i <= j) & (j <= k)
    n_sym = int(mask.sum())
    noise = host_gaussian(cfg.seed ^ 0x6E6F6973, n_sym) * sigma
    sym = np.zeros((dim, dim, dim))
    ii, jj, kk = i[mask], j[mask], k[mask]
    for p in ((ii, jj, kk), (ii, kk, jj), (jj, ii, kk), (jj, kk, ii), (kk, ii, jj), (kk, jj, ii)):
        sym[p] = noise
    return t + sym, lam, q


def c5_matrices(cfg: Config = C5, n: int = 512):
    g = host_gaussian(cfg.seed, 2 * n * n)
    return g[:n * n].reshape((n, n), order="F"), g[n * n:].reshape((n, n), order="F")


def composed_len(cfg: Config) -> int:
    return len(cfg.dims) * cfg.hash_len - len(cfg.dims) + 1


def algorithmic_bytes(cfg_key: str) -> int:
    """SURVEY.md §8(d) algorithmic bytes per launch (the roofline numerator)."""
    c = CONFIGS[cfg_key]
    jt = composed_len(c)
    if cfg_key == "c4":
        return int(np.prod(c.dims)) * 4 + c.sketch_count * sum(c.dims) * 5 + c.sketch_count * jt * 4
    if cfg_key == "c1":
        return int(np.prod(c.dims)) * 8 + c.sketch_count * sum(c.dims) * 5 + c.sketch_count * jt * 8
    if cfg_key == "c2":  # factors + weights + tables + output
        return 3 * 400 * c.rank * 8 + c.rank * 8 + c.sketch_count * sum(c.dims) * 5 + \
            c.sketch_count * jt * 8
    if cfg_key == "c5":  # two 512^2 fp64 operands + tables + output (4J - 3)
        return 2 * 512 * 512 * 8 + c.sketch_count * sum(c.dims) * 5 + c.sketch_count * jt * 8
    raise KeyError(cfg_key)


def c4_element_count() -> int:
    return int(math.prod(C4.dims))
