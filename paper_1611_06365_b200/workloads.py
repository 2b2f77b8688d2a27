"""Seeded synthetic inputs for the five BASELINE.json configs (frozen).

The reference measures on synthetic random matrices (matrix.py:44-59), so these
generators *are* the benchmark inputs, not a stand-in for a dataset.  Uniform configs use the
reference's own counter-based SplitMix64 stream (matrix.py:47-59): entry k = i + j*rows is drawn from
state seed + (k+1)*0x9E3779B97F4A7C15, mapped to (0,1) by ((z >> 11) + 1) / (2^53 + 2) and then to
(-1,1) by 2u-1.  Normal configs use numpy.random.default_rng(seed).standard_normal filled in
column-major order (one host source of truth, uploaded).

Host side only (numpy); the device twin of the uniform stream is the CUDA kernel behind
`paper_1611_06365_b200.fill_random`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


@dataclass(frozen=True)
class LuConfig:
    """One BASELINE.json config: order, generator, seed, outer/inner block widths."""

    name: str
    n: int
    dist: str          # "uniform" | "normal" | "uniform_rowscaled"
    seed: int
    b_outer: int
    b_inner: int


CONFIGS = {
    "config1": LuConfig("config1", 2048, "uniform", 0, 256, 32),
    "config2": LuConfig("config2", 8192, "normal", 1, 256, 32),
    "config3": LuConfig("config3", 16384, "uniform_rowscaled", 2, 512, 64),
    "config4": LuConfig("config4", 32768, "normal", 3, 512, 64),   # headline point of the b sweep {128,256,512,768}, b_i = b/8
    "config5": LuConfig("config5", 65536, "uniform", 4, 512, 64),
}


def splitmix64_uniform01(rows: int, cols: int, seed: int, col0: int = 0, ncols: int | None = None,
                         total_rows: int | None = None) -> np.ndarray:
    """Columns [col0, col0+ncols) of the rows x cols SplitMix64 fill, Fortran order, in (0,1).

    Bit-identical to the reference's fill_random (matrix.py:47-63) on the same seed; because the
    stream is counter-based any column block can be produced independently (used by the 1-D
    block-cyclic multi-GPU layout).
    """
    ncols = cols - col0 if ncols is None else ncols
    total_rows = rows if total_rows is None else total_rows
    out = np.empty((rows, ncols), dtype=np.float64, order="F")
    old = np.seterr(over="ignore")
    try:
        base = np.uint64(seed & (2 ** 64 - 1))
        i = np.arange(1, rows + 1, dtype=np.uint64)
        for jj in range(ncols):
            k0 = np.uint64(((col0 + jj) * total_rows) & (2 ** 64 - 1))
            z = base + (i + k0) * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
            out[:, jj] = ((z >> np.uint64(11)).astype(np.float64) + 1.0) / 9007199254740994.0
    finally:
        np.seterr(**old)
    return out


def row_scale_vector(n: int) -> np.ndarray:
    """config 3's exact float64 row scaling 10^(-6 i/n), computed once on the host."""
    return np.array([10.0 ** (-6.0 * i / n) for i in range(n)], dtype=np.float64)


def make_matrix(dist: str, n: int, seed: int, m: int | None = None) -> np.ndarray:
    """m x n (default square) Fortran-order float64 input of the named distribution."""
    m = n if m is None else m
    if dist == "uniform":
        a = splitmix64_uniform01(m, n, seed)
        a *= 2.0
        a -= 1.0
        return a
    if dist == "uniform_rowscaled":
        a = make_matrix("uniform", n, seed, m)
        a *= row_scale_vector(m)[:, None]
        return a
    if dist == "normal":
        rng = np.random.default_rng(seed)
        return rng.standard_normal(m * n).reshape((m, n), order="F")
    raise ValueError(f"unknown distribution {dist!r}")


def make_config_matrix(cfg: LuConfig | str, n: int | None = None) -> np.ndarray:
    cfg = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    return make_matrix(cfg.dist, cfg.n if n is None else n, cfg.seed)


def flops_lu(m: int, n: int) -> float:
    """Model flop count mn^2 - n^3/3 (reference costmodel.py:24-28)."""
    return (3 * m * n * n - n ** 3) / 3
