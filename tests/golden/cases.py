"""Golden-vector case list shared by make_golden.py (runs the REFERENCE) and the tests (run the
oracle / the CUDA path).  Inputs are functions of (shape, seed) only, so only outputs are stored."""
from __future__ import annotations

import numpy as np

# tiny cache config used with the reference to cross every k_c slicing edge on small matrices
# (same idea as the reference's TINY config, test_kernels.py:16); only k_c influences bits.
TINY_KC = 8

UNB = [dict(name="unb_20x20", m=20, n=20, seed=11), dict(name="unb_37x13", m=37, n=13, seed=12)]

LL = [dict(name="ll_64x48_b8", m=64, n=48, b=8, seed=13, stop_trip=0, k_c=256),
      dict(name="ll_64x48_b8_preset", m=64, n=48, b=8, seed=13, stop_trip=1, k_c=256),
      dict(name="ll_64x48_b8_trip3", m=64, n=48, b=8, seed=13, stop_trip=3, k_c=256),
      dict(name="ll_200x96_b32_kc8", m=200, n=96, b=32, seed=17, stop_trip=0, k_c=TINY_KC)]

RL = [dict(name="rl_60_b16", m=60, n=60, b=16, inner_b=None, seed=14),
      dict(name="rl_60_b16_i4", m=60, n=60, b=16, inner_b=4, seed=14),
      dict(name="rl_200x96_b32", m=200, n=96, b=32, inner_b=None, seed=17)]

LA = [dict(name="la_100_16_4", m=100, n=100, b_o=16, b_i=4, seed=15, k_c=256, variant="lu"),
      dict(name="la_90x70_32_8", m=90, n=70, b_o=32, b_i=8, seed=16, k_c=256, variant="lu_la"),
      dict(name="la_160_64_16_kc8", m=160, n=160, b_o=64, b_i=16, seed=18, k_c=TINY_KC, variant="lu_mb"),
      dict(name="la_97_32_32", m=97, n=97, b_o=32, b_i=32, seed=19, k_c=256, variant="lu")]

# ET replay: per-iteration trip poll (0 = no cut); injected deterministically into the reference
LA_ET = [dict(name="et_256_64_8", m=256, n=256, b_o=64, b_i=8, seed=21, k_c=256,
              sched=[2, 0, 1, 0, 0, 3, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0]),
         dict(name="et_200x150_32_8", m=200, n=150, b_o=32, b_i=8, seed=22, k_c=TINY_KC,
              sched=[1, 1, 1, 0, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0])]

GEMM = [dict(name="gemm_37x29x21", m=37, n=29, k=21, alpha=0.5, beta=-2.0, seed=31, k_c=TINY_KC),
        dict(name="gemm_130x70x300", m=130, n=70, k=300, alpha=1.0, beta=-1.0, seed=32, k_c=256)]

TRSM = [dict(name="trsm_24x17", w=24, c=17, seed=41)]

LASWP = [dict(name="laswp_30x9", rows=30, cols=9, seed=51,
              ipiv=[3, 1, 29, 3, 10, 5, 6, 29, 8, 12])]

# config-shaped cases: output stored as pivots + sha256 of the packed factors
BIG = [dict(name="config1_2048", dist="uniform", n=2048, seed=0, b_o=256, b_i=32),
       dict(name="config3_1024", dist="uniform_rowscaled", n=1024, seed=2, b_o=512, b_i=64),
       dict(name="config2_1536", dist="normal", n=1536, seed=1, b_o=256, b_i=32)]


def uniform_pm1(fill_random, m, n, seed, ld=None):
    """2u-1 on a fresh column-major array via the supplied fill_random(a, seed)."""
    ld = m if ld is None else ld
    a = np.zeros((max(ld, 1), n), dtype=np.float64, order="F")[:m, :]
    fill_random(a, seed)
    a *= 2.0
    a -= 1.0
    return a
