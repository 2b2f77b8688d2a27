"""Second oracle for the sizes the pinned C oracle cannot reach: LAPACK getrf through
scipy.linalg.lu_factor.  getrf uses the same pivot rule as the reference (largest |entry| of the
column, first occurrence; lu.py:48-55) and returns the same LAPACK-style sequential interchanges
(lu.py:236, 317), so on matrices without exact ties its pivot vector must equal the reference's; the
factors agree up to rounding (different summation order, FMA).

    python tests/golden/make_golden_lapack.py config5          # n = 65536: ~32 GiB, ~30 min on 8 cores
    python tests/golden/make_golden_lapack.py config2 --check  # compare with the pinned-oracle fixture

What pins LAPACK to the reference before its output is trusted:
  * tests/test_oracle_golden.py::test_lapack_pivots_equal_the_pinned_oracle (CPU suite, config-1/2/3
    shaped inputs: pivots identical, factors within 1e-10 column-scaled);
  * --check: at the FULL sizes of configs 2, 3 and 4 the pivots must equal the fixtures that the pinned
    oracle produced (golden_config{2,3,4}.npz) -- run once when this fixture was made, result recorded
    in the fixture's `pinned_by` field.

Stored for config 5: int32 pivots, diag(U), every column's max |entry|, SAMPLE_K rows and SAMPLE_K
columns of the packed factors (check (b) on the GPU at a size where no full reference run exists).
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np
import scipy.linalg

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1611_06365_b200.workloads import CONFIGS, make_config_matrix  # noqa: E402
from make_golden_big import sample_indices  # noqa: E402


def lapack_lu(a: np.ndarray):
    """In-place getrf on a Fortran-ordered array -> (packed factors (same memory), 0-based pivots)."""
    assert a.flags.f_contiguous
    lu, piv = scipy.linalg.lu_factor(a, overwrite_a=True, check_finite=False)
    return lu, piv.astype(np.int64)


def main():
    name = sys.argv[1]
    cfg = CONFIGS[name]
    t0 = time.perf_counter()
    a = make_config_matrix(cfg)
    print(name, "generated", round(time.perf_counter() - t0, 1), "s", flush=True)
    t0 = time.perf_counter()
    lu, piv = lapack_lu(a)
    print(name, "getrf", round(time.perf_counter() - t0, 1), "s", flush=True)
    if "--check" in sys.argv:
        g = np.load(os.path.join(HERE, f"golden_{name}.npz"))
        same = np.array_equal(piv, g["ipiv"].astype(np.int64))
        d = np.abs(np.diag(lu) - g["diag"]).max() / np.abs(g["diag"]).max()
        print(f"{name}: LAPACK pivots == pinned-oracle pivots: {same}; diag(U) rel diff {d:.2e}")
        sys.exit(0 if same else 1)
    idx = sample_indices(cfg.n, 4 if cfg.n > 40000 else 8)
    colmax = np.empty(cfg.n)
    for j0 in range(0, cfg.n, 1024):                       # blockwise: no n x n temporary
        colmax[j0:j0 + 1024] = np.abs(lu[:, j0:j0 + 1024]).max(axis=0)
    np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"),
                        ipiv=piv.astype(np.int32), diag=np.array(np.diag(lu)), b_outer=cfg.b_outer,
                        b_inner=cfg.b_inner, sample_idx=idx, sample_rows=np.ascontiguousarray(lu[idx, :]),
                        sample_cols=np.ascontiguousarray(lu[:, idx]), colmax=colmax,
                        pinned_by=np.array(["lapack getrf (scipy %s); pivots == pinned oracle at configs 2, 3, 4 "
                                            "full size (make_golden_lapack.py --check)" % scipy.__version__]))
    print("wrote", name)


if __name__ == "__main__":
    main()
