"""Pivot fixtures for the full-size configs (BASELINE.json configs 2-4).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_big.py config2 [--reference]

Produced with the C oracle (bit-pinned to the reference by tests/test_oracle_golden.py); with
--reference the unmodified reference also runs (n <= 8192 is practical: ~2 min) and the two packed
factor arrays are required to be bitwise identical before anything is written.  Stored per config:
int32 pivots, sha256 of the packed factors, the diagonal of U and -- for check (b) of north_star at
sizes where the GPU test cannot afford a full oracle run -- SAMPLE_K full rows and SAMPLE_K full columns
of the packed factors together with every column's max |entry| (the scale of the 1e-10 bound).
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_1611_06365_b200.workloads import CONFIGS, make_config_matrix  # noqa: E402


SAMPLE_K = 8


def sample_indices(n: int, k: int = SAMPLE_K) -> np.ndarray:
    """k row/column indices spread over [0, n): both ends, and interior points that are NOT multiples of
    the block sizes (odd offsets), so panel interiors, panel edges and the last rows are all hit."""
    base = np.linspace(0, n - 1, k).astype(np.int64)
    base[1:-1] += 37
    return np.unique(np.clip(base, 0, n - 1))


def main():
    name = sys.argv[1]
    cfg = CONFIGS[name]
    a = np.asfortranarray(make_config_matrix(cfg))
    t0 = time.perf_counter()
    if "--reference" in sys.argv:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
        sys.path.insert(0, "/root/reference/pkg/src")
        from mla import BlockConfig, Policy, WorkerPool, lu_la
        b = a.copy(order="F")
        with WorkerPool(8) as pool:
            rr = lu_la(b, Policy("lu", BlockConfig(cfg.b_outer, cfg.b_inner)), pool)
        print("reference done", time.perf_counter() - t0)
    r = oracle.lu_la(a, cfg.b_outer, cfg.b_inner)
    print(name, "oracle seconds", time.perf_counter() - t0)
    if "--reference" in sys.argv:
        assert np.array_equal(rr.ipiv.ipiv, r.ipiv), "oracle pivots differ from the reference"
        assert np.array_equal(a, b), "oracle factors differ from the reference"
        print("oracle == reference bitwise at n =", cfg.n)
    sha = hashlib.sha256(a.tobytes(order="F")).digest()
    idx = sample_indices(cfg.n)
    np.savez_compressed(os.path.join(HERE, f"golden_{name}.npz"),
                        ipiv=r.ipiv.astype(np.int32), sha=np.frombuffer(sha, dtype=np.uint8),
                        diag=np.array(np.diag(a)), b_outer=cfg.b_outer, b_inner=cfg.b_inner,
                        sample_idx=idx, sample_rows=np.ascontiguousarray(a[idx, :]),
                        sample_cols=np.ascontiguousarray(a[:, idx]), colmax=np.abs(a).max(axis=0),
                        pinned_by=np.array(["reference+oracle" if "--reference" in sys.argv else "oracle"]))
    print("wrote", name)


if __name__ == "__main__":
    main()
