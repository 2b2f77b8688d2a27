"""Flop model of the blocked LU (reference costmodel.py:1-94).

Host-side arithmetic only; bench.py's per-phase split and the trace report use it to turn device
times into GFLOP/s per operator.  Per outer iteration on an h x (w + c) trailing matrix
(h rows at and below the panel, w panel columns, c columns to its right):

    panel  h*w^2 - w^3/3        trsm  w^2*c        gemm  2*(h-w)*c*w

which telescopes to flops_lu(m, n) = m*n^2 - n^3/3 (costmodel.py:24-28).
"""
from __future__ import annotations

from .workloads import flops_lu

__all__ = ["flops_lu", "flops_panel_total", "flops_ll_partial", "flops_rl_partial",
           "iteration_flops", "schedule_flops", "cumulative_flop_share"]


def flops_panel_total(n, b) -> float:
    """All panel factorizations of an n x n LU with block b: n^2*b/2 (costmodel.py:31-33)."""
    return float(n) * float(n) * float(b) / 2


def _check_k(n, k):
    if k > n:
        raise ValueError("k must be <= n")


def flops_ll_partial(m, n, k) -> float:
    """Left-looking factorization cut at column k, published form m^2*k - m^3/3 (costmodel.py:36-40)."""
    _check_k(n, k)
    m, k = float(m), float(k)
    return m * m * k - m ** 3 / 3


def flops_rl_partial(m, n, k) -> float:
    """Right-looking cut at column k: the LL count + the updates already pushed to the right,
    2*(n-k)*(m*k - k^2/2) (costmodel.py:43-48)."""
    _check_k(n, k)
    m, n, k = float(m), float(n), float(k)
    return flops_ll_partial(m, n, k) + 2 * (n - k) * (m * k - k * k / 2)


def schedule_flops(m: int, n: int, widths) -> list[dict[str, float]]:
    """Per-iteration operator flops for an arbitrary panel-width schedule (e.g. LuResult.widths of an
    early-termination run).  Same record keys as iteration_flops."""
    if m < n:
        raise ValueError("need m >= n")
    rows, j = [], 0
    for w in widths:
        w = int(w)
        if w < 1 or j + w > n:
            raise ValueError("widths must be positive and sum to at most n")
        h, c = m - j, n - j - w
        rec = {"panel": float(h * w * w - w ** 3 / 3), "trsm": float(w * w * c),
               "gemm": float(2 * (h - w) * c * w)}
        rec["total"] = float(h * w * w - w ** 3 / 3 + w * w * c + 2 * (h - w) * c * w)
        rows.append(rec)
        j += w
    return rows


def iteration_flops(m: int, n: int, b: int) -> list[dict[str, float]]:
    """Panel / trsm / gemm flops of each outer iteration of a fixed-width schedule (costmodel.py:51-69)."""
    if m < n:
        raise ValueError("need m >= n")
    if b < 1:
        raise ValueError("block size must be >= 1")
    full, rest = divmod(n, b)
    return schedule_flops(m, n, [b] * full + ([rest] if rest else []))


def cumulative_flop_share(n: int, b: int, fraction: float) -> float:
    """Share of the flops spent on the first fraction*n columns; the iteration that straddles the cut
    counts pro rata, so the share is continuous in `fraction` (costmodel.py:72-94)."""
    if not 0 <= fraction <= 1:
        raise ValueError("fraction must be in [0, 1]")
    recs = iteration_flops(n, n, b)
    cut, head, total = n * fraction, 0.0, 0.0
    for i, r in enumerate(recs):
        j0 = i * b
        w = min(b, n - j0)
        total += r["total"]
        covered = min(max(cut - j0, 0.0), w)
        head += r["total"] if covered >= w else covered / w * r["total"]
    return head / total if total else 0.0
