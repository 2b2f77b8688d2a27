"""Blocking and scheduling parameters -- same types as the reference (config.py:12-84).

CacheConfig (CPU cache geometry, reference config.py:23-54) is accepted everywhere the reference
accepts it and ignored: GPU tile shapes are compile-time constants of the kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

VARIANTS = ("lu", "lu_la", "lu_ws_static", "lu_mb", "lu_et")


@dataclass(frozen=True)
class CacheConfig:
    """Accepted for signature compatibility; has no effect on the GPU path."""

    m_c: int = 256
    k_c: int = 256
    n_c: int = 4096
    m_r: int = 8
    n_r: int = 4

    @classmethod
    def from_env(cls, env=None, **overrides):
        return cls(**overrides)


@dataclass(frozen=True)
class BlockConfig:
    """Outer (panel) and inner (panel-of-panel) block widths (reference config.py:57-66)."""

    b_outer: int
    b_inner: int

    def __post_init__(self) -> None:
        if not 1 <= self.b_inner <= self.b_outer:
            raise ValueError("need 1 <= b_inner <= b_outer")


@dataclass(frozen=True)
class Policy:
    """Which variant runs and how the SMs are split (reference config.py:69-84).

    t_pf keeps its meaning "size of the panel team"; on the GPU the unit is SMs (CTAs of the
    persistent kernel) instead of threads.  t_pf=None lets the pool pick its default.
    """

    variant: str
    b: BlockConfig
    t_pf: int | None = None
    q: int = 4

    def __post_init__(self) -> None:
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}, expected one of {VARIANTS}")
        if self.t_pf is not None and self.t_pf < 1:
            raise ValueError("t_pf must be >= 1")
        if self.q < 1:
            raise ValueError("q must be >= 1")
