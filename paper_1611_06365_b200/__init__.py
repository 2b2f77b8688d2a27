"""paper_1611_06365_b200 -- B200-native drop-in for the LU hot path of the reference package `mla`
(arXiv 1611.06365): blocked right-looking LU with partial pivoting, look-ahead, worker sharing and
early termination, as one persistent sm_100a kernel behind the reference's Python entry points.

Names kept from the reference (pkg/src/mla/__init__.py:6-33): lu_la, lu_blk_ll, lu_blk_rl, lu_unb,
trsm_llu, gemm_malleable, laswp, LuResult, PivotVector, Policy, BlockConfig (+ the matrix helpers).
"""
from .config import VARIANTS, BlockConfig, CacheConfig, Policy
from .costmodel import (cumulative_flop_share, flops_ll_partial, flops_panel_total, flops_rl_partial,
                        iteration_flops, schedule_flops)
from .kernels import gemm_malleable, laswp, trsm_llu
from .lu import (CountingStop, LuResult, et_schedule_from, et_widths_from, lu_blk_ll, lu_blk_rl,
                 lu_la, lu_unb)
from .matrix import (PivotVector, alloc_matrix, fill_random, frobenius_norm, from_numpy,
                     leading_dimension, partition_2x2, residual_lu, residual_packed, split_lu,
                     swap_rows, to_numpy)
from .pool import CompletionFlag, SmPool, WorkerPool, default_pool, signal_complete
from .trace import TraceEvent, check_trace, load_jsonl
from .workloads import CONFIGS, LuConfig, flops_lu, make_config_matrix, make_matrix

__version__ = "0.1.0"

__all__ = [
    "BlockConfig", "CacheConfig", "CompletionFlag", "CONFIGS", "CountingStop", "LuConfig", "LuResult",
    "PivotVector", "Policy", "SmPool", "TraceEvent", "VARIANTS", "WorkerPool", "check_trace", "load_jsonl", "alloc_matrix", "default_pool",
    "et_schedule_from", "et_widths_from", "fill_random", "flops_lu", "frobenius_norm", "from_numpy",
    "gemm_malleable", "laswp", "leading_dimension", "lu_blk_ll", "lu_blk_rl", "lu_la", "lu_unb",
    "make_config_matrix", "make_matrix", "partition_2x2", "residual_lu", "residual_packed",
    "cumulative_flop_share", "flops_ll_partial", "flops_panel_total", "flops_rl_partial",
    "iteration_flops", "schedule_flops", "signal_complete", "split_lu", "swap_rows", "to_numpy", "trsm_llu",
]
