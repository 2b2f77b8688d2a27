"""Condense the raw-page CSVs that tools/profile_round.sh leaves in gpurun_out/ into
profiles/<round>_ncu_summary.txt (the handful of metrics DESIGN.md quotes).
usage: python tools/ncu_summarize.py r01"""
import csv, sys, os

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
KEEP = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes_read.sum.per_second",
        "dram__bytes_write.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"]
FILES = [("getrf_n16384", "k_getrf, n=16384 b=512/64 lu_et sm_pf 32 (same code path as the headline, 1/8 of the flops)"),
         ("gemm_16384_k256", "k_gemm, 16384 x 16384 x 256"),
         ("laswp_trsm", "k_laswp_apply / k_trsm (tools/dev_ops_time.py)"),
         ("panel", "k_panel (tools/dev_panel_time2.py)"),
         ("apply_panel", "k_apply_panel (multi-GPU driver's fused update step; tools/dev_dist_time.py 16384 512 lu_mb)"),
         ("gemm_deep", "k_gemm, 20480 x 20480 x 4096 -- the deep multiply of the host entry point's catch-up (tools/dev_gemm_one.py)")]
out = ["# ncu --set full --clock-control none summaries (tools/profile_round.sh, tools/ncu_summarize.py); one block per captured launch"]
for stem, title in FILES:
    path = f"gpurun_out/{R}_{stem}_raw.csv"
    if not os.path.exists(path):
        continue
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    out.append(f"==== {title} ====")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"-- {d.get('Kernel Name')}")
        for k in KEEP:
            if k in d:
                out.append(f"   {k} = {d[k]} {u.get(k, '')}")
open(f"profiles/{R}_ncu_summary.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out[:30]))
