#!/usr/bin/env python
"""Benchmark of the LU hot path (BASELINE.json metric: LU GFLOP/s = (2n^3/3) / time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config config4] [--n N] [--variant lu_et] [--b-outer B] [--b-inner b]

One "step" = one whole factorization of the config's synthetic matrix (seeded).
N=1 default workload: config4 (n=32768, N(0,1) seed 3) at b=512/64 -- the best point of config 4's block
sweep b in {128,256,512,768}, b_i = b/8, and the configuration the >= 60 % target is quoted on.  N>1:
config5 (n=65536, b=512/64, 1-D block-cyclic columns, NCCL panel broadcast, look-ahead + WS + ET per GPU).
Rank 0 prints ONE JSON line.  `value` is timed with CUDA events around the factorization only (inputs
resident in HBM, restored from a pristine device copy between steps, outside the timed region); `e2e` is
the mean of 5 timed calls of the C-ABI entry point with pinned host buffers (H2D + factor + D2H inside).
`--impl reference` times the CPU oracle port (oracle/, bit-identical to the reference package, which is
Python + numba and cannot travel to the GPU box) on all host cores: its `config` is this arm's, each step
is a BOUNDED SAMPLE of that workload (the leading n_s x n_s block of the same matrix, n_s chosen so the
run ends within a few minutes and printed as `sample_n`), next to a measured n-curve and the explicit
projection to the full size.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1611_06365_b200.workloads import CONFIGS, flops_lu, make_matrix  # noqa: E402

# DRAM bytes of ONE k_getrf launch on the default workload (n=32768, b=512/64, lu_et, sm_pf 32), from
# `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum` (profiles/r02_getrf_n32768_traffic.csv):
# 491.8 GB read + 231.0 GB written; the algorithmic minimum (the trailing matrix read and written once
# per iteration) is 2 * 8 * n^3 / (3 b) = 367 GB at b = 512 (ET cuts make the effective b smaller).
# It cannot be measured by the run that prints it (ncu replays the launch), hence the constant + its source.
DEFAULT_WORKLOAD_DRAM_BYTES = 491778257664 + 231039581696
DEFAULT_WORKLOAD_DRAM_SOURCE = ("profiles/r02_getrf_n32768_traffic.csv (ncu dram__bytes_read.sum + dram__bytes_write.sum of "
                                "the k_getrf launch of this same command, captured in a separate run under ncu)")

FP64_TENSOR_PEAK_TFLOPS = 37.0   # measured on this pool's B200: tools/fp64_peak.cu (DMMA.8x8x4
                                 # issue-bound, 3 s sustained) -> profiles/r01_fp64_peak.log.
                                 # MEASURED_PEAKS.json has no FP64 entry.


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--variant", default="lu_et")
    ap.add_argument("--b-outer", type=int, default=None)
    ap.add_argument("--b-inner", type=int, default=None)
    ap.add_argument("--sm-pf", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", action="store_true", help="also report the backward error")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.rows, self.proc, self.index = [], None, index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0])); mx = float(r[1])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = sorted(x for x in sm if mx is None or x > 0.3 * mx) or sorted(sm)
        med = busy[len(busy) // 2] if busy else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def phase_split(pool, res, n, b_o, flops):
    """Update-vs-panel split of the LAST factorization from the device trace (mla_getrf_trace) and the
    sampled update-team CTA (mla_getrf_debug): what BASELINE.json's config 4 asks for."""
    import ctypes
    from paper_1611_06365_b200 import _capi
    lib = _capi.lib()
    rows = max(0, len(res.widths) - 1)
    buf = (ctypes.c_uint64 * (5 * 1024))()
    got = lib.mla_getrf_trace(pool.handle, buf, 1024)
    t = np.array(buf[:5 * min(rows, got)], dtype=np.uint64).reshape(-1, 5).astype(np.int64)
    dbg = (ctypes.c_uint64 * 8)()
    lib.mla_getrf_debug(pool.handle, dbg)
    prof = (ctypes.c_uint64 * 16)()
    lib.mla_panel_profile(pool.handle, prof, 1)
    out = {}
    if len(t):
        ok = t[:, 3] > 0
        pq = (t[:, 1] - t[:, 0]).clip(min=0)
        panel = (t[:, 2] - t[:, 1]).clip(min=0)
        rq = np.where(ok, t[:, 3] - t[:, 0], 0).clip(min=0)
        nxt = np.append(t[1:, 0], max(t[-1, 2], t[-1, 3]))
        it = nxt - t[:, 0]
        bound_panel = int(np.sum((t[:, 2] > t[:, 3]) & ok))
        out.update({
            "iterations_traced": int(len(t)),
            "sum_iteration_ms": round(float(it.sum()) / 1e6, 2),
            "sum_update_queue_ms": round(float(rq.sum()) / 1e6, 2),
            "sum_panel_ms": round(float(panel.sum()) / 1e6, 2),
            "sum_panel_columns_update_ms": round(float(pq.sum()) / 1e6, 2),
            "iterations_panel_bound": bound_panel,
        })
    if dbg[6]:
        tile_us = dbg[0] / 1e3 / max(1, dbg[1])
        out["update_cta_sample"] = {
            "gemm_ms": round(dbg[0] / 1e6, 2), "tiles": int(dbg[1]), "us_per_tile": round(tile_us, 2),
            "prep_ms": round(dbg[2] / 1e6, 2), "left_swaps_ms": round(dbg[4] / 1e6, 2),
            "barrier_wait_ms": round(dbg[5] / 1e6, 2), "kernel_ms": round(dbg[6] / 1e6, 2)}
    out["panel_team_rank0_ms"] = {"gemm": round(prof[1] / 1e6, 2), "pivot_steps": round(prof[2] / 1e6, 2),
                                  "of_which_exchange": round(prof[5] / 1e6, 2),
                                  "swaps_and_u_rows": round(prof[3] / 1e6, 2), "barriers": round(prof[4] / 1e6, 2)}
    return out


def pick(args, world):
    name = args.config or ("config4" if world == 1 else "config5")
    cfg = CONFIGS[name]
    n = args.n or cfg.n
    default_b = cfg.b_outer
    if name == "config4" and args.b_outer is None:
        # config 4 is a block-size sweep b in {128, 256, 512, 768} with inner block b/8; the headline
        # line uses the best point of the sweep on B200 (profiles/r01_bench_config4_bsweep.json)
        default_b = 512
        if args.sm_pf is None:
            args.sm_pf = 32
    b_o = args.b_outer or default_b
    b_i = args.b_inner or (cfg.b_inner if b_o == cfg.b_outer else max(1, b_o // 8))
    return name, cfg, n, b_o, b_i


def workload_config(name, cfg, n, b_o, b_i, variant, sm_pf, world):
    """The `config` object of the JSON line -- identical for both arms (the reference arm times a bounded
    sample OF THIS workload and says so in `sample_n` / `cpu_baseline.sample`)."""
    c = {"workload": f"{name}: LU n={n} b={b_o}/{b_i} {cfg.dist} seed {cfg.seed}", "variant": variant,
         "l2": "inputs larger than L2 (8 B * n^2) and restored from a pristine copy between steps"}
    if world == 1:
        c["sm_pf"] = sm_pf
    else:
        c["layout"] = "1-D block-cyclic columns, NCCL panel+pivot broadcast, look-ahead+WS+ET per GPU"
    return c


_MATRIX_CACHE = {}


def cpu_oracle_run(cfg, n, b_o, b_i, threads=None):
    """Time the CPU oracle port (bit-identical to the reference) on the leading n x n block of cfg's
    generator family (same distribution and seed)."""
    import oracle
    if threads:
        oracle.set_num_threads(threads)
    key = (cfg.dist, cfg.seed, n)
    if key not in _MATRIX_CACHE:
        _MATRIX_CACHE.clear()
        _MATRIX_CACHE[key] = np.asfortranarray(make_matrix(cfg.dist, n, cfg.seed))
    a = _MATRIX_CACHE[key].copy(order="F")
    t0 = time.perf_counter()
    oracle.lu_la(a, b_o, b_i)
    dt = time.perf_counter() - t0
    return flops_lu(n, n) / dt / 1e9, dt, oracle.num_threads()


SAMPLE_SIZES = (16384, 12288, 8192, 6144, 4096, 3072, 2048)


def cpu_baseline(cfg, b_o, b_i, budget_s=15.0):
    """Bounded sample: probe at n=1536, then the largest n (<= 16384) whose predicted time fits the budget."""
    gf, dt, cores = cpu_oracle_run(cfg, 1536, b_o, b_i)
    n = 1536
    for cand in SAMPLE_SIZES:
        if flops_lu(cand, cand) / (gf * 1.5e9) <= budget_s:   # rate improves with n
            n = cand
            break
    if n > 1536:
        gf, dt, cores = cpu_oracle_run(cfg, n, b_o, b_i)
    return {"value": round(gf, 3), "unit": "GFLOP/s", "cores": cores, "kind": "port",
            "sample": f"oracle lu_la on the {cfg.dist} seed-{cfg.seed} matrix at n={n}, "
                      f"b={b_o}/{b_i}, {dt:.1f} s (bounded sample; the full n is projected, not run)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    name, cfg, n_full, b_o, b_i = pick(args, args.gpus)
    import oracle
    cores = oracle.num_threads()
    # measured n-curve (one run each): shows the CPU rate is flat in n, which is what the projection to
    # the full size rests on
    curve = {}
    for nn in (min(2048, n_full), min(4096, n_full)):
        gf, dt, _ = cpu_oracle_run(cfg, nn, b_o, b_i)
        curve[str(nn)] = {"gflops": round(gf, 2), "seconds": round(dt, 2)}
    gf = curve[str(min(4096, n_full))]["gflops"]
    # the bounded sample: the largest size whose K+W steps end within ~4 minutes at the measured rate
    total = max(1, args.steps + args.warmup)
    n = min(2048, n_full)
    for cand in SAMPLE_SIZES:
        if cand <= n_full and total * flops_lu(cand, cand) / (gf * 1e9) <= 240.0:
            n = cand
            break
    for _ in range(args.warmup):
        cpu_oracle_run(cfg, n, b_o, b_i)
    times = []
    for _ in range(args.steps):
        _, dt, _ = cpu_oracle_run(cfg, n, b_o, b_i)
        times.append(dt)
    dt = sum(times) / len(times)
    val = flops_lu(n, n) / dt / 1e9
    curve[str(n)] = {"gflops": round(val, 2), "seconds": round(dt, 2)}
    proj_s = flops_lu(n_full, n_full) / (val * 1e9)
    sample = (f"oracle port of the reference lu_la (bit-identical, tests/test_oracle_golden.py) on the "
              f"{cfg.dist} seed-{cfg.seed} matrix at n={n} (bounded sample of the n={n_full} workload), "
              f"b={b_o}/{b_i}, all {cores} host threads; projected full-size step at this rate: {proj_s:.0f} s")
    t_pf = 32 if args.sm_pf is None else args.sm_pf
    print(json.dumps({
        "impl": "reference", "metric": "LU GFLOP/s (2n^3/3 / time)", "value": round(val, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(name, cfg, n_full, b_o, b_i, args.variant, t_pf, args.gpus),
        "sample_n": n, "n_curve": curve,
        "projected_full_size": {"n": n_full, "seconds_per_step": round(proj_s, 1), "gflops": round(val, 3),
                                "basis": "GFLOP/s measured at sample_n; the n-curve shows the rate is flat in n"},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback); use --impl reference for the CPU arm")
    if args.gpus != world:
        raise SystemExit(f"bench.py --gpus {args.gpus} must be launched with torchrun --nproc-per-node {args.gpus} "
                         f"(WORLD_SIZE is {world}); one process per GPU")
    if torch.cuda.device_count() < world:
        raise SystemExit(f"bench.py --gpus {world}: only {torch.cuda.device_count()} CUDA device(s) visible on this node")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1611_06365_b200 as mla
    name, cfg, n, b_o, b_i = pick(args, world)
    dev = torch.device("cuda", local)
    pool = mla.default_pool(local)
    policy = mla.Policy(args.variant, mla.BlockConfig(b_o, b_i), t_pf=args.sm_pf)
    flops = flops_lu(n, n)
    sampler = ClockSampler(local)

    if world > 1:
        from paper_1611_06365_b200.distributed import DistLU
        dlu = DistLU(n, b_o, b_i, cfg, dev, variant=args.variant if args.variant in DistLU.VARIANTS else "lu_et", pool=pool)
        dlu.generate()
        for _ in range(args.warmup):
            dlu.restore(); dlu.factor()
        times = []
        torch.cuda.synchronize(); dist.barrier()
        if rank == 0:
            sampler.start()
        for _ in range(args.steps):
            dlu.restore()
            torch.cuda.synchronize(); dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); dlu.factor(); e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1)], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            times.append(float(t.item()))
        clocks = sampler.stop() if rank == 0 else None
        ms = sum(times) / len(times)
        # end to end: every rank uploads its column blocks from pinned host memory, the factorization
        # runs, the packed factors come back to the host
        e2e = None
        if not args.no_e2e and dlu.nloc:
            host0 = torch.empty((dlu.nloc, n), dtype=torch.float64).pin_memory()
            host0.copy_(dlu.a0.t())
            back = torch.empty_like(host0).pin_memory()
            torch.cuda.synchronize(); dist.barrier()
            t0 = time.perf_counter()
            dlu.a.t().copy_(host0, non_blocking=True)
            dlu.factor()
            back.copy_(dlu.a.t(), non_blocking=True)
            torch.cuda.synchronize()
            t = torch.tensor([time.perf_counter() - t0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e = float(t.item())
            e2e = {"value": round(flops / e / 1e9, 1), "unit": "GFLOP/s",
                   "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 8 * n * n + 4 * n,
                   "ms_per_step": round(e * 1e3, 2), "api": "DistLU.factor with pinned host blocks per rank"}
        if rank == 0:
            val = flops / (ms * 1e-3) / 1e9
            print(json.dumps({
                "metric": "LU GFLOP/s (2n^3/3 / time)", "value": round(val, 1), "unit": "GFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(name, cfg, n, b_o, b_i, args.variant, None, world),
                "run": {"panels": len(dlu.widths), "et_events": dlu.et_events, "host_waits": dlu.host_waits},
                "roofline": {"bound": "tensor", "achieved": round(val / 1e3, 3), "peak": FP64_TENSOR_PEAK_TFLOPS * world,
                             "unit": "TFLOP/s", "frac": round(val / 1e3 / (FP64_TENSOR_PEAK_TFLOPS * world), 4),
                             "traffic": None, "peak_source": "measured DMMA issue rate x n_gpus (tools/fp64_peak.cu)"},
                "e2e": e2e, "gpu_launches": dlu.launches_per_factor * args.steps, "clocks": clocks,
            }), flush=True)
        dist.destroy_process_group()
        return

    # ---- single GPU ----------------------------------------------------------------------------
    t_gen = time.perf_counter()
    if cfg.dist == "normal":
        host = make_matrix(cfg.dist, n, cfg.seed)
        a0 = mla.from_numpy(host, device=dev)
    else:
        host = None
        a0 = mla.alloc_matrix(n, n, device=dev)
        rs = None
        if cfg.dist == "uniform_rowscaled":
            from paper_1611_06365_b200.workloads import row_scale_vector
            rs = torch.from_numpy(row_scale_vector(n)).to(dev)
        mla.fill_random(a0, cfg.seed, 2.0, -1.0, row_scale=rs, pool=pool)
    a = mla.alloc_matrix(n, n, device=dev)
    gen_s = time.perf_counter() - t_gen
    res = None
    def factor(x):
        return mla.lu_la(x, policy, pool)
    for _ in range(args.warmup):
        a.copy_(a0)
        res = factor(a)
    torch.cuda.synchronize()
    sampler.start()
    times = []
    for step in range(args.steps):
        a.copy_(a0)            # restore (outside the timed region; also evicts L2: 8 GiB >> 126 MB)
        torch.cuda.synchronize()
        if step == args.steps - 1:   # the phase split below describes the last step only
            import ctypes
            from paper_1611_06365_b200 import _capi
            _capi.lib().mla_panel_profile(pool.handle, (ctypes.c_uint64 * 16)(), 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = factor(a)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    clocks = sampler.stop()
    ms = sum(times) / len(times)
    val = flops / (ms * 1e-3) / 1e9

    phases = phase_split(pool, res, n, b_o, flops)
    residual = None
    if args.check:
        chk = mla.alloc_matrix(n, n, device=dev)
        chk.copy_(a0)
        residual = mla.residual_packed(chk, a, res.ipiv) / (n * np.finfo(np.float64).eps)
        del chk

    e2e = None
    if not args.no_e2e:
        import ctypes
        from paper_1611_06365_b200 import _capi
        del a
        if host is None:
            host = mla.to_numpy(a0)
        host_t = torch.from_numpy(np.ascontiguousarray(host.T)).pin_memory()   # (n, n) rows = columns
        work = torch.empty_like(host_t).pin_memory()
        ipiv_h = torch.empty(n, dtype=torch.int32).pin_memory()
        info = _capi.LuInfo()
        t_pf = pool.t_pf if args.sm_pf is None else args.sm_pf
        e_times = []
        for i in range(6):                 # one warm-up call (allocates the cached device buffers) + 5 timed
            work.copy_(host_t)
            t0 = time.perf_counter()
            rc = _capi.lib().mla_getrf_la_host(pool.handle, work.data_ptr(), n, n, n, ipiv_h.data_ptr(), b_o, b_i,
                                               _capi.VARIANT_CODES[args.variant], t_pf, 4, ctypes.byref(info))
            dt = time.perf_counter() - t0
            _capi.check(rc, pool.handle, "mla_getrf_la_host")
            if i > 0:
                e_times.append(dt)
        e = sum(e_times) / len(e_times)
        e2e = {"value": round(flops / e / 1e9, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * n * n,
               "d2h_bytes_per_step": 8 * n * n + 4 * n, "ms_per_step": round(e * 1e3, 2), "timed_calls": len(e_times),
               "ms_min_max": [round(min(e_times) * 1e3, 2), round(max(e_times) * 1e3, 2)],
               "api": "mla_getrf_la_host (C ABI, pinned host buffers; chunked upload, windows n/32 n/8 3n/8 factored "
                      "behind it, finished rows streamed out under the last window)"}

    cpu = None if args.no_cpu else cpu_baseline(cfg, b_o, b_i)
    out = {
        "metric": "LU GFLOP/s (2n^3/3 / time)", "value": round(val, 1), "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(name, cfg, n, b_o, b_i, args.variant, pool.t_pf if args.sm_pf is None else args.sm_pf, 1),
        "run": {"et_events": res.et_events, "ws_joins": res.ws_joins, "panels": len(res.widths),
                "gen_seconds": round(gen_s, 1)},
        "roofline": {"bound": "tensor", "achieved": round(val / 1e3, 3), "peak": FP64_TENSOR_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": round(val / 1e3 / FP64_TENSOR_PEAK_TFLOPS, 4),
                     "traffic": DEFAULT_WORKLOAD_DRAM_BYTES if (name == "config4" and n == 32768 and b_o == 512
                                                                and args.variant == "lu_et") else None,
                     "traffic_source": DEFAULT_WORKLOAD_DRAM_SOURCE,
                     "kernel": "k_getrf (persistent; algorithmic flops 2n^3/3 per launch)",
                     "peak_source": "measured: DMMA.8x8x4 issue-bound rate, tools/fp64_peak.cu, "
                                    "profiles/r01_fp64_peak.log (MEASURED_PEAKS.json has no FP64 entry)"},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": args.steps, "clocks": clocks,
        "phases": phases,
    }
    if residual is not None:
        out["backward_error_over_n_eps"] = round(float(residual), 4)
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
