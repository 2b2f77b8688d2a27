"""`mla-bench` for the GPU path: same flags and CSV columns as the reference CLI (bench.py:33-200).

    python -m paper_1611_06365_b200.bench_cli --algo lu_et --n 8192 --b-outer 256 --b-inner 32 --check

One CSV record per run on stdout: variant,n,b_outer,b_inner,threads,t_pf,seed,wall_seconds,gflops,
residual,et_events.  `threads` reports the SM count of the pool, `--t-pf` is the panel team's SM count.
GFLOPS uses the model count 2n^3/3 regardless of variant; the clock covers the factorization call only
(generation, warm-up and checking excluded; bench.py:3-9).  Inputs are the reference's own (0,1)
SplitMix64 fill (matrix.py:44-63), produced on the device.  --gepp sweeps k for C += A*B with m = n.
"""
from __future__ import annotations

import argparse
import csv
import sys
import time

import numpy as np

CSV_FIELDS = ("variant", "n", "b_outer", "b_inner", "threads", "t_pf", "seed", "wall_seconds", "gflops",
              "residual", "et_events")
RESIDUAL_TOL_FACTOR = 100.0
VARIANTS = ("lu", "lu_la", "lu_ws_static", "lu_mb", "lu_et")


def _span(text: str) -> list[int]:
    parts = text.split(":")
    if len(parts) != 3:
        raise argparse.ArgumentTypeError("expected lo:hi:step")
    try:
        lo, hi, step = (int(p) for p in parts)
    except ValueError:
        raise argparse.ArgumentTypeError("expected lo:hi:step") from None
    if lo < 1 or hi < lo or step < 1:
        raise argparse.ArgumentTypeError("need 1 <= lo <= hi and step >= 1")
    return list(range(lo, hi + 1, step))


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="mla-bench-b200",
                                 description="Time LU variants on a B200 (CSV to stdout) or the gepp curve.")
    ap.add_argument("--algo", choices=VARIANTS, default="lu")
    ap.add_argument("--n", type=int, help="matrix order (required unless --sweep-n)")
    ap.add_argument("--b-outer", type=int, default=256)
    ap.add_argument("--b-inner", type=int, default=32)
    ap.add_argument("--threads", type=int, help="accepted for compatibility; the pool is the GPU's SMs")
    ap.add_argument("--t-pf", type=int, default=16, help="SMs of the panel team")
    ap.add_argument("--q", type=int, default=4)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--trace", metavar="PATH", help="write the device trace as reference-schema JSON lines")
    ap.add_argument("--sweep-b", type=_span, metavar="lo:hi:step")
    ap.add_argument("--sweep-n", type=_span, metavar="lo:hi:step")
    ap.add_argument("--gepp", action="store_true")
    return ap


def validate(ap, args) -> None:
    """Same exit-code-2 rules as the reference (bench.py:168-183)."""
    if args.n is None and not args.sweep_n:
        ap.error("--n is required unless --sweep-n is given")
    if args.gepp and args.n is None:
        ap.error("--gepp needs --n")
    if args.b_inner < 1 or args.b_outer < 1:
        ap.error("block sizes must be >= 1")
    if args.b_inner > args.b_outer:
        ap.error("need b_inner <= b_outer")
    if args.t_pf < 1:
        ap.error("need t_pf >= 1")


def run_factorizations(args, writer) -> int:
    import torch
    import paper_1611_06365_b200 as mla
    from paper_1611_06365_b200 import trace as mtrace
    pool = mla.default_pool()
    if args.trace:
        mtrace.enable(pool)
    ns = args.sweep_n if args.sweep_n else [args.n]
    bs = args.sweep_b if args.sweep_b else [args.b_outer]
    eps = float(np.finfo(np.float64).eps)
    worst = 0
    warm = mla.alloc_matrix(96, 96)
    mla.fill_random(warm, 7)
    mla.lu_la(warm, mla.Policy(args.algo, mla.BlockConfig(32, 16), t_pf=min(args.t_pf, pool.t - 1), q=args.q), pool)
    first = True
    for n in ns:
        for b_outer in bs:
            b_inner = min(args.b_inner, b_outer)
            policy = mla.Policy(args.algo, mla.BlockConfig(b_outer, b_inner), t_pf=min(args.t_pf, pool.t - 1), q=args.q)
            a = mla.alloc_matrix(n, n)
            mla.fill_random(a, args.seed)
            a0 = a.clone() if args.check else None
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            result = mla.lu_la(a, policy, pool)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            if args.trace:
                evs = mtrace.events(pool)
                mtrace.write_jsonl(evs, args.trace, append=not first)
                first = False
            residual = None
            if args.check:
                residual = mla.residual_packed(a0, a, result.ipiv)
                if not residual <= n * RESIDUAL_TOL_FACTOR * eps:
                    worst = 1
            writer.writerow([args.algo, n, b_outer, b_inner, pool.t, policy.t_pf, args.seed, f"{wall:.6f}",
                             f"{mla.flops_lu(n, n) / wall / 1e9:.4f}",
                             "" if residual is None else f"{residual:.17g}", result.et_events])
            sys.stdout.flush()
    if args.trace:
        mtrace.enable(pool, False)
    return worst


def run_gepp(args, writer) -> int:
    import torch
    import paper_1611_06365_b200 as mla
    n = args.n
    ks = args.sweep_b if args.sweep_b else list(range(16, 257, 16))
    a, b, c = mla.alloc_matrix(n, max(ks)), mla.alloc_matrix(max(ks), n), mla.alloc_matrix(n, n)
    mla.fill_random(a, args.seed)
    mla.fill_random(b, args.seed + 1)
    mla.fill_random(c, args.seed + 2)
    mla.gemm_malleable(c, a[:, :min(8, max(ks))], b[:min(8, max(ks)), :], 1.0, 1.0)
    torch.cuda.synchronize()
    for k in ks:
        t0 = time.perf_counter()
        mla.gemm_malleable(c, a[:, :k], b[:k, :], 1.0, 1.0)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        writer.writerow([str(k), f"{2.0 * n * n * k / wall / 1e9:.4f}"])
        sys.stdout.flush()
    return 0


def main(argv=None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)
    validate(ap, args)
    writer = csv.writer(sys.stdout, lineterminator="\n")
    if args.gepp:
        writer.writerow(["k", "gflops"])
        return run_gepp(args, writer)
    writer.writerow(list(CSV_FIELDS))
    return run_factorizations(args, writer)


if __name__ == "__main__":
    sys.exit(main())
