"""CPU-only checks: host-side logic, workload generators, and that the C-ABI library loads and
exports every symbol include/mla_b200.h declares (no compute calls without a GPU)."""
import os
import re
import sys

import numpy as np
import pytest

import oracle
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200 import _capi
from paper_1611_06365_b200.workloads import (CONFIGS, make_matrix, row_scale_vector,
                                             splitmix64_uniform01)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    import __graft_entry__
    __graft_entry__.build()
    hdr = open(os.path.join(ROOT, "include", "mla_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = set(re.findall(r"\b(mla_[a-z0-9_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = _capi.lib()
    for name in sorted(declared):
        assert getattr(lib, name) is not None, name
    assert declared == set(_capi.EXPORTS), (declared ^ set(_capi.EXPORTS))
    assert b"sm_100a" in lib.mla_version()


def test_sass_is_blackwell_fp64_tensor_path():
    """The shipped library carries sm_100a SASS with DMMA (FP64 tensor) and LDGSTS (cp.async)."""
    import shutil
    import subprocess
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA.8x8x4" in out and "LDGSTS" in out
    assert "STG.E.128.STRONG.GPU" in out  # fence-free tagged exchange words of the panel


def test_policy_validation_matches_reference():  # reference config.py:57-84, test_config.py
    with pytest.raises(ValueError):
        mla.BlockConfig(16, 32)
    with pytest.raises(ValueError):
        mla.BlockConfig(16, 0)
    with pytest.raises(ValueError):
        mla.Policy("lu_xx", mla.BlockConfig(32, 8))
    with pytest.raises(ValueError):
        mla.Policy("lu", mla.BlockConfig(32, 8), t_pf=0)
    with pytest.raises(ValueError):
        mla.Policy("lu", mla.BlockConfig(32, 8), q=0)
    assert mla.VARIANTS == ("lu", "lu_la", "lu_ws_static", "lu_mb", "lu_et")


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        mla.SmPool()
    with pytest.raises(ValueError):
        mla.lu_la(torch.zeros(4, 4, dtype=torch.float64).t(), mla.Policy("lu", mla.BlockConfig(2, 1)))


@pytest.mark.parametrize("sched", [[2, 0, 1, 0, 0, 3] + [0] * 20, [1, 1, 1, 0, 2] + [0] * 30, []])
def test_et_schedule_roundtrip(sched):
    """widths -> (et_widths, schedule) replays lu.py:318-323 exactly like the oracle does."""
    n, b_o, b_i = 256, 64, 8
    a = np.asfortranarray(make_matrix("uniform", n, 21))
    r = oracle.lu_la(a, b_o, b_i, et_sched=sched)
    assert sum(r.widths) == n
    again = mla.et_schedule_from(r.widths, n, b_o, b_i)
    b = np.asfortranarray(make_matrix("uniform", n, 21))
    r2 = oracle.lu_la(b, b_o, b_i, et_sched=again)
    assert r2.widths == r.widths and np.array_equal(a, b)
    cuts = mla.et_widths_from(r.widths, n, b_o, b_i)
    assert len(cuts) == r.et_events and all(c > 0 and c % b_i == 0 for c in cuts)


def test_workload_generators():
    u = splitmix64_uniform01(33, 7, 5)
    ref = oracle.alloc(33, 7)
    oracle.fill_random(ref, 5)
    assert np.array_equal(u, ref)
    a = make_matrix("uniform", 64, 0)
    assert a.flags.f_contiguous and a.min() > -1.0 and a.max() < 1.0
    rs = row_scale_vector(64)
    assert rs[0] == 1.0 and np.isclose(rs[-1], 10.0 ** (-6 * 63 / 64))
    b = make_matrix("uniform_rowscaled", 64, 0)
    assert np.array_equal(b, a * rs[:, None])
    c = make_matrix("normal", 32, 1)
    assert np.array_equal(c.ravel(order="F"), np.random.default_rng(1).standard_normal(32 * 32))
    assert set(CONFIGS) == {"config1", "config2", "config3", "config4", "config5"}


def test_config3_pivot_distance_is_reported_not_assumed():
    """SURVEY.md 8d caveat: the row scaling as written keeps pivots NEAR the diagonal."""
    n = 512
    a = np.asfortranarray(make_matrix("uniform_rowscaled", n, 2))
    r = oracle.lu_la(a, 128, 16)
    dist_scaled = float(np.mean(r.ipiv - np.arange(n)))
    b = np.asfortranarray(make_matrix("normal", n, 2))
    dist_normal = float(np.mean(oracle.lu_la(b, 128, 16).ipiv - np.arange(n)))
    assert dist_scaled < dist_normal


def test_bench_cli_argument_rules():  # reference test_bench.py: exit code 2 on bad arguments, CSV header
    from paper_1611_06365_b200 import bench_cli
    assert bench_cli.CSV_FIELDS == ("variant", "n", "b_outer", "b_inner", "threads", "t_pf", "seed",
                                    "wall_seconds", "gflops", "residual", "et_events")
    for argv in ([], ["--gepp"], ["--n", "64", "--b-outer", "8", "--b-inner", "16"],
                 ["--n", "64", "--b-inner", "0"], ["--n", "64", "--algo", "nope"], ["--n", "64", "--sweep-b", "3:1:1"]):
        with pytest.raises(SystemExit) as ei:
            ap = bench_cli.build_parser()
            bench_cli.validate(ap, ap.parse_args(argv))
        assert ei.value.code == 2
    ap = bench_cli.build_parser()
    args = ap.parse_args(["--n", "128", "--algo", "lu_et", "--sweep-b", "32:96:32"])
    bench_cli.validate(ap, args)
    assert args.sweep_b == [32, 64, 96]


def _synthetic_traces():
    from paper_1611_06365_b200.trace import TraceEvent
    ok = [TraceEvent(0, "PF", "GEMM", 0, 10, 1), TraceEvent(0, "PF", "PANEL", 10, 50, 1),
          TraceEvent(1, "PF", "PANEL", 11, 52, 1), TraceEvent(0, "MERGED", "GEMM", 51, 80, 1),
          TraceEvent(16, "RU", "GEMM", 0, 80, 1), TraceEvent(0, "ALL", "PANEL", -20, -1, 0)]
    bad = {
        "merged before any panel ended": [TraceEvent(0, "PF", "PANEL", 10, 50, 1), TraceEvent(1, "MERGED", "GEMM", 40, 80, 1)],
        "merged without a panel": [TraceEvent(1, "MERGED", "GEMM", 40, 80, 2)],
        "overlap on one worker": [TraceEvent(0, "PF", "GEMM", 0, 10, 1), TraceEvent(0, "PF", "PANEL", 5, 50, 1)],
        "unknown task": [TraceEvent(0, "PF", "NOPE", 0, 1, 1)],
        "negative duration": [TraceEvent(0, "RU", "GEMM", 5, 1, 1)],
    }
    return ok, bad


def test_trace_rules():  # the structural rules of reference trace.py:69-99 on this package's checker
    from paper_1611_06365_b200.trace import check_trace, idle_fraction, iteration_spans, validate
    ok, bad = _synthetic_traces()
    validate(ok)
    assert check_trace is validate
    assert iteration_spans(ok)[1] == (0, 80)
    assert abs(idle_fraction(ok, worker=16)[1]) < 1e-12
    for why, evs in bad.items():
        with pytest.raises(ValueError):
            validate(evs)


GPU_TRACE = os.path.join(ROOT, "tests", "golden", "gpu_trace_lu_mb.jsonl.gz")


@pytest.mark.skipif(not os.path.exists(GPU_TRACE), reason="no committed GPU trace")
def test_committed_gpu_trace_is_valid_and_merges():
    """A per-CTA trace recorded on a B200 (tests/golden/make_gpu_trace.py, lu_mb): structurally valid, every
    CTA of the grid contributed, panel-team CTAs joined the update (MERGED) after their panel, and with
    merging the panel team's lead has almost no idle gap in the early iterations (acceptance 4,
    test_acceptance.py:192-218)."""
    from paper_1611_06365_b200 import trace as mtrace
    evs = mtrace.load_jsonl(GPU_TRACE)
    mtrace.validate(evs)
    workers = {e.worker for e in evs}
    assert len(workers) >= 100 and workers == set(range(len(workers)))
    merged = [e for e in evs if e.team == "MERGED"]
    assert merged and all(e.t_start >= min(p.t_end for p in evs if p.team == "PF" and p.task == "PANEL"
                                           and p.iter_index == e.iter_index) for e in merged[:200])
    idle = mtrace.idle_fraction(evs, worker=0)
    early = [it for it in sorted({e.iter_index for e in merged}) if it >= 1][:4]
    assert early and all(idle[it] < 0.10 for it in early)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src/mla"), reason="reference not present (GPU box)")
def test_reference_checker_accepts_gpu_traces_and_agrees_on_violations():
    """the UNMODIFIED reference's check_trace / iteration_spans / load_jsonl run on the GPU
    trace file, and the reference's checker and this package's agree on every synthetic good / bad trace."""
    import gzip
    import importlib.util
    import tempfile
    spec = importlib.util.spec_from_file_location("ref_trace", "/root/reference/pkg/src/mla/trace.py")
    ref = importlib.util.module_from_spec(spec)
    sys.modules["ref_trace"] = ref
    spec.loader.exec_module(ref)
    from paper_1611_06365_b200 import trace as mtrace
    ok, bad = _synthetic_traces()
    as_ref = lambda evs: [ref.TraceEvent(e.worker, e.team, e.task, e.t_start, e.t_end, e.iter_index) for e in evs]
    ref.check_trace(as_ref(ok))
    assert ref.iteration_spans(as_ref(ok)) == mtrace.spans(ok)
    for why, evs in bad.items():
        with pytest.raises(ValueError):
            ref.check_trace(as_ref(evs))
        with pytest.raises(ValueError):
            mtrace.validate(evs)
    if os.path.exists(GPU_TRACE):
        with tempfile.NamedTemporaryFile("wb", suffix=".jsonl", delete=False) as tmp:
            tmp.write(gzip.open(GPU_TRACE, "rb").read())
        try:
            revs = ref.load_jsonl(tmp.name)                 # the reference's own reader
            ref.check_trace(revs)                           # ... and its own checker, unmodified
            assert ref.iteration_spans(revs) == mtrace.spans(mtrace.load_jsonl(GPU_TRACE))
            assert any(e.team == "MERGED" for e in revs)
        finally:
            os.unlink(tmp.name)


def test_packed_panel_layout_agrees_between_c_and_python():
    """mla_pack_panel's buffer layout (header + int32 pivots + panel) as the C side sizes it must be what
    distributed.py's views assume, for every scheduled width (ET makes widths vary per panel)."""
    from paper_1611_06365_b200 import _capi
    from paper_1611_06365_b200.distributed import DistLU
    lib = _capi.lib()
    for rows, w in [(65536, 512), (1216, 64), (300, 300), (97, 1), (1000, 24), (513, 130)]:
        assert int(lib.mla_packed_panel_doubles(rows, w)) == DistLU._hdr_doubles(w) + rows * w
        assert DistLU._hdr_doubles(w) * 2 >= 4 + w and (DistLU._hdr_doubles(w) * 8) % 16 == 0
