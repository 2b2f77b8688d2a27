"""Device trace -> the reference's trace schema (trace.py:13-108).

The reference records per-worker events (worker, team, task, t_start, t_end, iter_index) as JSON
lines and validates two structural rules: events of one worker never overlap, and a MERGED-team event
only starts after that iteration's PF PANEL has ended (a merge can only consume workers the panel team
released).  The persistent kernel stamps every outer iteration with globaltimer values
(mla_getrf_trace: iteration start, panel-columns update complete, panel end, remainder complete);
here those stamps are mapped onto two representative workers -- worker 0 (rank 0 of the panel team)
and worker t_pf (first CTA of the update team) -- so that the reference's check_trace and the
acceptance-4 idle-gap metric (test_acceptance.py:171-218) run unchanged on GPU traces.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import asdict, dataclass

import numpy as np

from . import _capi

TASKS = ("PACK_A", "PACK_B", "GEMM", "TRSM", "LASWP", "PANEL", "BARRIER")
TRACE_ROWS = 1024


@dataclass(frozen=True)
class TraceEvent:
    worker: int
    team: str
    task: str
    t_start: int
    t_end: int
    iter_index: int


def device_trace(pool, n_iterations: int) -> np.ndarray:
    """Raw stamps of the last lu_la call: int64 array (iterations, 5), see include/mla_b200.h."""
    buf = (ctypes.c_uint64 * (5 * TRACE_ROWS))()
    got = _capi.lib().mla_getrf_trace(pool.handle, buf, TRACE_ROWS)
    rows = max(0, min(int(got), int(n_iterations)))
    return np.array(buf[:5 * rows], dtype=np.uint64).reshape(-1, 5).astype(np.int64)


def events_from_result(pool, result, variant: str, t_pf: int | None = None) -> list[TraceEvent]:
    """TraceEvents of the last lu_la call (`result` = its LuResult)."""
    t = device_trace(pool, len(result.widths) - 1)
    if len(t) == 0:
        return []
    t_pf = pool.t_pf if t_pf is None else t_pf
    origin = int(t[0, 0])
    ws = variant in ("lu_mb", "lu_et", "lu_ws_static")
    out: list[TraceEvent] = []
    for i, (s0, pq, pe, rq, _wk) in enumerate(t):
        it = i + 1
        s0, pq, pe, rq = (int(x) - origin for x in (s0, pq, pe, rq))
        rq = max(rq, s0) if rq > 0 - origin else s0
        if variant == "lu":
            continue
        out.append(TraceEvent(0, "PF", "GEMM", s0, pq, it))          # panel columns' update (PF1+PF2)
        out.append(TraceEvent(0, "PF", "PANEL", pq, pe, it))         # PF3
        if ws and rq > pe:
            out.append(TraceEvent(0, "MERGED", "GEMM", pe, rq, it))  # joined the remainder update (WS)
        out.append(TraceEvent(t_pf, "RU", "GEMM", s0, rq, it))       # RU1+RU2
    return out


def write_jsonl(events, path: str, append: bool = False) -> None:
    with open(path, "a" if append else "w", encoding="utf-8") as fh:
        for ev in events:
            fh.write(json.dumps(asdict(ev), separators=(",", ":")) + "\n")


def load_jsonl(path: str) -> list[TraceEvent]:
    out = []
    with open(path, encoding="utf-8") as fh:
        for line in fh:
            if line.strip():
                out.append(TraceEvent(**json.loads(line)))
    return out


def check_trace(events) -> None:
    """The reference's structural rules (trace.py:69-99), restated."""
    by_worker: dict[int, list[TraceEvent]] = {}
    for ev in events:
        if ev.task not in TASKS:
            raise ValueError(f"unknown task {ev.task!r}")
        if ev.t_end < ev.t_start:
            raise ValueError(f"event ends before it starts: {ev}")
        by_worker.setdefault(ev.worker, []).append(ev)
    for worker, evs in by_worker.items():
        evs.sort(key=lambda e: e.t_start)
        for a, b in zip(evs, evs[1:]):
            if b.t_start < a.t_end:
                raise ValueError(f"worker {worker} events overlap: {a} .. {b}")
    panel_end: dict[int, int] = {}
    for ev in events:
        if ev.team == "PF" and ev.task == "PANEL":
            panel_end[ev.iter_index] = min(panel_end.get(ev.iter_index, ev.t_end), ev.t_end)
    for ev in events:
        if ev.team == "MERGED":
            end = panel_end.get(ev.iter_index)
            if end is None or end > ev.t_start:
                raise ValueError(f"MERGED event with no completed PF panel before it: {ev}")


def iteration_spans(events) -> dict[int, tuple[int, int]]:
    spans: dict[int, tuple[int, int]] = {}
    for ev in events:
        lo, hi = spans.get(ev.iter_index, (ev.t_start, ev.t_end))
        spans[ev.iter_index] = (min(lo, ev.t_start), max(hi, ev.t_end))
    return spans


def pf_idle_fraction(events) -> dict[int, float]:
    """Acceptance-4 metric (test_acceptance.py:171-218): per iteration, the share of the iteration span
    in which the panel worker runs nothing."""
    spans = iteration_spans(events)
    busy: dict[int, int] = {}
    for ev in events:
        if ev.worker == 0:
            busy[ev.iter_index] = busy.get(ev.iter_index, 0) + (ev.t_end - ev.t_start)
    return {it: 1.0 - busy.get(it, 0) / max(1, hi - lo) for it, (lo, hi) in spans.items()}
