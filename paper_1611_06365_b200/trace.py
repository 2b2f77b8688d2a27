"""Device trace -> the reference's trace schema (reference trace.py:13-66).

The reference's Tracer keeps one private event buffer per worker thread and serialises
(worker, team, task, t_start, t_end, iter_index) records as JSON lines.  Here the workers are the CTAs of
the persistent kernel: with tracing on (`enable(pool)`), thread 0 of EVERY CTA appends one record per phase
it actually ran -- drained the next panel's update queue, factored the look-ahead panel as a member of
the panel team, drained the remainder queue as a member of the update team, or (worker sharing) entered
that queue after its panel ended -- stamped with the GPU's globaltimer where the phase really starts and
ends (include/mla_b200.h: mla_set_trace / mla_getrf_events).  `events()` maps those records onto
TraceEvents, so a trace file written here is a valid input to the reference's own `check_trace` /
`iteration_spans` and to its acceptance-4 idle-gap metric (test_acceptance.py:171-218); the tests run the
unmodified reference checker over a GPU trace committed under tests/golden/.

`validate` is this package's own structural checker (the GPU box has no copy of the reference).
"""
from __future__ import annotations

import ctypes
import gzip
import json
from dataclasses import asdict, dataclass

import numpy as np

from . import _capi

TASKS = ("PACK_A", "PACK_B", "GEMM", "TRSM", "LASWP", "PANEL", "BARRIER")    # reference trace.py:13
EVENTS_PER_CTA = 4096

# kind of a device record -> (team, task) of the reference's vocabulary (pool.py:22-25, trace.py:13)
_KIND = {1: ("{role}", "GEMM"), 2: ("PF", "PANEL"), 3: ("RU", "GEMM"), 4: ("MERGED", "GEMM"), 5: ("ALL", "PANEL")}

_REC = np.dtype([("t_start", "<u8"), ("t_end", "<u8"), ("iter", "<i4"), ("kind", "<i4"), ("items", "<i4"),
                 ("team", "<i4")])


@dataclass(frozen=True)
class TraceEvent:
    worker: int
    team: str
    task: str
    t_start: int
    t_end: int
    iter_index: int


def enable(pool, on: bool = True) -> None:
    """Switch the per-CTA event rings of the persistent kernel on (19 MB of device memory) or off."""
    _capi.check(_capi.lib().mla_set_trace(pool.handle, int(bool(on))), pool.handle, "mla_set_trace")


def device_records(pool) -> np.ndarray:
    """Raw records of the last lu_la call: structured array (ctas, EVENTS_PER_CTA); kind 0 = unused."""
    buf = np.zeros((160, EVENTS_PER_CTA), dtype=_REC)
    got = _capi.lib().mla_getrf_events(pool.handle, buf.ctypes.data_as(ctypes.c_void_p), EVENTS_PER_CTA)
    if got < 0:
        _capi.check(got, pool.handle, "mla_getrf_events")
    return buf[:got]


def events(pool, variant: str | None = None) -> list[TraceEvent]:
    """TraceEvents of the last lu_la call, one worker per CTA, times in ns relative to the first stamp,
    sorted like the reference's Tracer.events() (trace.py:41-46)."""
    rec = device_records(pool)
    used = rec["kind"] > 0
    if not used.any():
        return []
    origin = int(rec["t_start"][used].min())
    out: list[TraceEvent] = []
    for cta in range(rec.shape[0]):
        for r in rec[cta][used[cta]]:
            team, task = _KIND[int(r["kind"])]
            if team == "{role}":
                # the next panel's columns are updated by everybody before the teams part (lu.py:279-289):
                # a panel-team CTA does it as PF1/PF2, an update-team CTA as a helper of that step
                team = "PF" if cta < int(r["team"]) else "RU"
            out.append(TraceEvent(cta, team, task, int(r["t_start"]) - origin, int(r["t_end"]) - origin, int(r["iter"])))
    out.sort(key=lambda e: (e.t_start, e.worker, e.t_end))
    return out


def write_jsonl(evs, path: str, append: bool = False) -> None:
    """One JSON object per line, the reference's serialisation (trace.py:52-56); *.gz is gzip-compressed."""
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "at" if append else "wt", encoding="utf-8") as fh:
        for ev in evs:
            fh.write(json.dumps(asdict(ev), separators=(",", ":")) + "\n")


def load_jsonl(path: str) -> list[TraceEvent]:
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        return [TraceEvent(**json.loads(line)) for line in fh if line.strip()]


def validate(evs) -> None:
    """Structural rules a trace of this package must satisfy; raises ValueError naming the first violation.
      1. every task name belongs to the reference's vocabulary, no event has negative duration;
      2. a worker (CTA) never runs two phases at once;
      3. worker sharing: a MERGED record of iteration i needs a PANEL record of the panel team in the same
         iteration that ended before it starts (the donors join after their panel, pool.py:211-223); like
         the reference's rule (trace.py:90-99) the comparison is with the EARLIEST panel end: the members
         leave the team's last barrier, and stamp, a few hundred ns apart."""
    if not evs:
        return
    worker = np.array([e.worker for e in evs])
    t0 = np.array([e.t_start for e in evs], dtype=np.int64)
    t1 = np.array([e.t_end for e in evs], dtype=np.int64)
    it = np.array([e.iter_index for e in evs])
    bad = [e.task for e in evs if e.task not in TASKS]
    if bad:
        raise ValueError(f"task name outside the reference vocabulary: {bad[0]!r}")
    neg = np.nonzero(t1 < t0)[0]
    if neg.size:
        raise ValueError(f"negative duration: {evs[int(neg[0])]}")
    order = np.lexsort((t0, worker))
    same = worker[order][1:] == worker[order][:-1]
    clash = np.nonzero(same & (t0[order][1:] < t1[order][:-1]))[0]
    if clash.size:
        k = int(clash[0])
        raise ValueError(f"CTA {int(worker[order][k])} runs two phases at once: {evs[int(order[k])]} and {evs[int(order[k + 1])]}")
    panel = np.array([e.team == "PF" and e.task == "PANEL" for e in evs])
    merged = np.array([e.team == "MERGED" for e in evs])
    first_end: dict[int, int] = {}
    for i in np.nonzero(panel)[0]:
        first_end[int(it[i])] = min(first_end.get(int(it[i]), int(t1[i])), int(t1[i]))
    for i in np.nonzero(merged)[0]:
        end = first_end.get(int(it[i]))
        if end is None or int(t0[i]) < end:
            raise ValueError(f"worker-sharing join before the panel team was done: {evs[int(i)]}")


def spans(evs) -> dict[int, tuple[int, int]]:
    """[first start, last end] of every outer iteration."""
    out: dict[int, list[int]] = {}
    for e in evs:
        s = out.setdefault(e.iter_index, [e.t_start, e.t_end])
        s[0], s[1] = min(s[0], e.t_start), max(s[1], e.t_end)
    return {k: (v[0], v[1]) for k, v in out.items()}


def idle_fraction(evs, worker: int = 0) -> dict[int, float]:
    """Per iteration, the share of the iteration's span in which `worker` ran nothing -- acceptance 4's
    question (test_acceptance.py:171-218: does merging keep the panel worker busy?) asked of a CTA."""
    sp = spans(evs)
    busy: dict[int, int] = {}
    for e in evs:
        if e.worker == worker:
            busy[e.iter_index] = busy.get(e.iter_index, 0) + (e.t_end - e.t_start)
    return {k: 1.0 - busy.get(k, 0) / max(1, hi - lo) for k, (lo, hi) in sp.items()}


# the reference's names for the same things (trace.py:69-108), kept so that callers of `mla.check_trace` /
# `mla.trace.iteration_spans` find them here
check_trace = validate
iteration_spans = spans
