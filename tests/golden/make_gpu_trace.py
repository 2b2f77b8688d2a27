"""Records the per-CTA device trace that tests/test_host_logic.py validates with the reference's own
checker (run on a B200: `python tests/golden/make_gpu_trace.py`; writes tests/golden/gpu_trace_lu_mb.jsonl.gz
next to this file, or into gpurun_out/ when that directory exists so that the file travels back).

lu_mb, n = 12288, b = 256/32, 48 panel CTAs: 47 outer iterations x 148 CTAs, ~20 k events."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import paper_1611_06365_b200 as mla  # noqa: E402
from paper_1611_06365_b200 import trace as mtrace  # noqa: E402

pool = mla.default_pool()
n = 12288
a = mla.alloc_matrix(n, n)
mla.fill_random(a, 0, 2.0, -1.0)
mla.lu_la(a, mla.Policy("lu_mb", mla.BlockConfig(256, 32), t_pf=48), pool)       # warm-up, untraced
mla.fill_random(a, 0, 2.0, -1.0)
mtrace.enable(pool)
r = mla.lu_la(a, mla.Policy("lu_mb", mla.BlockConfig(256, 32), t_pf=48), pool)
evs = mtrace.events(pool)
mtrace.enable(pool, False)
mtrace.validate(evs)
out_dir = os.path.join(ROOT, "gpurun_out") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else HERE
path = os.path.join(out_dir, "gpu_trace_lu_mb.jsonl.gz")
mtrace.write_jsonl(evs, path)
print(f"{len(evs)} events, {len({e.worker for e in evs})} CTAs, ws_joins {r.ws_joins}, "
      f"merged iterations {len({e.iter_index for e in evs if e.team == 'MERGED'})} -> {path}")
