"""Dry run of the multi-GPU driver with its CUDA operator table on ONE GPU: world_size ranks (gloo
rendezvous, all on cuda:0, no kernel waits on another rank's kernel) factor a small matrix; rank 0
checks the assembled factors against the oracle.
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dev_dist_check.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
import oracle
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.distributed import DistLU, assemble_global, et_schedule_from_widths
from paper_1611_06365_b200.workloads import LuConfig
for n, b_o, b_i, dname, variant in [(1024, 128, 32, "uniform", "lu_et"), (1536, 256, 32, "normal", "lu_mb"),
                                    (1000, 128, 16, "uniform_rowscaled", "lu_et")]:
    cfg = LuConfig("t", n, dname, 4, b_o, b_i)
    dlu = DistLU(n, b_o, b_i, cfg, "cuda:0", variant=variant)
    dlu.generate()
    ipiv = dlu.factor()
    full = assemble_global(dlu)
    wl = [None] * world
    dist.all_gather_object(wl, (tuple(dlu.widths), bool(dlu.singular)))
    assert all(x == wl[0] for x in wl), "ranks disagree on the width schedule / singular flag"
    if rank == 0:
        ref = np.asfortranarray(mla.make_matrix(dname, n, 4))
        ro = oracle.lu_la(ref, b_o, b_i, et_sched=et_schedule_from_widths(dlu.widths, n, b_o, b_i, b_o), clamp=b_o)
        assert tuple(ro.widths) == tuple(dlu.widths), "width schedule not replayable on the oracle"
        piv_ok = np.array_equal(ipiv, ro.ipiv)
        scale = np.maximum(np.abs(ref), np.abs(ref).max(axis=0, keepdims=True))
        err = float((np.abs(full - ref) / scale).max())
        print(f"dist world={world} n={n} b={b_o}/{b_i} {dname} {variant} et_events={dlu.et_events}: pivots_equal={piv_ok} col-scaled err={err:.2e} launches={dlu.launches_per_factor}", flush=True)
        assert piv_ok and err < 1e-10
dist.barrier()
dist.destroy_process_group()
