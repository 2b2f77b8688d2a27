"""The multi-GPU driver through a real NCCL communicator with ONE rank (all this run's single GPU allows):
init_process_group("nccl"), every panel broadcast issued on the communication stream with the buffer-reuse
events in place, look-ahead + WS + ET on; checked against the oracle replay.
    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 tools/dev_dist_nccl1.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import oracle
import paper_1611_06365_b200 as mla
from paper_1611_06365_b200.distributed import DistLU, et_schedule_from_widths
from paper_1611_06365_b200.workloads import LuConfig
for n, b_o, b_i, variant in [(1536, 256, 32, "lu_et"), (2000, 128, 16, "lu_mb"), (3072, 256, 32, "lu_et")]:
    cfg = LuConfig("t", n, "uniform", 4, b_o, b_i)
    dlu = DistLU(n, b_o, b_i, cfg, "cuda:0", variant=variant, comm_always=True)
    assert dlu.comm_always
    dlu.generate()
    ipiv = dlu.factor()
    ref = np.asfortranarray(mla.make_matrix("uniform", n, 4))
    ro = oracle.lu_la(ref, b_o, b_i, et_sched=et_schedule_from_widths(dlu.widths, n, b_o, b_i, b_o), clamp=b_o)
    piv_ok = np.array_equal(ipiv, ro.ipiv) and tuple(ro.widths) == tuple(dlu.widths)
    scale = np.maximum(np.abs(ref), np.abs(ref).max(axis=0, keepdims=True))
    err = float((np.abs(dlu.local_to_numpy() - ref) / scale).max())
    print(f"nccl world=1 n={n} b={b_o}/{b_i} {variant} et_events={dlu.et_events}: pivots_equal={piv_ok} col-scaled err={err:.2e}", flush=True)
    assert piv_ok and err < 1e-10
dist.barrier()
dist.destroy_process_group()
