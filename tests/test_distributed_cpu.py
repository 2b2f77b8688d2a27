"""Multi-process (gloo, world_size 2 and 3) test of the 1-D block-cyclic LU host logic
(paper_1611_06365_b200/distributed.py) with a CPU operator table built on the oracle: ownership maps,
panel packing / broadcast schedule, look-ahead ordering and pivot bookkeeping are exactly the code the
NCCL path runs.  Because the per-element arithmetic is that of the serial schedule, the assembled
factors must be BITWISE equal to oracle.lu_la (reference lu.py:197-334) run with the same injected ET
cut schedule and the driver's one extra schedule rule (panels never cross a column block: clamp)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class CpuOps:
    """Operator table over CPU torch tensors (column-major views) -> numpy views -> oracle."""

    def __init__(self):
        import oracle
        self.o = oracle

    @staticmethod
    def _np(t):
        a = t.numpy()
        assert a.shape[0] <= 1 or a.strides[0] == 8
        return a

    def alloc(self, rows, cols, device):
        return torch.zeros((cols, max(rows, 1)), dtype=torch.float64).t()[:rows, :]

    crout = False    # the oracle's panel is the reference's left-looking lu_blk_ll: after a cut the
                     # untouched columns carry the interchanges only (lu.py:177-179)

    def panel(self, a, b_inner, stop_trip=0):
        r = self.o.lu_blk_ll(self._np(a), b_inner, stop_trip=stop_trip)
        return torch.from_numpy(r.ipiv.astype(np.int32)), r.singular, r.cols_factored

    def laswp(self, a, ipiv):
        self.o.laswp(self._np(a), np.asarray(ipiv, dtype=np.int64))

    def trsm(self, l11, b):
        self.o.trsm_llu(self._np(l11), self._np(b))

    def gemm(self, c, a, b):
        self.o.gemm(self._np(c), self._np(a), self._np(b), 1.0, -1.0)

    def fill(self, a, seed, col0, total_rows, scale, shift, row_scale):
        from paper_1611_06365_b200.workloads import splitmix64_uniform01
        rows, cols = a.shape
        u = splitmix64_uniform01(rows, col0 + cols, seed, col0=col0, ncols=cols, total_rows=total_rows)
        u = scale * u + shift
        if row_scale is not None:
            u = u * row_scale.numpy()[:, None]
        a.copy_(torch.from_numpy(np.ascontiguousarray(u.T)).t())


def _worker(rank, world, port, n, b_o, b_i, dist_name, out, et_sched=None):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1611_06365_b200.distributed import DistLU, assemble_global
        from paper_1611_06365_b200.workloads import LuConfig, make_matrix
        cfg = LuConfig("t", n, dist_name, 7, b_o, b_i)
        dlu = DistLU(n, b_o, b_i, cfg, "cpu", ops=CpuOps(), et_sched=et_sched)
        dlu.generate()
        # generated shares must equal the corresponding columns of the global generator
        full0 = make_matrix(dist_name, n, 7)
        assert np.array_equal(dlu.local_to_numpy(), full0[:, dlu.map.global_cols(rank)])
        ipiv = dlu.factor()
        full = assemble_global(dlu)
        ok = True
        if rank == 0:
            ref = np.asfortranarray(full0.copy(order="F"))
            ro = oracle.lu_la(ref, b_o, b_i, et_sched=et_sched, clamp=b_o)
            ok = np.array_equal(ipiv, ro.ipiv) and np.array_equal(full, ref)
            ok = ok and tuple(dlu.widths) == tuple(ro.widths) and dlu.et_events == ro.et_events
            if et_sched:
                ok = ok and dlu.et_events > 0
        # every rank holds the same pivot vector, width schedule and singular flag
        t = torch.from_numpy(ipiv.copy())
        dist.broadcast(t, src=0)
        ok = ok and np.array_equal(t.numpy(), ipiv)
        wl = [None] * world
        dist.all_gather_object(wl, (tuple(dlu.widths), bool(dlu.singular)))
        ok = ok and all(x == wl[0] for x in wl)
        dlu.restore()
        assert np.array_equal(dlu.local_to_numpy(), full0[:, dlu.map.global_cols(rank)])
        out.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


ET_A = [2, 0, 1, 0, 0, 3, 1, 0, 0, 2] + [0] * 40
ET_B = [1, 1, 1, 0, 2, 0, 0, 1, 0, 0, 3] + [0] * 40


@pytest.mark.parametrize("world,n,b_o,b_i,dist_name,et", [(2, 96, 16, 4, "uniform", None), (2, 100, 32, 8, "normal", None),
                                                          (3, 130, 16, 8, "uniform_rowscaled", None),
                                                          (2, 160, 32, 4, "uniform", ET_A), (3, 200, 32, 8, "normal", ET_B)])
def test_block_cyclic_lu_gloo(world, n, b_o, b_i, dist_name, et):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b_o, b_i, dist_name, out, et)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    results = {}
    while not out.empty():
        r, ok = out.get()
        results[r] = ok
    for p in procs:
        assert p.exitcode == 0
    assert results == {r: True for r in range(world)}


def test_block_cyclic_map():
    from paper_1611_06365_b200.distributed import BlockCyclic
    m = BlockCyclic(1000, 128, 3)
    assert m.nblocks == 8 and m.width(7) == 104
    allc = np.sort(np.concatenate([m.global_cols(r) for r in range(3)]))
    assert np.array_equal(allc, np.arange(1000))
    assert sum(m.local_cols(r) for r in range(3)) == 1000
    assert m.owner(5) == 2 and m.local_offset(5) == 128
    assert m.local_start_after(0, 0) == 128 and m.local_start_after(1, 0) == 0
    assert m.local_start_after(1, 7) == m.local_cols(1)


@pytest.mark.parametrize("n,b_o,b_i,et", [(100, 16, 4, None), (150, 32, 8, ET_A), (97, 32, 4, ET_B), (64, 64, 8, None),
                                          (130, 16, 16, ET_A)])
def test_single_rank_host_logic_with_et(n, b_o, b_i, et):
    """World size 1 (no process group): the schedule / pend / skip bookkeeping of DistLU.factor alone,
    bitwise against the oracle's replay, with and without injected ET cuts."""
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1611_06365_b200.distributed import DistLU, PanelSchedule, et_schedule_from_widths
    from paper_1611_06365_b200.workloads import LuConfig, make_matrix
    cfg = LuConfig("t", n, "uniform", 3, b_o, b_i)
    dlu = DistLU(n, b_o, b_i, cfg, "cpu", ops=CpuOps(), rank=0, world=1, et_sched=et)
    dlu.generate()
    ipiv = dlu.factor()
    ref = np.asfortranarray(make_matrix("uniform", n, 3))
    ro = oracle.lu_la(ref, b_o, b_i, et_sched=et, clamp=b_o)
    assert np.array_equal(ipiv, ro.ipiv) and np.array_equal(dlu.local_to_numpy(), ref)
    assert tuple(dlu.widths) == tuple(ro.widths) and sum(dlu.widths) == n
    # the width list alone reproduces the trips (what the GPU tests use to replay a timing-dependent run)
    again = np.asfortranarray(make_matrix("uniform", n, 3))
    r2 = oracle.lu_la(again, b_o, b_i, et_sched=et_schedule_from_widths(dlu.widths, n, b_o, b_i, b_o), clamp=b_o)
    assert tuple(r2.widths) == tuple(dlu.widths) and np.array_equal(again, ref)
    # no panel crosses a column-block boundary
    q = 0
    for w in dlu.widths:
        assert q // b_o == (q + w - 1) // b_o
        q += w


def test_local_lt_matches_the_block_cyclic_map():
    from paper_1611_06365_b200.distributed import BlockCyclic, DistLU
    for n, b, P in [(1000, 128, 3), (512, 64, 2), (130, 16, 4), (65, 64, 2)]:
        m = BlockCyclic(n, b, P)
        for r in range(P):
            d = DistLU(n, b, max(1, b // 8), None, "cpu", ops=CpuOps(), rank=r, world=P)
            cols = m.global_cols(r)
            for c in list(range(0, n + 1, 7)) + [n]:
                assert d.local_lt(c) == int((cols < c).sum())
