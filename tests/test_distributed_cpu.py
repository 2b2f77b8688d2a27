"""Multi-process (gloo, world_size 2 and 3) test of the 1-D block-cyclic LU host logic
(paper_1611_06365_b200/distributed.py) with a CPU operator table built on the oracle: ownership maps,
panel packing / broadcast schedule, look-ahead ordering and pivot bookkeeping are exactly the code the
NCCL path runs.  Because the per-element arithmetic is that of the serial schedule, the assembled
factors must be BITWISE equal to oracle.lu_la (reference lu.py:197-334, variant "lu")."""
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

    def panel(self, a, b_inner):
        r = self.o.lu_blk_ll(self._np(a), b_inner)
        return torch.from_numpy(r.ipiv.astype(np.int32)), r.singular

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


def _worker(rank, world, port, n, b_o, b_i, dist_name, out):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1611_06365_b200.distributed import DistLU, assemble_global
        from paper_1611_06365_b200.workloads import LuConfig, make_matrix
        cfg = LuConfig("t", n, dist_name, 7, b_o, b_i)
        dlu = DistLU(n, b_o, b_i, cfg, "cpu", ops=CpuOps())
        dlu.generate()
        # generated shares must equal the corresponding columns of the global generator
        full0 = make_matrix(dist_name, n, 7)
        assert np.array_equal(dlu.local_to_numpy(), full0[:, dlu.map.global_cols(rank)])
        ipiv = dlu.factor()
        full = assemble_global(dlu)
        ok = True
        if rank == 0:
            ref = np.asfortranarray(full0.copy(order="F"))
            ro = oracle.lu_la(ref, b_o, b_i)
            ok = np.array_equal(ipiv, ro.ipiv) and np.array_equal(full, ref)
        # every rank holds the same pivot vector
        t = torch.from_numpy(ipiv.copy())
        dist.broadcast(t, src=0)
        ok = ok and np.array_equal(t.numpy(), ipiv)
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


@pytest.mark.parametrize("world,n,b_o,b_i,dist_name", [(2, 96, 16, 4, "uniform"), (2, 100, 32, 8, "normal"),
                                                       (3, 130, 16, 8, "uniform_rowscaled")])
def test_block_cyclic_lu_gloo(world, n, b_o, b_i, dist_name):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b_o, b_i, dist_name, out)) for r in range(world)]
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
