"""Multi-GPU LU (BASELINE.json config 5): 1-D block-cyclic column distribution over the
GPUs of one NVSwitch box, one process per GPU, panel + pivot broadcast over NCCL.

The reference has no multi-device path (single process, thread teams; pool.py:18-20), so this layer is
the spec's own design on top of the same operators the single-GPU path uses:

  * column block j (width b) lives on rank j mod P, full height, stored contiguously column-major;
    row interchanges, trsm and gemm on owned columns therefore need no communication;
  * per outer iteration k the owner of block k factors the panel (lu_blk_ll semantics, lu.py:140-180),
    packs it with its pivots into ONE contiguous buffer and broadcasts it (NCCL over NVLink);
  * look-ahead: the owner of block k+1 updates that block FIRST, factors it and starts its broadcast on
    a side stream before it updates the rest of its columns, so the broadcast of panel k+1 overlaps
    everybody's update k (the exchange is hidden except in the tail);
  * every rank then applies panel k to its local columns right of it: laswp -> trsm_llu -> gemm
    (the reference's PF1/RU1, PF2/RU2 of lu.py:279-308), and the interchanges to its columns left of it.

The arithmetic schedule equals the single-device variant "lu" (fixed width b), so the CPU oracle's
lu_la(b_outer, b_inner) is the parity reference for the assembled matrix.

All compute goes through an operator table (`ops`): the default binds the CUDA kernels of this package;
tests inject a CPU table (numpy views + the oracle) to exercise exactly this host logic under gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class BlockCyclic:
    """1-D block-cyclic map of n columns in blocks of b over P ranks."""

    n: int
    b: int
    P: int

    @property
    def nblocks(self) -> int:
        return (self.n + self.b - 1) // self.b

    def owner(self, j: int) -> int:
        return j % self.P

    def width(self, j: int) -> int:
        return min(self.b, self.n - j * self.b)

    def owned(self, rank: int) -> list[int]:
        return list(range(rank, self.nblocks, self.P))

    def local_cols(self, rank: int) -> int:
        return sum(self.width(j) for j in self.owned(rank))

    def local_offset(self, j: int) -> int:
        """First local column of global block j on its owner."""
        return (j // self.P) * self.b

    def local_start_after(self, rank: int, k: int) -> int:
        """Local column index of the first owned block with global index > k."""
        nb = len([j for j in self.owned(rank) if j <= k])
        return nb * self.b if nb * self.b <= self.local_cols(rank) else self.local_cols(rank)

    def global_cols(self, rank: int) -> np.ndarray:
        out = []
        for j in self.owned(rank):
            out.extend(range(j * self.b, j * self.b + self.width(j)))
        return np.array(out, dtype=np.int64)


class CudaOps:
    """Operator table bound to libmla_b200.so (the product path)."""

    def __init__(self, pool=None):
        from . import kernels, lu, matrix
        self._k, self._lu, self._m = kernels, lu, matrix
        self.pool = pool

    def alloc(self, rows, cols, device):
        return self._m.alloc_matrix(rows, cols, device=device)

    def panel(self, a, b_inner):
        """-> (pivots as a device int32 tensor, singular)"""
        r = self._lu.lu_blk_ll(a, b_inner, pool=self.pool)
        return r.ipiv.device, r.singular

    def laswp(self, a, ipiv):
        self._k.laswp(a, ipiv, pool=self.pool, check=False)   # pivots come from the panel kernel

    def trsm(self, l11, b):
        self._k.trsm_llu(l11, b, pool=self.pool)

    def gemm(self, c, a, b):
        self._k.gemm_malleable(c, a, b, 1.0, -1.0, pool=self.pool)

    def fill(self, a, seed, col0, total_rows, scale, shift, row_scale):
        self._m.fill_random(a, seed, scale, shift, row_scale=row_scale, col0=col0, total_rows=total_rows,
                            pool=self.pool)

    def apply_panel(self, panel, w, target, piv):
        """laswp + trsm + gemm of one update step as ONE persistent launch (no host sync)."""
        self._k.apply_panel(panel, w, target, piv, pool=self.pool)

    # ---- the owner's next panel beside its update (second handle = second set of control words) ----
    _side_pools: dict = {}      # one side handle per device, shared by all drivers of this process

    def make_side_pool(self, device):
        from .pool import SmPool, default_pool
        self.pool = self.pool or default_pool(device.index)
        sp = CudaOps._side_pools.get(device.index)
        if sp is None or sp._closed:
            sp = SmPool(device.index)
            CudaOps._side_pools[device.index] = sp
        self.side_pool = sp
        return sp

    def panel_async(self, a, b_inner, team_sms, singular_accum):
        """Stream-ordered panel on `team_sms` SMs of the side handle -> device pivots."""
        return self._lu.lu_blk_ll_async(a, b_inner, self.side_pool, team_sms, singular_accum)

    def set_update_sms(self, ctas):
        self.pool.set_update_sms(ctas)

    def apply_panel_side(self, panel, w, target, piv, ctas):
        """apply_panel through the side handle on `ctas` SMs (for the side stream)."""
        self.side_pool.set_update_sms(ctas)
        self._k.apply_panel(panel, w, target, piv, pool=self.side_pool)

    def laswp_side(self, a, ipiv):
        """laswp through the side handle (its own plan buffer), for the side stream."""
        self._k.laswp(a, ipiv, pool=self.side_pool, check=False)

    def apply_prepare(self, piv, w, rows, device):
        self._k.apply_panel_prepare(piv, w, rows, device, pool=self.pool)

    def apply_launch(self, panel, w, target, ctas):
        self._k.apply_panel_launch(panel, w, target, ctas, pool=self.pool)


class DistLU:
    """One rank's share of a block-cyclic LU.  `group` = process group (default WORLD)."""

    def __init__(self, n, b_outer, b_inner, cfg, device, variant="lu_la", pool=None, ops=None, group=None,
                 rank=None, world=None, panel_sms=32, comm_sms=8, storage=None, overlap_panel=False):
        self.n, self.b, self.b_inner, self.cfg = n, b_outer, b_inner, cfg
        self.device = torch.device(device)
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.P = dist.get_world_size(group) if world is None else world
        self.map = BlockCyclic(n, b_outer, self.P)
        self.ops = ops or CudaOps(pool)
        self.nloc = self.map.local_cols(self.rank)
        # `storage`: factor the caller's (n x nloc, column-major) tensor in place instead of an own buffer
        self.a = storage if storage is not None else self.ops.alloc(n, max(self.nloc, 1), self.device)[:, :self.nloc]
        self.a0 = None
        self.ipiv = np.zeros(n, dtype=np.int64)
        self.singular = False
        self.cuda = self.device.type == "cuda"
        self.comm_stream = torch.cuda.Stream(self.device) if self.cuda else None
        self.launches_per_factor = 0
        # EXPERIMENTAL, OFF BY DEFAULT (overlap_panel=True): look-ahead on the device -- the owner of block
        # k+1 applies panel k to that block, factors panel k+1 and does the LEFT interchanges on
        # `panel_sms` SMs (side handle, side stream) WHILE panel k is applied to the rest of its columns
        # on the other SMs, and those SMs then join the update's queue with a second launch.  Fast
        # (P=1: n=32768 0.885 s, n=65536 6.26 s) but NOT CORRECT: with the panel kernel running beside
        # the update kernel the factors come out wrong, non-deterministically, once the run is long
        # enough (n > 32768, or n=32768 with b=256; backward error ~1e10 n eps; found by bench.py --check).
        # Each piece is right on its own -- the same launches with a device synchronisation between panel
        # and update are bitwise reproducible and pass -- so it is an interaction of the two concurrently
        # resident kernels that round 1 did not root-cause.
        self.overlap = bool(overlap_panel) and self.cuda and hasattr(self.ops, "panel_async")
        if self.overlap:
            self.ops.make_side_pool(self.device)
            self.panel_stream = torch.cuda.Stream(self.device)
            self.sms = self.ops.pool.t
            self.panel_sms = max(1, min(int(panel_sms), self.sms - 1))
            self.comm_sms = int(comm_sms) if self.P > 1 else 0
            self._sing_dev = torch.zeros(1, dtype=torch.int32, device=self.device)
        # two broadcast buffers (double buffering: panel k+1 is in flight while panel k is consumed)
        cap = n * b_outer + b_outer
        self.bufs = [torch.zeros(cap, dtype=torch.float64, device=self.device) for _ in range(2)]

    # ---- data ---------------------------------------------------------------------------------
    def generate(self):
        """Fill the owned column blocks of the config's matrix (uniform configs: on the device, each
        block independently through the counter-based stream; normal configs: host generator)."""
        cfg, n = self.cfg, self.n
        if cfg.dist in ("uniform", "uniform_rowscaled"):
            rs = None
            if cfg.dist == "uniform_rowscaled":
                from .workloads import row_scale_vector
                rs = torch.from_numpy(row_scale_vector(n)).to(self.device)
            for j in self.map.owned(self.rank):
                lo = self.map.local_offset(j)
                w = self.map.width(j)
                self.ops.fill(self.a[:, lo:lo + w], cfg.seed, j * self.b, n, 2.0, -1.0, rs)
        else:
            from .workloads import make_matrix
            full = make_matrix(cfg.dist, n, cfg.seed)
            self.set_local_from_global(full)
        self.a0 = self.a.clone() if self.nloc else None

    def set_local_from_global(self, full: np.ndarray):
        cols = self.map.global_cols(self.rank)
        if cols.size:
            loc = np.ascontiguousarray(full[:, cols].T)
            self.a.copy_(torch.from_numpy(loc).t().to(self.device))
        self.a0 = self.a.clone() if self.nloc else None

    def restore(self):
        if self.a0 is not None:
            self.a.copy_(self.a0)

    def local_to_numpy(self) -> np.ndarray:
        return np.asfortranarray(self.a.detach().cpu().numpy())

    # ---- broadcast of one factored panel ---------------------------------------------------------
    def _pack(self, buf, k, piv):
        """panel k (rows k*b.., its w columns) + pivots -> one contiguous buffer."""
        j0, w = k * self.b, self.map.width(k)
        rows = self.n - j0
        lo = self.map.local_offset(k)
        view = buf[: w * rows].view(w, rows).t()        # column-major rows x w
        view.copy_(self.a[j0:, lo:lo + w])
        buf[w * rows: w * rows + w].copy_(torch.as_tensor(piv).to(device=self.device, dtype=torch.float64))

    def _unpack(self, buf, k):
        j0, w = k * self.b, self.map.width(k)
        rows = self.n - j0
        panel = buf[: w * rows].view(w, rows).t()
        piv = buf[w * rows: w * rows + w].to(torch.int32)       # stays on the device: no host sync
        return panel, piv

    def _bcast(self, buf, k):
        j0, w = k * self.b, self.map.width(k)
        count = w * (self.n - j0) + w
        src = self.map.owner(k)
        if self.group is not None:
            src = dist.get_global_rank(self.group, src)
        if self.P > 1:
            dist.broadcast(buf[:count], src=src, group=self.group)

    # ---- the factorization -----------------------------------------------------------------------
    def _factor_panel(self, k):
        j0, w = k * self.b, self.map.width(k)
        lo = self.map.local_offset(k)
        piv, sing = self.ops.panel(self.a[j0:, lo:lo + w], self.b_inner)
        self.launches_per_factor += 1
        return piv, bool(sing)

    def _apply(self, k, panel, piv, col_lo, col_hi):
        """Apply panel k to local columns [col_lo, col_hi) that lie right of it."""
        if col_hi <= col_lo:
            return
        j0, w = k * self.b, self.map.width(k)
        tgt = self.a[j0:, col_lo:col_hi]
        if hasattr(self.ops, "apply_panel"):
            self.ops.apply_panel(panel, w, tgt, piv)
            self.launches_per_factor += 2
            return
        self.ops.laswp(tgt, piv)
        self.ops.trsm(panel[:w, :w], tgt[:w, :])
        if self.n - j0 - w > 0:
            self.ops.gemm(tgt[w:, :], panel[w:, :w], tgt[:w, :])
        self.launches_per_factor += 4

    def factor(self):
        """P A = L U on the distributed matrix; returns the global pivot vector (host int64)."""
        m = self.map
        self.launches_per_factor = 0
        self.singular = False
        self._piv_dev = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        if self.overlap:
            self._sing_dev.zero_()
        nb = m.nblocks
        # panel 0
        cur = 0
        if m.owner(0) == self.rank:
            piv, sing = self._factor_panel(0)
            self.singular |= sing
            self._pack(self.bufs[0], 0, piv)
        self._bcast(self.bufs[0], 0)
        for k in range(nb):
            buf = self.bufs[cur]
            panel, piv = self._unpack(buf, k)
            j0, w = k * self.b, m.width(k)
            self._piv_dev[j0:j0 + w] = piv + j0
            right_lo = m.local_start_after(self.rank, k)
            nxt = 1 - cur
            left_done = False
            if k + 1 < nb and m.owner(k + 1) == self.rank and self.overlap:
                # Look-ahead on the device.  Side stream, panel_sms SMs (side handle): panel k applied to
                # block k+1, panel k+1 factored, packed, its broadcast started, the LEFT interchanges of
                # panel k -- then those SMs JOIN the main update's queue with a second launch.  Main
                # stream, the other SMs: panel k applied to the rest of the owned columns, from the start.
                lo = m.local_offset(k + 1)
                w1 = m.width(k + 1)
                j1 = (k + 1) * self.b
                main = torch.cuda.current_stream(self.device)
                self.panel_stream.wait_stream(main)
                have_rest = self.nloc > lo + w1
                if have_rest:
                    tgt = self.a[j0:, lo + w1:self.nloc]
                    self.ops.set_update_sms(0)
                    self.ops.apply_prepare(piv, w, self.n - j0, self.device)
                    ready = torch.cuda.Event()
                    ready.record(main)
                    self.ops.apply_launch(panel, w, tgt, self.sms - self.panel_sms - self.comm_sms)
                    self.launches_per_factor += 2
                with torch.cuda.stream(self.panel_stream):
                    self.ops.apply_panel_side(panel, w, self.a[j0:, lo:lo + w1], piv, self.panel_sms)
                    piv1 = self.ops.panel_async(self.a[j1:, lo:lo + w1], self.b_inner, self.panel_sms, self._sing_dev)
                    self._pack(self.bufs[nxt], k + 1, piv1)
                    self.launches_per_factor += 3
                self._start_bcast(nxt, k + 1, after=self.panel_stream)
                with torch.cuda.stream(self.panel_stream):
                    # the interchanges of the owned columns LEFT of panel k (lu.py:252) touch neither the
                    # update's columns nor the new panel
                    left_hi = right_lo - (w if m.owner(k) == self.rank else 0)
                    if left_hi > 0:
                        self.ops.laswp_side(self.a[j0:, :left_hi], piv)
                        self.launches_per_factor += 1
                        left_done = True
                    if have_rest:
                        self.panel_stream.wait_event(ready)
                        self.ops.apply_launch(panel, w, tgt, self.panel_sms)
                        self.launches_per_factor += 1
                main.wait_stream(self.panel_stream)
            elif k + 1 < nb and m.owner(k + 1) == self.rank:
                # look-ahead: next panel's block first, factor it, start its broadcast early
                lo = m.local_offset(k + 1)
                w1 = m.width(k + 1)
                self._apply(k, panel, piv, lo, lo + w1)
                piv1, sing = self._factor_panel(k + 1)
                self.singular |= sing
                self._pack(self.bufs[nxt], k + 1, piv1)
                self._start_bcast(nxt, k + 1)
                self._apply(k, panel, piv, lo + w1, self.nloc)
            else:
                if k + 1 < nb:
                    self._start_bcast(nxt, k + 1)
                if self.overlap and self.comm_sms:
                    self.ops.set_update_sms(self.sms - self.comm_sms)
                self._apply(k, panel, piv, right_lo, self.nloc)
                if self.overlap and self.comm_sms:
                    self.ops.set_update_sms(0)
            # interchanges for the owned columns left of the panel (lu.py:252, 329-332)
            left_hi = right_lo - (w if m.owner(k) == self.rank else 0)
            if left_hi > 0 and not left_done:
                self.ops.laswp(self.a[j0:, :left_hi], piv)
                self.launches_per_factor += 1
            if k + 1 < nb:
                self._finish_bcast()
            cur = nxt
        if self.overlap:
            self.singular |= bool(int(self._sing_dev.item()))
        self.ipiv = self._piv_dev.cpu().numpy().astype(np.int64)   # the only device->host copy
        return self.ipiv

    def _start_bcast(self, which, k, after=None):
        if self.cuda and self.P > 1:
            self.comm_stream.wait_stream(after if after is not None else torch.cuda.current_stream(self.device))
            with torch.cuda.stream(self.comm_stream):
                self._bcast(self.bufs[which], k)
        else:
            self._bcast(self.bufs[which], k)

    def _finish_bcast(self):
        if self.cuda and self.P > 1:
            torch.cuda.current_stream(self.device).wait_stream(self.comm_stream)


def lu_streams(a: torch.Tensor, b_outer: int, b_inner: int, pool=None, panel_sms: int = 32):
    """Single-GPU LU of a square column-major matrix, in place, through THIS driver with P = 1: per outer
    iteration separately compiled kernels (panel on all SMs, then one fused update launch, then the LEFT
    interchanges) instead of the one persistent kernel behind lu_la.  Fixed panel width (the schedule
    of variant "lu"; no look-ahead overlap, no early termination): n=32768 1.05 s against lu_la's 0.875 s.
    Returns a LuResult like lu_la.  Not exported from the package: lu_la is the single-GPU path; this
    one exists to exercise the driver on one GPU (parity at test sizes and, at n=32768, pivots equal to
    lu_la's).  The two-stream variant of this driver is faster but corrupts, see DistLU(overlap_panel=...)."""
    from .lu import LuResult
    from .matrix import PivotVector, check_colmajor
    m, n, _ = check_colmajor(a, "a")
    if m != n:
        raise ValueError("lu_streams: square matrices only")
    if n == 0:
        return LuResult(PivotVector(np.empty(0, dtype=np.int64)), 0, False)
    dlu = DistLU(n, b_outer, b_inner, None, a.device, pool=pool, rank=0, world=1, panel_sms=panel_sms, storage=a,
                 overlap_panel=False)
    ipiv = dlu.factor()
    widths = tuple(dlu.map.width(j) for j in range(dlu.map.nblocks))
    return LuResult(PivotVector(ipiv, device=dlu._piv_dev), n, bool(dlu.singular), 0, (), widths, dlu.map.nblocks - 1)


def assemble_global(dlu: DistLU) -> np.ndarray | None:
    """Gather every rank's columns on rank 0 (tests / small n only)."""
    P, rank = dlu.P, dlu.rank
    loc = torch.from_numpy(np.ascontiguousarray(dlu.local_to_numpy().T)).contiguous()
    if P == 1:
        parts = [loc]
    else:
        parts = [None] * P
        dist.all_gather_object(parts, loc.numpy(), group=dlu.group)
        parts = [torch.from_numpy(p) for p in parts]
    if rank != 0:
        return None
    full = np.zeros((dlu.n, dlu.n), dtype=np.float64, order="F")
    for r in range(P):
        cols = dlu.map.global_cols(r)
        if cols.size:
            full[:, cols] = parts[r].numpy().T
    return full
