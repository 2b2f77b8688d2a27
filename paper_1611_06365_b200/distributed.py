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

Per GPU the step is the paper's look-ahead + worker sharing + early termination (DistLU docstring); the
panel schedule is lu_la's (lu.py:314-326) with one extra rule -- a panel never crosses a column-block
boundary -- so the CPU oracle's lu_la(b_outer, b_inner, et_sched, clamp=b_outer) replays any run and is
the parity reference for the assembled matrix.

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


class PanelSchedule:
    """Panel-width bookkeeping of lu_la (lu.py:224-241, 314-326) plus the one rule the block-cyclic layout
    adds: a panel never crosses a multiple of `clamp` columns (the column block is the unit of ownership,
    so a panel always lives on ONE rank).  After an ET cut the leftover columns of the block become the
    next panel(s) of the same owner; b_target shrinks to max(b_i, k_new) and regrows by doubling."""

    def __init__(self, n: int, b_outer: int, b_inner: int, clamp: int = 0):
        self.n, self.b_o, self.b_i, self.clamp = n, b_outer, b_inner, clamp
        self.q0 = self.q1 = self.pend = 0
        self.b_target = b_outer
        self.widths: list[int] = []
        self.et_events = 0

    def _clamped(self, q: int, w: int) -> int:
        w = min(w, self.n - q)
        if self.clamp > 0:
            w = min(w, self.clamp - q % self.clamp)
        return w

    def first_width(self) -> int:
        return self._clamped(0, self.b_o)

    def start(self, w: int, k_new: int) -> None:           # the prologue panel is never cut
        self.q0, self.q1, self.pend = 0, k_new, w
        self.widths.append(k_new)

    def next_width(self) -> int:
        return self._clamped(self.q1, self.b_target)

    def advance(self, w: int, k_new: int) -> None:          # lu.py:318-326
        if k_new < w:
            self.et_events += 1
            self.b_target = max(self.b_i, k_new)
        else:
            self.b_target = min(self.b_o, 2 * self.b_target)
        self.pend = self.q1 + w
        self.q0, self.q1 = self.q1, self.q1 + k_new
        self.widths.append(k_new)


def et_schedule_from_widths(widths, n: int, b_o: int, b_i: int, clamp: int = 0) -> list[int]:
    """Per-iteration 'trip poll' list (0 = not cut) that makes the CPU oracle's lu_la(clamp=...) replay the
    width sequence a run produced."""
    out: list[int] = []
    if not widths:
        return out
    s = PanelSchedule(n, b_o, b_i, clamp)
    s.start(s.first_width(), widths[0])
    for k_new in widths[1:]:
        w = s.next_width()
        out.append(k_new // b_i if k_new < w else 0)
        s.advance(w, k_new)
    return out


class CudaOps:
    """Operator table bound to libmla_b200.so (the product path): every method is stream-ordered on the
    current stream and returns without synchronising."""

    crout = True      # a cut panel leaves its leftover columns with the interchanges AND their U rows

    def __init__(self, pool=None):
        from . import kernels, lu, matrix
        self._k, self._lu, self._m = kernels, lu, matrix
        self.pool = pool
        self.side_pool = None

    def alloc(self, rows, cols, device):
        return self._m.alloc_matrix(rows, cols, device=device)

    def fill(self, a, seed, col0, total_rows, scale, shift, row_scale):
        self._m.fill_random(a, seed, scale, shift, row_scale=row_scale, col0=col0, total_rows=total_rows,
                            pool=self.pool)

    # one side handle per device (second set of control words / exchange slots for the look-ahead panel
    # that runs beside the update), shared by all drivers of this process
    _side_pools: dict = {}

    def bind(self, device):
        from .pool import SmPool, default_pool
        self.pool = self.pool or default_pool(device.index)
        sp = CudaOps._side_pools.get(device.index)
        if sp is None or sp._closed:
            sp = SmPool(device.index)
            CudaOps._side_pools[device.index] = sp
        self.side_pool = sp
        return self.pool.t

    def panel(self, a, b_inner, piv_out, sing_accum, side=False, team_sms=0, stop=None):
        """Stream-ordered panel factorization; pivots -> piv_out (device int32), width -> device record."""
        self._lu.lu_blk_ll_async(a, b_inner, self.side_pool if side else self.pool, team_sms, sing_accum, stop, piv_out)

    def pack(self, panel, piv, out, side=False):
        self._k.pack_panel(panel, piv, out, pool=self.side_pool if side else self.pool)

    def apply_prepare(self, panel, piv, w, side=False):
        self._k.apply_panel_prepare(panel, piv, w, pool=self.side_pool if side else self.pool)

    def apply_launch(self, panel, w, target, ctas=0, skip_cols=0, left=None, side=False):
        self._k.apply_panel_launch(panel, w, target, ctas, pool=self.side_pool if side else self.pool,
                                   skip_cols=skip_cols, left=left)

    def step_flag(self):
        return self._k.step_flag(self.pool)


class DistLU:
    """One rank's share of a block-cyclic LU.  `group` = process group (default WORLD).

    variant (the paper's ladder, per GPU):
      "lu"     update, then the next panel on every SM (no overlap);
      "lu_la"  look-ahead: the owner of the next panel applies the current panel to that panel's columns
               and factors it on `panel_sms` SMs (side stream, side handle) WHILE the other SMs apply the
               current panel to the rest of the owned columns; its broadcast starts as soon as it is packed;
      "lu_mb"  + worker sharing: the panel SMs then join the update's work queue (second launch);
      "lu_et"  + early termination: the update's last work item publishes the step flag, the panel polls it
               after every inner block and stops there; the factored width travels in the broadcast header,
               the leftover columns become the next panel of the same owner (lu.py:177-179, 309-326).
    On a CPU operator table (tests) every variant runs the same sequential order; `et_sched` injects cuts
    deterministically (entry it-1 = number of inner blocks after which iteration it's panel stops)."""

    VARIANTS = ("lu", "lu_la", "lu_mb", "lu_et")

    def __init__(self, n, b_outer, b_inner, cfg, device, variant="lu_et", pool=None, ops=None, group=None,
                 rank=None, world=None, panel_sms=32, comm_sms=8, storage=None, et_sched=None, comm_always=False):
        if variant not in self.VARIANTS:
            raise ValueError(f"unknown variant {variant!r}; expected one of {self.VARIANTS}")
        if b_inner < 1 or b_outer < b_inner:
            raise ValueError("need b_outer >= b_inner >= 1")
        self.n, self.b, self.b_inner, self.cfg = n, b_outer, b_inner, cfg
        self.variant = variant
        self.device = torch.device(device)
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.P = dist.get_world_size(group) if world is None else world
        self.map = BlockCyclic(n, b_outer, self.P)
        self.cuda = self.device.type == "cuda"
        self.ops = ops or CudaOps(pool)
        self.et_sched = list(et_sched) if et_sched is not None else None
        # comm_always: issue the broadcasts (and use the communication stream) even with a single rank -- a
        # 1-rank NCCL communicator exercises the whole collective path (stream handoff, buffer events) on one GPU
        self.comm_always = bool(comm_always) and dist.is_available() and dist.is_initialized()
        self.nloc = self.map.local_cols(self.rank)
        # `storage`: factor the caller's (n x nloc, column-major) tensor in place instead of an own buffer
        self.a = storage if storage is not None else self.ops.alloc(n, max(self.nloc, 1), self.device)[:, :self.nloc]
        self.a0 = None
        self.ipiv = np.zeros(n, dtype=np.int64)
        self.singular = False
        self.widths: tuple = ()
        self.et_events = 0
        self.host_waits = 0            # times factor() blocked the host on a device event
        self.launches_per_factor = 0
        self.comm_stream = torch.cuda.Stream(self.device) if self.cuda else None
        if self.cuda:
            self.sms = self.ops.bind(self.device)
            self.overlap = variant != "lu" and self.sms >= 4
            self.panel_sms = max(1, min(int(panel_sms), self.sms - 2))
            self.comm_sms = max(0, min(int(comm_sms), self.sms - self.panel_sms - 1)) if self.P > 1 else 0
            self.panel_stream = torch.cuda.Stream(self.device)
            self._sing_dev = torch.zeros(1, dtype=torch.int32, device=self.device)
            self._piv_next = torch.zeros(b_outer, dtype=torch.int32, device=self.device)
            self._hdr_host = [torch.zeros(4, dtype=torch.int32).pin_memory() for _ in range(2)]
        else:
            self.overlap = False
        # two broadcast buffers (double buffering: panel it+1 is in flight while panel it is consumed);
        # layout of one: [int32 x 4 header][int32 pivots, padded][rows x w doubles]  (mla_pack_panel)
        cap = self._hdr_doubles(b_outer) + n * b_outer
        self.bufs = [torch.zeros(cap, dtype=torch.float64, device=self.device) for _ in range(2)]
        self._buf_free = [None, None]     # event: last reader of the buffer has been enqueued and finished

    # ---- data ---------------------------------------------------------------------------------
    def generate(self):
        """Fill the owned column blocks of the config's matrix (uniform configs: on the device, each
        block independently through the counter-based stream; normal configs: host generator -- numpy's
        stream cannot be entered mid-way, so every rank draws the full matrix and keeps its columns)."""
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

    # ---- layout helpers --------------------------------------------------------------------------
    def local_lt(self, c: int) -> int:
        """Number of this rank's columns whose global index is < c."""
        j, r = divmod(min(c, self.n), self.b)
        cnt = max(0, (j - self.rank + self.P - 1) // self.P) * self.b
        if j % self.P == self.rank and j < self.map.nblocks:
            cnt += r
        return min(cnt, self.nloc)

    def _views(self, which: int, rows: int, w: int):
        """(int32 header view, int32 pivot view, rows x w column-major panel view) of buffer `which`."""
        buf = self.bufs[which]
        hd = self._hdr_doubles(w)
        i32 = buf[:hd].view(torch.int32)
        panel = buf[hd: hd + rows * w].view(w, rows).t()
        return i32[:4], i32[4:4 + w], panel

    @staticmethod
    def _hdr_doubles(w: int) -> int:
        """Header + pivots of a packed panel of scheduled width w, in doubles (mla_pack_panel's layout:
        the panel's doubles start right behind them, 16-byte aligned)."""
        return (4 + ((w + 3) & ~3)) // 2

    def _count(self, rows: int, w: int) -> int:
        return self._hdr_doubles(w) + rows * w

    # ---- producing a panel (owner) ------------------------------------------------------------------
    def _produce_host(self, which, q, w, trip):
        """CPU operator table: factor a[q:, local cols of [q, q+w)] and pack it."""
        lo = self.local_lt(q)
        view = self.a[q:, lo:lo + w]
        piv, sing, k_new = self.ops.panel(view, self.b_inner, trip)
        hdr, pv, panel = self._views(which, self.n - q, w)
        hdr.copy_(torch.tensor([k_new, int(bool(sing)), w, self.n - q], dtype=torch.int32))
        pv[:k_new].copy_(torch.as_tensor(piv[:k_new]).to(torch.int32))
        panel.copy_(view)
        self.launches_per_factor += 1

    # ---- consuming a panel ----------------------------------------------------------------------------
    def _apply_host(self, panel, piv, kk, q0, col_lo, col_hi, pend_lo):
        """Operator chain laswp -> trsm -> gemm (lu.py:251-253, 280-281, 289, 306-308) on local columns
        [col_lo, col_hi); columns below pend_lo are leftovers of a cut panel: they already carry the
        interchanges (lu.py:178, 247-255) and -- Crout-order panels only -- their U rows."""
        if col_hi <= col_lo:
            return
        sw_lo = max(col_lo, pend_lo)
        tr_lo = sw_lo if getattr(self.ops, "crout", False) else col_lo
        if col_hi > sw_lo:
            self.ops.laswp(self.a[q0:, sw_lo:col_hi], piv)
        if col_hi > tr_lo:
            self.ops.trsm(panel[:kk, :kk], self.a[q0:q0 + kk, tr_lo:col_hi])
        if self.n - q0 - kk > 0:
            self.ops.gemm(self.a[q0 + kk:, col_lo:col_hi], panel[kk:, :kk], self.a[q0:q0 + kk, col_lo:col_hi])
        self.launches_per_factor += 3

    # ---- exchange -------------------------------------------------------------------------------------
    def _bcast(self, which, q, w):
        if self.P == 1 and not self.comm_always:
            return
        src = self.map.owner(q // self.b)
        if self.group is not None:
            src = dist.get_global_rank(self.group, src)
        dist.broadcast(self.bufs[which][: self._count(self.n - q, w)], src=src, group=self.group)

    def _exchange(self, which, q, w, after, need_host_width):
        """Broadcast panel buffer `which` (owner: once `after` -- the stream that packed it -- is there;
        receivers: once the buffer's last reader is done) and, when the width is dynamic (ET), bring the
        header to the host.  Returns (factored width, singular or None)."""
        if not self.cuda:
            self._bcast(which, q, w)
            hdr = self._views(which, self.n - q, w)[0]
            return int(hdr[0]), bool(int(hdr[1]))
        use_comm = self.P > 1 or self.comm_always
        stream = self.comm_stream if use_comm else after
        if use_comm:
            if after is not None:                         # owner: the stream that packed the buffer
                self.comm_stream.wait_stream(after)
            if self._buf_free[which] is not None:
                self.comm_stream.wait_event(self._buf_free[which])
            with torch.cuda.stream(self.comm_stream):
                self._bcast(which, q, w)
        if not need_host_width:
            return w, None
        with torch.cuda.stream(stream):
            self._hdr_host[which].copy_(self._views(which, self.n - q, w)[0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        ev.synchronize()          # waits for the panel / its broadcast only -- the update stream keeps running
        self.host_waits += 1
        return int(self._hdr_host[which][0]), bool(int(self._hdr_host[which][1]))

    # ---- the factorization -----------------------------------------------------------------------
    def factor(self):
        """P A = L U on the distributed matrix; returns the global pivot vector (host int64)."""
        n, b, m = self.n, self.b, self.map
        self.launches_per_factor = 0
        self.host_waits = 0
        self.singular = False
        sched = PanelSchedule(n, b, self.b_inner, clamp=b)
        self._piv_dev = torch.zeros(n, dtype=torch.int32, device=self.device)
        et_dev = self.cuda and self.variant == "lu_et" and self.overlap
        if self.cuda:
            self._sing_dev.zero_()
            main = torch.cuda.current_stream(self.device)
            self._buf_free = [None, None]
        if n == 0:
            self.ipiv = np.zeros(0, dtype=np.int64)
            return self.ipiv
        # ---- prologue: panel 0, never cut (lu.py:224-241) ------------------------------------------
        cur, w = 0, sched.first_width()
        if m.owner(0) == self.rank:
            if self.cuda:
                view = self.a[:, :w]
                self.ops.panel(view, self.b_inner, self._piv_next, self._sing_dev)
                self.ops.pack(view, self._piv_next, self.bufs[0])
                self.launches_per_factor += 2
            else:
                self._produce_host(0, 0, w, 0)
        k_new, sing = self._exchange(0, 0, w, main if self.cuda else None, False) if self.cuda else \
            self._exchange(0, 0, w, None, True)
        if sing:
            self.singular = True
        sched.start(w, k_new)
        w_cur = w
        it = 0
        while True:
            it += 1
            q0, q1, pend = sched.q0, sched.q1, sched.pend
            kk, rows = q1 - q0, n - q0
            if self.cuda and (self.P > 1 or self.comm_always):
                main.wait_stream(self.comm_stream)        # panel `cur` has arrived
            hdr, piv, panel = self._views(cur, rows, w_cur)
            self._piv_dev[q0:q1] = piv[:kk] + q0
            if self.cuda and not et_dev:
                self._sing_dev |= hdr[1:2]                # stays on the device until the end
            left_hi = self.local_lt(q0)
            if q1 >= n:
                # ---- final_sync (lu.py:329-332): last panel's interchanges for the columns to its left ----
                if left_hi > 0:
                    if self.cuda:
                        self.ops.apply_prepare(panel, piv, kk)
                        self.ops.apply_launch(panel, kk, None, left=self.a[q0:, :left_hi])
                        self.launches_per_factor += 2
                    else:
                        self.ops.laswp(self.a[q0:, :left_hi], piv[:kk])
                break
            w = sched.next_width()
            own_next = m.owner(q1 // b) == self.rank
            nxt = 1 - cur
            lo1 = self.local_lt(q1)                        # first local column with global index >= q1
            pend_lo = self.local_lt(pend)
            trip = self.et_sched[it - 1] if (self.et_sched is not None and it - 1 < len(self.et_sched)) else 0
            if not self.cuda:
                # ---- host operator table: the serial order of lu.py:259-269 ------------------------------
                self._apply_host(panel, piv[:kk], kk, q0, lo1, self.nloc, pend_lo)
                if left_hi > 0:
                    self.ops.laswp(self.a[q0:, :left_hi], piv[:kk])
                if own_next:
                    self._produce_host(nxt, q1, w, trip)
                k_new, sing = self._exchange(nxt, q1, w, None, True)
            elif own_next and self.overlap:
                # ---- look-ahead on the device ------------------------------------------------------------
                side = self.panel_stream
                nview = self.a[q1:, lo1:lo1 + w]
                rest_lo = lo1 + w
                have_main = self.nloc > rest_lo or left_hi > 0
                side.wait_stream(main)        # update it-1 is complete: it touched these columns and read bufs[nxt]
                stop = None
                ready = None
                if have_main:
                    self.ops.pool.set_update_sms(0)
                    self.ops.apply_prepare(panel, piv, kk)
                    ready = torch.cuda.Event()
                    ready.record(main)
                    self.ops.apply_launch(panel, kk, self.a[q0:, rest_lo:self.nloc],
                                          ctas=self.sms - self.panel_sms - self.comm_sms,
                                          skip_cols=max(0, pend_lo - rest_lo), left=self.a[q0:, :left_hi])
                    self.launches_per_factor += 2
                    if et_dev:
                        stop = self.ops.step_flag()
                with torch.cuda.stream(side):
                    self.ops.side_pool.set_update_sms(self.panel_sms)
                    self.ops.apply_prepare(panel, piv, kk, side=True)
                    self.ops.apply_launch(panel, kk, self.a[q0:, lo1:lo1 + w], skip_cols=max(0, pend_lo - lo1), side=True)
                    self.ops.panel(nview, self.b_inner, self._piv_next, self._sing_dev, side=True,
                                   team_sms=self.panel_sms, stop=stop)
                    self.ops.pack(nview, self._piv_next, self.bufs[nxt], side=True)
                    self.launches_per_factor += 4
                    if have_main and self.variant in ("lu_mb", "lu_et"):
                        # worker sharing (pool.py:377-414): the quiesced panel SMs join the update's queue
                        side.wait_event(ready)
                        self.ops.apply_launch(panel, kk, self.a[q0:, rest_lo:self.nloc], ctas=self.panel_sms,
                                              skip_cols=max(0, pend_lo - rest_lo), left=self.a[q0:, :left_hi])
                        self.launches_per_factor += 1
                k_new, sing = self._exchange(nxt, q1, w, side, et_dev)
                main.wait_stream(side)
            else:
                # ---- no look-ahead overlap on this rank: update, then (owner) the panel on every SM --------
                if self.nloc > lo1 or left_hi > 0:
                    self.ops.pool.set_update_sms(self.sms - self.comm_sms if self.P > 1 else 0)
                    self.ops.apply_prepare(panel, piv, kk)
                    self.ops.apply_launch(panel, kk, self.a[q0:, lo1:self.nloc], skip_cols=max(0, pend_lo - lo1),
                                          left=self.a[q0:, :left_hi])
                    self.launches_per_factor += 2
                if own_next:
                    nview = self.a[q1:, lo1:lo1 + w]
                    self.ops.panel(nview, self.b_inner, self._piv_next, self._sing_dev)
                    self.ops.pack(nview, self._piv_next, self.bufs[nxt])
                    self.launches_per_factor += 2
                # receivers post the broadcast at once: it must not wait for their own update
                k_new, sing = self._exchange(nxt, q1, w, main if (own_next or self.P == 1) else None, et_dev)
            if self.cuda:
                ev = torch.cuda.Event()
                ev.record(main)
                self._buf_free[cur] = ev                   # bufs[cur] may be overwritten once this is reached
            if sing:
                self.singular = True
            sched.advance(w, k_new)
            w_cur = w
            cur = nxt
        self.widths = tuple(sched.widths)
        self.et_events = sched.et_events
        if self.cuda:
            # leave the shared handles as they were found: every SM for whoever launches an update next
            self.ops.pool.set_update_sms(0)
            self.ops.side_pool.set_update_sms(0)
            self.singular |= bool(int(self._sing_dev.item()))
            self.ipiv = self._piv_dev.cpu().numpy().astype(np.int64)   # the only bulk device->host copy
        else:
            self.ipiv = self._piv_dev.numpy().astype(np.int64)
        return self.ipiv


def lu_streams(a: torch.Tensor, b_outer: int, b_inner: int, pool=None, panel_sms: int = 32, variant: str = "lu_et"):
    """Single-GPU LU of a square column-major matrix, in place, through THIS driver with P = 1: per outer
    iteration separately compiled kernels on two streams (update || look-ahead panel, worker sharing by a
    joining launch, early termination through the step flag) instead of the one persistent kernel behind
    lu_la.  Returns a LuResult like lu_la (widths = the factored panel widths; replayable on the oracle with
    clamp = b_outer).  Not exported from the package: lu_la is the single-GPU path; this one exercises the
    multi-GPU driver's per-GPU step on one GPU."""
    from .lu import LuResult
    from .matrix import PivotVector, check_colmajor
    m, n, _ = check_colmajor(a, "a")
    if m != n:
        raise ValueError("lu_streams: square matrices only")
    if n == 0:
        return LuResult(PivotVector(np.empty(0, dtype=np.int64)), 0, False)
    dlu = DistLU(n, b_outer, b_inner, None, a.device, variant=variant, pool=pool, rank=0, world=1,
                 panel_sms=panel_sms, storage=a)
    ipiv = dlu.factor()
    widths = dlu.widths
    cuts = []
    s = PanelSchedule(n, b_outer, b_inner, b_outer)
    s.start(s.first_width(), widths[0])
    for k_new in widths[1:]:
        w = s.next_width()
        if k_new < w:
            cuts.append(k_new)
        s.advance(w, k_new)
    return LuResult(PivotVector(ipiv, device=dlu._piv_dev), n, bool(dlu.singular), dlu.et_events, tuple(cuts), widths, 0)


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
