"""The GPU stand-in for the reference's WorkerPool (pool.py:226-374).

The reference's pool is a set of CPU threads dispatched as one or two teams; here the "workers" are
the SMs of one B200 and the dispatch happens inside the persistent kernel, so the pool only owns the
library handle (workspace, flags, queues) and the default split.  `t` is the number of SMs, `t_pf`
the default size of the panel team, `t_pf_max` how far the panel team may grow between iterations
when the panel is the critical path (0 = fixed split, the reference's behaviour; the pivots do not
depend on it).  CompletionFlag is a device word (pool.py:28-49).
"""
from __future__ import annotations

import ctypes

import torch

from . import _capi


class SmPool:
    """One per device.  Context manager like the reference's WorkerPool."""

    def __init__(self, device: int | None = None, t_pf: int = 32, t_pf_max: int | None = None) -> None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1611_06365_b200 needs a CUDA device; there is no CPU fallback")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._h = ctypes.c_void_p()
        _capi.check(_capi.lib().mla_create(self.device, ctypes.byref(self._h)), None, "mla_create")
        self.t = int(_capi.lib().mla_num_sms(self._h))
        self.t_pf = max(1, min(int(t_pf), self.t - 1))
        # default 0: fixed split (measured on B200: growing the team in the panel-bound tail only moves
        # time from the panel to the update, the total is unchanged -- DESIGN.md)
        self._t_pf_max = None
        self._closed = False
        self.t_pf_max = 0 if t_pf_max is None else t_pf_max

    @property
    def t_pf_max(self) -> int:
        return self._t_pf_max

    @t_pf_max.setter
    def t_pf_max(self, value: int) -> None:
        value = int(value)
        if value < 0:
            raise ValueError("t_pf_max must be >= 0")
        _capi.check(_capi.lib().mla_set_panel_sms_max(self.handle, min(value, self.t - 1)), self._h,
                    "mla_set_panel_sms_max")
        self._t_pf_max = min(value, self.t - 1)

    def set_update_sms(self, ctas: int) -> None:
        """SMs that apply_panel launches on (0 = all): a multi-GPU driver keeps a few free for the
        communication kernels and for the next panel running beside the update."""
        _capi.check(_capi.lib().mla_set_update_sms(self.handle, int(ctas)), self._h, "mla_set_update_sms")

    @property
    def handle(self):
        if self._closed:
            raise RuntimeError("pool is shut down")
        return self._h

    def shutdown(self) -> None:
        if not self._closed:
            _capi.lib().mla_destroy(self._h)
            self._closed = True

    def __enter__(self) -> "SmPool":
        return self

    def __exit__(self, *exc) -> None:
        self.shutdown()


WorkerPool = SmPool  # the reference's name

_default_pools: dict[int, SmPool] = {}


def default_pool(device: int | None = None) -> SmPool:
    dev = torch.cuda.current_device() if device is None else int(device)
    p = _default_pools.get(dev)
    if p is None or p._closed:
        p = SmPool(dev)
        _default_pools[dev] = p
    return p


class CompletionFlag:
    """One-shot done signal living in device memory (reference pool.py:28-49)."""

    def __init__(self, writer: str | None = None, device=None) -> None:
        self.writer = writer
        self._word = torch.zeros(1, dtype=torch.int32, device=device or "cuda")

    def is_set(self) -> bool:
        return bool(self._word.item() != 0)

    def set(self) -> None:
        self._word.fill_(1)

    @property
    def ptr(self) -> int:
        return self._word.data_ptr()


def signal_complete(flag: CompletionFlag) -> None:
    flag.set()
