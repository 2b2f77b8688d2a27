"""Regenerates tests/golden/*.npz by running the UNMODIFIED reference package (`mla`, imported
read-only from /root/reference/pkg/src).  Run in the build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference is Python+numba and cannot travel to the GPU box; these vectors are the pin that
tests/test_oracle_golden.py holds the C oracle to (bit for bit) and that the GPU tests reuse.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import mla  # noqa: E402  (the reference)
import mla.lu as mla_lu  # noqa: E402
from mla import (BlockConfig, CacheConfig, Policy, WorkerPool, alloc_matrix, fill_random,  # noqa: E402
                 gemm_malleable, laswp, lu_blk_ll, lu_blk_rl, lu_la, lu_unb, trsm_llu)

import cases  # noqa: E402
from paper_1611_06365_b200.workloads import make_matrix  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(a).tobytes(order="F")).hexdigest()


def gen(m, n, seed):
    return cases.uniform_pm1(fill_random, m, n, seed)


class TripFlag:
    """Deterministic stand-in for ru_done: set from poll number `trip` on (test_lu.py:149-156)."""

    def __init__(self, trip):
        self.trip, self.polls = trip, 0

    def is_set(self):
        self.polls += 1
        return self.trip > 0 and self.polls >= self.trip

    def set(self):
        pass


def cache(k_c):
    return CacheConfig(m_c=16, k_c=k_c, n_c=32, m_r=4, n_r=2) if k_c != 256 else CacheConfig()


def main():
    out = {}
    # fill_random itself (ld-independence included)
    a = alloc_matrix(7, 5, ld=9)
    fill_random(a, 3)
    out["fill_7x5_seed3"] = np.array(a)

    for c in cases.UNB:
        a = gen(c["m"], c["n"], c["seed"])
        r = lu_unb(a)
        out[c["name"] + "/lu"], out[c["name"] + "/ipiv"] = np.array(a), r.ipiv.ipiv

    for c in cases.LL:
        a = gen(c["m"], c["n"], c["seed"])
        stop = TripFlag(c["stop_trip"]) if c["stop_trip"] else None
        r = lu_blk_ll(a, c["b"], stop=stop, cfg=cache(c["k_c"]))
        out[c["name"] + "/lu"], out[c["name"] + "/ipiv"] = np.array(a), r.ipiv.ipiv
        out[c["name"] + "/cols"] = np.array([r.cols_factored])

    for c in cases.RL:
        a = gen(c["m"], c["n"], c["seed"])
        r = lu_blk_rl(a, c["b"], inner_b=c["inner_b"])
        out[c["name"] + "/lu"], out[c["name"] + "/ipiv"] = np.array(a), r.ipiv.ipiv

    with WorkerPool(4) as pool:
        for c in cases.LA:
            a = gen(c["m"], c["n"], c["seed"])
            r = lu_la(a, Policy(c["variant"], BlockConfig(c["b_o"], c["b_i"]), t_pf=1), pool,
                      cfg=cache(c["k_c"]))
            out[c["name"] + "/lu"], out[c["name"] + "/ipiv"] = np.array(a), r.ipiv.ipiv

        # ET with an injected, deterministic cut schedule: the reference's own lu_la(lu_et) runs,
        # only the panel's stop flag is replaced (per iteration) by a TripFlag.
        orig_ll = mla_lu.lu_blk_ll
        for c in cases.LA_ET:
            calls = {"it": -1, "widths": []}
            flags = {}

            def patched(a_, b_, ipiv=None, stop=None, team=None, cfg=None, _c=c, _calls=calls,
                        _flags=flags):
                if stop is None:
                    res = orig_ll(a_, b_, ipiv=ipiv, stop=None, team=team, cfg=cfg)
                else:
                    # one shared TripFlag per outer iteration (all PF workers poll collectively
                    # through team.collective, so exactly one poll per block happens)
                    key = id(stop)
                    if key not in _flags:
                        _calls["it"] += 1
                        sched = _c["sched"]
                        trip = sched[_calls["it"]] if _calls["it"] < len(sched) else 0
                        _flags[key] = (stop, TripFlag(trip))  # holding `stop` pins its id
                    res = orig_ll(a_, b_, ipiv=ipiv, stop=_flags[key][1], team=team, cfg=cfg)
                return res

            mla_lu.lu_blk_ll = patched
            try:
                a = gen(c["m"], c["n"], c["seed"])
                r = lu_la(a, Policy("lu_et", BlockConfig(c["b_o"], c["b_i"]), t_pf=1), pool,
                          cfg=cache(c["k_c"]))
            finally:
                mla_lu.lu_blk_ll = orig_ll
            out[c["name"] + "/lu"], out[c["name"] + "/ipiv"] = np.array(a), r.ipiv.ipiv
            out[c["name"] + "/et_widths"] = np.array(r.et_widths, dtype=np.int64)
            out[c["name"] + "/et_events"] = np.array([r.et_events])
            print(c["name"], "et_events", r.et_events, "widths", r.et_widths)

        for c in cases.BIG:
            a = np.asfortranarray(make_matrix(c["dist"], c["n"], c["seed"]))
            r = lu_la(a, Policy("lu", BlockConfig(c["b_o"], c["b_i"]), t_pf=1), pool)
            out[c["name"] + "/ipiv"] = r.ipiv.ipiv.astype(np.int32)
            out[c["name"] + "/sha"] = np.frombuffer(bytes.fromhex(sha(a)), dtype=np.uint8)
            out[c["name"] + "/diag"] = np.array(np.diag(a))
            print(c["name"], "done", sha(a)[:16])

    for c in cases.GEMM:
        a = gen(c["m"], c["k"], c["seed"])
        b = gen(c["k"], c["n"], c["seed"] + 100)
        cc = gen(c["m"], c["n"], c["seed"] + 200)
        gemm_malleable(cc, a, b, c["alpha"], c["beta"], cfg=cache(c["k_c"]))
        out[c["name"] + "/c"] = np.array(cc)

    for c in cases.TRSM:
        low = gen(c["w"], c["w"], c["seed"])
        x = gen(c["w"], c["c"], c["seed"] + 100)
        trsm_llu(low, x)
        out[c["name"] + "/x"] = np.array(x)

    for c in cases.LASWP:
        a = gen(c["rows"], c["cols"], c["seed"])
        laswp(a, np.array(c["ipiv"], dtype=np.int64))
        out[c["name"] + "/fwd"] = np.array(a)
        laswp(a, np.array(c["ipiv"], dtype=np.int64), reverse=True)
        out[c["name"] + "/back"] = np.array(a)

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)
    print("wrote", len(out), "arrays; reference version", mla.__version__)


if __name__ == "__main__":
    main()
