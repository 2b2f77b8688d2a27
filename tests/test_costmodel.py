"""Flop model vs values produced by the reference's costmodel (tests/golden/make_golden_costmodel.py);
the identities follow the reference's own tests (test_costmodel.py: telescoping, continuity)."""
import json
import os

import pytest

from paper_1611_06365_b200 import costmodel as cm

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_costmodel.json")))


def test_closed_forms_match_reference():
    for m, n, v in G["lu"]:
        assert cm.flops_lu(m, n) == v
    for n, b, v in G["panel_total"]:
        assert cm.flops_panel_total(n, b) == v
    for m, n, k, v in G["ll"]:
        assert cm.flops_ll_partial(m, n, k) == v
    for m, n, k, v in G["rl"]:
        assert cm.flops_rl_partial(m, n, k) == v


def test_iteration_flops_match_reference():
    for m, n, b, recs in G["iter"]:
        assert cm.iteration_flops(m, n, b) == recs


def test_share_matches_reference():
    for n, b, f, v in G["share"]:
        assert cm.cumulative_flop_share(n, b, f) == pytest.approx(v, rel=1e-14, abs=1e-15)


@pytest.mark.parametrize("m,n,b", [(2048, 2048, 256), (1000, 777, 100), (32768, 32768, 512)])
def test_iterations_telescope_to_total(m, n, b):
    total = sum(r["total"] for r in cm.iteration_flops(m, n, b))
    assert total == pytest.approx(cm.flops_lu(m, n), rel=1e-12)


def test_schedule_flops_is_width_independent_in_total():
    a = sum(r["total"] for r in cm.schedule_flops(4096, 4096, [512, 64, 128, 256] + [512] * 6 + [64]))
    assert a == pytest.approx(cm.flops_lu(4096, 4096), rel=1e-12)


def test_errors():
    with pytest.raises(ValueError):
        cm.iteration_flops(3, 4, 2)
    with pytest.raises(ValueError):
        cm.iteration_flops(4, 4, 0)
    with pytest.raises(ValueError):
        cm.flops_ll_partial(4, 4, 5)
    with pytest.raises(ValueError):
        cm.cumulative_flop_share(10, 2, 1.5)
    with pytest.raises(ValueError):
        cm.schedule_flops(8, 8, [4, 5])
