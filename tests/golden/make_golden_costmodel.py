"""Generates tests/golden/golden_costmodel.json from the reference's costmodel (run in the build
container, where /root/reference exists):  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_costmodel.py"""
import json, os
from mla import costmodel as cm

out = {"lu": [], "panel_total": [], "ll": [], "rl": [], "iter": [], "share": []}
for m, n in [(1, 1), (7, 5), (2048, 2048), (4096, 1000), (32768, 32768)]:
    out["lu"].append([m, n, cm.flops_lu(m, n)])
for n, b in [(2048, 256), (10000, 256), (32768, 512)]:
    out["panel_total"].append([n, b, cm.flops_panel_total(n, b)])
for m, n, k in [(100, 100, 0), (100, 100, 37), (512, 256, 256), (8192, 8192, 1024)]:
    out["ll"].append([m, n, k, cm.flops_ll_partial(m, n, k)])
    out["rl"].append([m, n, k, cm.flops_rl_partial(m, n, k)])
for m, n, b in [(5, 5, 2), (64, 48, 16), (2048, 2048, 256), (1000, 777, 100), (32768, 32768, 768)]:
    out["iter"].append([m, n, b, cm.iteration_flops(m, n, b)])
for n, b, f in [(10000, 256, 0.5), (10000, 256, 0.0), (10000, 256, 1.0), (2048, 256, 0.3), (1000, 96, 0.77)]:
    out["share"].append([n, b, f, cm.cumulative_flop_share(n, b, f)])
with open(os.path.join(os.path.dirname(__file__), "golden_costmodel.json"), "w") as f:
    json.dump(out, f)
