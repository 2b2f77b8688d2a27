"""profiles/<round>_results_table.md and <round>_launches_bench_n32768.txt from the bench JSON lines and the
ncu launch list that tools/profile_round.sh produced.  usage: python tools/results_table.py r01"""
import csv, glob, json, sys, collections

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for f in ["config1", "config2_variants", "config3", "config4_bsweep", "n32768", "n65536_1gpu"]:
    try:
        for l in open(f"profiles/{R}_bench_{f}.json"):
            if l.startswith("{"):
                rows.append(json.loads(l))
    except FileNotFoundError:
        pass
out = ["| workload | variant | sm_pf | ms | TFLOP/s | frac of 37.0 | backward err / (n eps) | ET events | panels | e2e GFLOP/s | CPU oracle GFLOP/s |",
       "|---|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    c = d["config"]
    be = d.get("backward_error_over_n_eps", "")
    out.append("| %s | %s | %s | %.3f | %.3f | %.3f | %s | %s | %s | %s | %s |" % (
        c["workload"], c.get("variant"), c.get("sm_pf"), d["ms_per_step"], d["value"] / 1e3, d["value"] / 1e3 / 37.0,
        ("%.4f" % be) if be != "" else "", d.get("run", c).get("et_events", ""), d.get("run", c).get("panels", ""),
        ("%.1f" % d["e2e"]["value"]) if d.get("e2e") else "", ("%.3f" % d["cpu_baseline"]["value"]) if d.get("cpu_baseline") else ""))
open(f"profiles/{R}_results_table.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))

rows = [r for r in csv.reader(l for l in open(f"profiles/{R}_launches_bench_n32768.csv") if l.startswith('"'))]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.OrderedDict()
per = []
for r in rows[1:]:
    name = r[ki].split("(")[0][:70]
    ns = float(r[vi])
    t = tot.setdefault(name, [0.0, 0])
    t[0] += ns; t[1] += 1
    if name.startswith("k_getrf"):
        per.append(ns / 1e6)
total = sum(v[0] for v in tot.values())
txt = ["# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e",
       "# (n=32768, b=512/64, lu_et, sm_pf 32; per-launch times are serialised/cold-cache: compare SHARES)",
       "# total device time %.1f ms over %d launches" % (total / 1e6, sum(v[1] for v in tot.values()))]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0]):
    txt.append("%10.2f ms  %5.1f%%  x%-4d %s" % (v[0] / 1e6, 100 * v[0] / total, v[1], k))
txt += ["", "# per-launch k_getrf durations (ms):"] + ["%.2f" % x for x in per]
open(f"profiles/{R}_launches_bench_n32768.txt", "w").write("\n".join(txt) + "\n")
print("\n".join(txt))

# launch list of the same command with the e2e leg on (mla_getrf_la_host: one persistent launch per window +
# the catch-up launches between them), if it was captured
import os
if os.path.exists(f"profiles/{R}_launches_bench_e2e.csv"):
    rows = [r for r in csv.reader(l for l in open(f"profiles/{R}_launches_bench_e2e.csv") if l.startswith('"'))]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0][:70]
        t = tot.setdefault(name, [0.0, 0])
        t[0] += float(r[vi]); t[1] += 1
    total = sum(v[0] for v in tot.values())
    txt = ["# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 1 --warmup 3 --no-cpu",
           "# (value leg: 4 k_getrf launches of the whole matrix; e2e leg: 6 calls of mla_getrf_la_host, each 4 windowed",
           "#  k_getrf launches + catch-up = k_laswp_* + k_diag_inv + k_apply_panel + k_gemm; serialised, cold cache: SHARES)",
           "# total device time %.1f ms over %d launches" % (total / 1e6, sum(v[1] for v in tot.values()))]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        txt.append("%10.2f ms  %5.1f%%  x%-4d %s" % (v[0] / 1e6, 100 * v[0] / total, v[1], k))
    open(f"profiles/{R}_launches_bench_e2e.txt", "w").write("\n".join(txt) + "\n")
    print("\n".join(txt))
