"""Write profiles/r02_summary.md from the committed round-2 bench lines
(profiles/r02_bench*.json), the ncu launch list (profiles/r02_launches_bench.csv)
and the ncu --set full findings recorded below the marker (kept verbatim)."""
import collections
import csv
import json
import os

P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles") + "/"
MARK = "## ncu --set full captures (round 2)"


def load(f):
    return json.loads(open(P + f).read().strip().splitlines()[-1])


r1 = {c: load(f) for c, f in [("cfg2", "r01_bench.json"), ("cfg3", "r01_bench_cfg3.json"),
                              ("cfg4", "r01_bench_cfg4.json"), ("cfg5", "r01_bench_cfg5.json"),
                              ("adv32", "r01_bench_adv32.json"), ("rrqr cfg2", "r01_bench_rrqr_cfg2.json")]}
r2 = {c: load(f) for c, f in [("cfg2", "r02_bench.json"), ("cfg3", "r02_bench_cfg3.json"),
                              ("cfg4", "r02_bench_cfg4.json"), ("cfg5", "r02_bench_cfg5.json"),
                              ("adv32", "r02_bench_adv32.json"), ("rrqr cfg2", "r02_bench_rrqr_cfg2.json")]}
d = r2["cfg2"]
cb = d["cpu_baseline"]
out = ["# Round 2 profile summary (1 x B200)\n",
       "Commands: `tools/r02_profile_cmd.sh` (bench lines `r02_bench*.json`, the ncu launch list, the ncu\n"
       "captures).  Regenerate this head with `python tools/profile_summary_r02.py`.\n",
       f"Headline (cfg2, 2D Poisson 256^2, n = 65,536, eps = 1e-3): factorization {d['value']/1e6:.3f} M unknowns/s\n"
       f"({d['factor_ms']:.2f} ms / re-factorization), PCG to 1e-10 in {d['krylov_iters']} iterations "
       f"{d['krylov_ms']:.2f} ms; e2e (C ABI, pinned host buffers, copies inside) {d['e2e']['value']/1e6:.3f} M "
       f"unknowns/s; first factorization of the process {d['first_factor_ms']:.1f} ms (with one-time context / "
       f"module-load costs), of a fresh handle in the warm process {d['first_factor_fresh_handle_ms']:.1f} ms (analyze "
       f"{1e3*d['analyze_s']:.1f} ms host); re-factorization with changed values (ranks change) "
       f"{d['refactor_new_values']['ms_first']:.1f} ms, then {d['refactor_new_values']['ms_second']:.1f} ms; "
       f"paper residual (Eq. GMRES_residual) at the final iterate {d['paper_residual']:.2e}.\n",
       f"CPU baseline: the C++ oracle, {cb['cores']} threads of `{cb['cpu_model']}`: {cb['value']/1e3:.1f} K "
       f"unknowns/s ({cb['factor_s']:.2f} s); 1 thread {cb['single_thread']['value']/1e3:.1f} K "
       f"({cb['single_thread']['factor_s']:.2f} s).  Clocks {d['clocks']}.\n",
       "| workload | n | factor ms r01 -> r02 | unknowns/s r02 | model TFLOP/s | Krylov ms (it) | first factor ms (process / fresh handle) | dominant class, roofline frac |",
       "|---|---|---|---|---|---|---|---|"]
for c in r2:
    a, b = r1[c], r2[c]
    out.append(f"| {c} | {b['config']['n']:,} | {a['factor_ms']:.1f} -> {b['factor_ms']:.1f} | {b['value']/1e6:.2f} M | "
               f"{b['tflops_model']:.2f} | {b['krylov_ms']:.1f} ({b['krylov_iters']}) | {b['first_factor_ms']:.0f} / {b.get('first_factor_fresh_handle_ms') or float('nan'):.0f} | "
               f"{b['roofline']['kernel'].replace(' | ', ' or ')}, {b['roofline']['frac']:.3f} |")
o4 = d.get("other_configs", {}).get("cfg4")
if o4:
    out.append(f"\ncfg4 measured inside the default cfg2 run (`other_configs`): factor {o4['factor_ms']:.1f} ms "
               f"({o4['value']/1e6:.2f} M unknowns/s), PCG {o4['krylov_iters']} it {o4['krylov_ms']:.1f} ms, "
               f"first factor {o4['first_factor_ms']:.0f} ms.\n")
out.append("## Per-kernel-class time, cfg2 (CUDA events on the library stream, last warm-up step)\n")
out.append("| class | kernels | ms r01 -> r02 | launches | alg. GFLOP | alg. TFLOP/s |\n|---|---|---|---|---|---|")
k1 = r1["cfg2"]["kernels_warmup_step"]
for k, v in sorted(d["kernels_warmup_step"].items(), key=lambda kv: -kv[1]["ms"]):
    tf = v["alg_flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] > 0 else 0
    old = k1.get(k, {}).get("ms", 0.0)
    out.append(f"| {k} | {v['kernel'].replace(' | ', ' or ')} | {old:.3f} -> {v['ms']:.3f} | {v['launches']} | {v['alg_flops']/1e9:.2f} | {tf:.2f} |")
rows = list(csv.reader(open(P + "r02_launches_bench.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("lorasp::", "")
    unit = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ix["Metric Unit"]], 1e-6)
    agg[name][0] += 1
    agg[name][1] += float(r[ix["Metric Value"]].replace(",", "")) * unit
tot = sum(v[1] for v in agg.values())
out.append("\n## ncu launch list, cfg2 (`ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 "
           "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --extra none`; serialised, cold "
           "cache, so shares not absolute times are comparable with the bench line)\n\n"
           "Raw CSV: `r02_launches_bench.csv`.\n\n| kernel | launches | total ms (ncu) | share |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"| {k} | {v[0]} | {v[1]:.3f} | {100*v[1]/tot:.1f}% |")
out.append(f"\nTotal over the listed launches: {tot:.2f} ms.\n")
path = P + "r02_summary.md"
tail = ""
if os.path.exists(path):
    old = open(path).read()
    if MARK in old:
        tail = old[old.index(MARK):]
open(path, "w").write("\n".join(out) + "\n" + tail)
print("ok")
