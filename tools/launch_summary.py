"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of tools/prof_step.py:
per-kernel total time, share, launches, average.  python tools/launch_summary.py in.csv out.txt
[header note] -- only the last step's launches are summarised when the run had 2 steps."""
import collections
import csv
import sys

src, dst = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
data = [r for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
# launches of the second step only: split at the second k_schur_coef launch of level 0
starts = [i for i, r in enumerate(data) if "k_schur_coef" in r[ix["Kernel Name"]]]
if len(starts) >= 2:
    n_lv = len(starts) // 2
    data = data[starts[n_lv]:]
agg = collections.defaultdict(lambda: [0.0, 0, ""])
for r in data:
    name = r[ix["Kernel Name"]]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    key = (name.split("(")[0], r[ix["Grid Size"]])
    agg[key][0] += us
    agg[key][1] += 1
tot = sum(a[0] for a in agg.values())
with open(dst, "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, tools/prof_step.py 2 (C4, batch 32)\n")
    f.write(f"# fwd+bwd incl. build, second step only; cold-cache serialised per-launch times. {note}\n")
    f.write(f"# launches {sum(a[1] for a in agg.values())}; total {tot:.0f} us\n")
    f.write("# total_us share launches avg_us grid kernel\n")
    for (name, grid), (us, n, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
        f.write(f"{us:10.1f} {100 * us / tot:5.1f}% {n:6d} {us / n:8.2f} {grid:>14s}  {name}\n")
print(open(dst).read()[:3000])
