"""Per-kernel-class table of an ncu capture with --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum (tools/prof_step.py, C4 fwd+bwd, batch 32):
launches, total/avg duration, DRAM bytes per launch and DRAM GB/s per class (cold-cache,
serialised per-launch replay numbers; shares, not the bench's absolute times).
  python tools/kernel_table.py in.csv out.txt"""
import collections
import csv
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
per = collections.defaultdict(dict)  # launch id -> metrics
names = {}
for r in rows[1:]:
    lid = r[ix["ID"]]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    m = r[ix["Metric Name"]]
    if m == "gpu__time_duration.sum":
        v = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    elif m.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(unit, 1)
        v = v * scale
    per[lid][m] = v
    names[lid] = (r[ix["Kernel Name"]].split("(")[0].replace("void ", ""), r[ix["Grid Size"]])
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for lid, mm in per.items():
    key = names[lid]
    a = agg[key]
    a[0] += 1
    a[1] += mm.get("gpu__time_duration.sum", 0.0)
    a[2] += mm.get("dram__bytes_read.sum", 0.0) + mm.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
with open(dst, "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
            "--clock-control none, tools/prof_step.py 1 (C4 (32,64,64), batch 32, build+fwd+bwd)\n")
    f.write(f"# {sum(a[0] for a in agg.values())} launches, {tot / 1e3:.1f} ms summed (cold, serialised)\n")
    f.write("# launches  total_ms  share  avg_us  MB/launch  DRAM_GB/s  frac_of_6551  grid  kernel\n")
    for (name, grid), (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = by / (us * 1e-6) / 1e9 if us else 0.0
        f.write(f"{n:8d} {us / 1e3:9.2f} {100 * us / tot:5.1f}% {us / n:8.2f} {by / n / 1e6:9.2f} "
                f"{gbs:9.0f} {gbs / 6551.4:6.2f}  {grid:>14s}  {name}\n")
print(open(dst).read()[:6000])
