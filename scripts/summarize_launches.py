"""Development aid: filter an ncu launch list (--metrics gpu__time_duration.sum --csv) to this
library's kernels and print the per-kernel table used in profiles/*.md.
    python scripts/summarize_launches.py gpurun_out/launches.csv profiles/r01_launches_vN.csv"""
import collections
import re
import csv
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = []
with open(src) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum" or "sv::" not in r["Kernel Name"]:
        continue
    ns = float(r["Metric Value"]) * (1000.0 if r["Metric Unit"] == "us" else 1.0)
    rows.append((r["Kernel Name"], ns))
with open(dst, "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "duration_ns"])
    w.writerows(rows)
agg = collections.OrderedDict()
for k, ns in rows:
    agg.setdefault(k, []).append(ns)
total = sum(ns for _, ns in rows)
print("| kernel | launches | avg us | min us | max us | share of listed time |")
print("|---|---|---|---|---|---|")
for k, v in agg.items():
    short = re.sub(r"^void ", "", k.split("(")[0]).split("::")[-1]
    print(f"| {short} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {min(v) / 1e3:.1f} | {max(v) / 1e3:.1f} | "
          f"{100 * sum(v) / total:.1f}% |")
