"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch):
per-kernel launch count and share of the total device time."""
import csv, io, sys
from collections import defaultdict

path = sys.argv[1]
text = open(path).read()
start = text.find('"ID"')
rows = list(csv.reader(io.StringIO(text[start:])))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:60]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:<60} launches={cnt[k]:>5} share={100 * v / s:5.1f}% total_ms={v * 1e-6:8.3f}")
