"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    try:
        d[r[ki].split("(")[0][-48:]].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:50s} n={len(v):5d} mean={sum(v)/len(v)/1e3:9.1f}us max={max(v)/1e3:9.1f}us "
          f"tot={sum(v)/1e6:8.3f}ms {100*sum(v)/tot:5.1f}%")
