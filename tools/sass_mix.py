"""Executed-instruction mix per SASS opcode of one kernel in an ncu report (dev tool).

usage: python tools/sass_mix.py REPORT.ncu-rep KERNEL_REGEX [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Source" in r and "Instructions Executed" in r)
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
i_st = hdr.index("Warp Stall Sampling (All Samples)")
cnt, st = collections.Counter(), collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= i_ex or not r[i_ex].strip().isdigit():
        continue
    ops = r[i_src].strip().split()
    if not ops:
        continue
    op = (ops[1] if ops[0].startswith("@") and len(ops) > 1 else ops[0]).split(".")[0]
    cnt[op] += int(r[i_ex])
    st[op] += int(r[i_st]) if r[i_st].strip().isdigit() else 0
tot, stt = sum(cnt.values()), max(1, sum(st.values()))
for op, c in cnt.most_common(top):
    print(f"{op:10s} {c / 1e6:9.2f}M {100 * c / tot:5.1f}%  stall samples {100 * st[op] / stt:5.1f}%")
print(f"total {tot / 1e6:.2f}M instructions")
