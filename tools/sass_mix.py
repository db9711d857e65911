#!/usr/bin/env python
"""Executed-instruction mix by SASS opcode of one kernel from an ncu source-page export:
  ncu -i rep --page source --csv --print-source sass -k regex:NAME > k.csv; python tools/sass_mix.py k.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cnt, stall, tot = collections.Counter(), collections.Counter(), 0
h = None
for r in rows:
    if "Instructions Executed" in r:
        h = r
        ie, src, st = r.index("Instructions Executed"), r.index("Source"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if h is None or len(r) <= ie or not r[ie].isdigit():
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    n = int(r[ie])
    cnt[o] += n
    tot += n
    stall[o] += int(r[st] or 0)
ts = sum(stall.values())
for o, n in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {n / 1e6:9.2f}M {100 * n / tot:5.1f}%   stall samples {100 * stall[o] / max(ts, 1):5.1f}%")
print(f"total {tot / 1e6:.1f}M warp instructions")
