#!/usr/bin/env python
"""Per-source-line stall samples and executed instructions of one kernel from an ncu report
(needs -lineinfo and --import-source on):

  python tools/ncu_lines.py rep.ncu-rep 'k_flux1<\\(int\\)3, \\(int\\)0' [top]

Prints the hottest lines (stall samples, instructions) and the totals per file."""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
import re
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, recs = None, None, []
seen = set()
want = False
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        hdr = None
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        want = re.search(pat, r[1]) is not None
        hdr = None
        continue
    if not want:
        continue
    if r and r[0] == "Line No":
        hdr = r
        try:
            i_st = r.index("Warp Stall Sampling (All Samples)")
            i_ie = r.index("Instructions Executed")
        except ValueError:
            hdr = None
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    key = (fname, int(r[0]), r[1][:40])
    if key in seen:  # a kernel listed twice: keep the first
        continue
    seen.add(key)
    st = int(r[i_st] or 0) if r[i_st].isdigit() else 0
    ie = int(r[i_ie] or 0) if r[i_ie].isdigit() else 0
    if st or ie:
        recs.append((fname, int(r[0]), st, ie, r[1].strip()[:90]))
ts = sum(x[2] for x in recs) or 1
ti = sum(x[3] for x in recs) or 1
print(f"total stall samples {ts}, instructions {ti / 1e6:.1f}M")
for f in sorted(set(x[0] for x in recs)):
    s = sum(x[2] for x in recs if x[0] == f)
    i = sum(x[3] for x in recs if x[0] == f)
    print(f"  {f:24s} stall {100 * s / ts:5.1f}%  instr {100 * i / ti:5.1f}%")
print("hottest lines (stall %, instr %):")
for x in sorted(recs, key=lambda x: -x[2])[:top]:
    print(f"  {x[0]}:{x[1]:<5d} {100 * x[2] / ts:5.1f}% {100 * x[3] / ti:5.1f}%  {x[4]}")
