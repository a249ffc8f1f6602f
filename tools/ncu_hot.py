#!/usr/bin/env python
"""Top stall instructions of one kernel launch in an ncu report (source page, SASS)."""
import csv, io, subprocess, sys
rep, regex, skip = sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{regex}",
                      "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][:2])
h = rows[1]
si, ci = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ci]), r[si]) for r in rows[2:] if len(r) > ci and r[ci].isdigit()]
tot = sum(d[0] for d in data) or 1
for n, s in sorted(data, reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 15]:
    print(f"{100*n/tot:5.1f}%  {s.strip()[:110]}")
