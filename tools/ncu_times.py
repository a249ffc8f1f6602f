#!/usr/bin/env python
"""Print kernel name + gpu__time_duration (us) from `ncu --csv --metrics gpu__time_duration.sum` logs."""
import csv
import sys

for path in sys.argv[1:]:
    print("==", path)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    start = [i for i, r in enumerate(rows) if "Kernel Name" in r]
    if not start:
        continue
    rows = rows[start[0]:]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            print(f"  {r[ki].split('(')[0][:48]:48s} {float(r[vi].replace(',', '')) / 1e3:9.1f} us")
