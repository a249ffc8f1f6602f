#!/usr/bin/env python
"""Summarise an ncu report (`ncu -i REP --page raw --csv`) into a compact markdown table.

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_ncu_<name>.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem %"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    kn = idx.get("Kernel Name")
    cols = [(m, lab) for m, lab in METRICS if m in idx]
    print("| kernel | " + " | ".join(f"{lab} ({units[idx[m]]})" if units[idx[m]] else lab for m, lab in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in rows[2:]:
        name = r[kn]
        if "(" in name:
            name = name[:name.index("(")]
        print(f"| {name} | " + " | ".join(r[idx[m]] for m, _ in cols) + " |")


if __name__ == "__main__":
    main()
