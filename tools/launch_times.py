"""Print (kernel, duration) rows of an ncu --csv launch list: python tools/launch_times.py file.csv [n_last]."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
out = [(r[ki], r[vi]) for r in rows[1:] if r[ki] != "Kernel Name"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(out)
for k, v in out[-n:]:
    print(f"{v:>12} ns  {k[:90]}")
