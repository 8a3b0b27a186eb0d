"""Top SASS instructions by warp-stall samples from an ncu report's source page:
python tools/ncu_hot.py report.ncu-rep [top] [kernel-regex]."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 3:
    cmd += ["-k", "regex:" + sys.argv[3]]
raw = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(raw))]
hdr = None
data = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print(f"instructions {len(data)}, samples {tot}")
data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
for d in data[:top]:
    smp = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{smp:7d} {100.0 * smp / max(tot, 1):5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:80]}")
