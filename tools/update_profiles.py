"""Copy a measurement pass from gpurun_out/ into profiles/: the bench line, the
ncu launch-list summary, the full-capture summary of K1 and the DRAM traffic
(mean of the launches in ncu_traffic.log) into profiles/ncu_traffic.json.

  python tools/update_profiles.py TAG
"""
import collections
import csv
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    rows = list(csv.reader(open(os.path.join(OUT, "launches_final.csv"))))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for x in data:
        if x["Metric Name"] == "gpu__time_duration.sum":
            v = float(x["Metric Value"].replace(",", ""))
            u = x["Metric Unit"]
            v = v / 1e3 if u in ("usecond", "us") else (v / 1e6 if u in ("nsecond", "ns") else v)
            agg[x["Kernel Name"].split("(")[0]].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none, command:",
             "  python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 1",
             f"(cold-cache, serialised launch times; compare SHARES). {tag}.", "",
             f"{'kernel':64s} {'n':>3s} {'avg ms':>9s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:64]:64s} {len(v):3d} {sum(v) / len(v):9.4f} {100 * sum(v) / tot:6.1f}%")
    open(os.path.join(PROF, "launches_r01_final_summary.txt"), "w").write("\n".join(lines) + "\n")
    shutil.copy(os.path.join(OUT, "launches_final.csv"), os.path.join(PROF, "launches_r01_final.csv"))


def full(tag):
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                          os.path.join(OUT, "fx_final.ncu-rep")], capture_output=True,
                         text=True).stdout
    open(os.path.join(PROF, "ncu_c4_fx_r01_final.txt"), "w").write(
        f"ncu --set full --clock-control none, tools/prof_c4.py --reps 2 (second launch). {tag}.\n"
        + txt)


def traffic(tag):
    log = open(os.path.join(OUT, "ncu_traffic.log")).read()
    rd = [float(x) for x in re.findall(r"dram__bytes_read.sum\s+Gbyte\s+([\d.]+)", log)]
    wr = [float(x) for x in re.findall(r"dram__bytes_write.sum\s+Mbyte\s+([\d.]+)", log)]
    d = {"source": "profiles/ncu_traffic_r01b.log (ncu --metrics dram__bytes_read.sum,"
                   "dram__bytes_write.sum --clock-control none, tools/prof_c4.py --reps 6)",
         "dram_bytes_read": int(sum(rd) / len(rd) * 1e9),
         "dram_bytes_write": int(sum(wr) / len(wr) * 1e6),
         "algorithmic_bytes_per_launch": 4295815136,
         "note": f"mean of {len(rd)} launches of fcs_dense_fx_kernel at config 4, {tag}"}
    d["c4_fcs_dense_fx_kernel_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
    json.dump(d, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
    shutil.copy(os.path.join(OUT, "ncu_traffic.log"), os.path.join(PROF, "ncu_traffic_r01b.log"))


def bench():
    shutil.copy(os.path.join(OUT, "bench_r01_final.json"), os.path.join(PROF, "bench_r01.json"))


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "round 1"
    launches(tag)
    full(tag)
    traffic(tag)
    bench()
    print(open(os.path.join(PROF, "launches_r01_final_summary.txt")).read())
    print(open(os.path.join(PROF, "ncu_c4_fx_r01_final.txt")).read())
    print(json.load(open(os.path.join(PROF, "ncu_traffic.json"))))
