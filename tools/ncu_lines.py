"""Map ncu per-instruction warp-stall samples to CUDA source lines.

  python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [TOP] [COLUMN]

COLUMN defaults to "Warp Stall Sampling (All Samples)"; any numeric column of
ncu's source page works, e.g. "L1 Wavefronts Shared Excessive".

Extracts the cubins from the library, disassembles the kernel with line info
(nvdisasm -g), aligns it with ncu's SASS page by instruction order, and prints
the source lines holding the most stall samples.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2106_13062_b200", "_lib", "libfcs_b200.so")


def main(rep, kname, top=30, column="Warp Stall Sampling (All Samples)"):
    raw = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kname, "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    iw = hdr.index(column)
    samples = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        try:
            samples.append(float(r[iw].replace(",", "") or 0))
        except ValueError:  # a repeated header (several kernels in the report)
            break
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=tmp, capture_output=True)
    lines = None
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        # split per function
        for m in re.finditer(r"\.text\.(\S+):\n(.*?)(?=\n\s*\.section|\Z)", out, re.S):
            if kname in m.group(1):
                cur = None
                lines = []
                for ln in m.group(2).splitlines():
                    mm = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                    if mm:
                        cur = f"{os.path.basename(mm.group(1))}:{mm.group(2)}"
                    if re.search(r"/\*[0-9a-f]{4,}\*/", ln):
                        lines.append(cur)
                break
        if lines:
            break
    if not lines:
        print("kernel not found in cubins")
        return
    n = min(len(lines), len(samples))
    agg = collections.Counter()
    for i in range(n):
        agg[lines[i]] += samples[i]
    tot = sum(agg.values()) or 1
    src_cache = {}
    for loc, s in agg.most_common(top):
        text = ""
        if loc:
            f, l = loc.split(":")
            path = next(iter(glob.glob(os.path.join(ROOT, "**", f), recursive=True)), None)
            if path:
                src_cache.setdefault(path, open(path).read().splitlines())
                text = src_cache[path][int(l) - 1].strip()[:80]
        print(f"{100 * s / tot:5.1f}%  {loc}  {text}")
    print(f"(aligned {n} of {len(samples)} sampled instructions with {len(lines)} disassembled)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30,
         *(sys.argv[4:5]))
