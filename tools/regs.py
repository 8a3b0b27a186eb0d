"""Per-kernel registers / stack / spills from `nvcc -Xptxas -v` for one source file.

    python tools/regs.py paper_2106_13062_b200/csrc/spectral.cu [filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++20",
       "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Iinclude", "-Ipaper_2106_13062_b200/csrc",
       "-c", src, "-o", "/dev/null", "-Xptxas", "-v"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
name = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        d = re.search(r"_ZN3fcs\d+(\w+?)E|_ZN3fcs\d+(\w+)", name)
        short = re.sub(r"^_ZN3fcs\d+", "", name)[:40]
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and name:
        stack, spill = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if flt in name:
            print(f"{short:42s} regs {m.group(1):>4s} stack {stack:>4s} spill {spill:>4s}")
        name = None
