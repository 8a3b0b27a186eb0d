"""bench.secondary(x) with the config-4 tensor resident (as run_gpu passes it)."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2106_13062_b200 import _lib as L
n = 1 << 30
x = torch.empty(n, dtype=torch.float32, device="cuda")
L.check(L.lib().st_device_gaussian(L.ST_F32, 4, n, C.c_void_p(x.data_ptr()), None))
r = bench.secondary(x, cpu=False)
print(json.dumps(r["c3_rtpm"]["pipelined_ms"]), r["c3_rtpm"]["rtpm_total_s"])
