"""A/B of the TMA-staged K1 probe (ST_FXT / ST_FXT_QUADS) at config-4
geometry: ms per call and a digest of the D x J~ output (the fixed point is
exact, so every variant must give the same bits)."""
import hashlib
import os
import sys

sys.argv = [sys.argv[0], "paper_2106_13062_b200/_lib/libfcs_b200.so"] + sys.argv[1:]
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "k1_ab_raw.py")).read()
exec(compile(src, "k1_ab_raw.py", "exec"))
torch.cuda.synchronize()
print("env", os.environ.get("ST_FXT"), os.environ.get("ST_FXT_QUADS"),
      "digest", hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:16])
