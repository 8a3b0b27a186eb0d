import json, os, sys
sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import fp64_dense_time as T
print(os.environ.get("ST_DENSE_GLOBAL_SMALL"), json.dumps({k: round(v["ms"] * 1e3, 1) for k, v in {
    "c1": T.run((100, 100, 100), 1000, 1), "c5_operand": T.run((512, 512), 2048, 8, seed=5),
    "c1_D4": T.run((100, 100, 100), 1000, 4)}.items()}))
