"""fp32 dense FCS with J~ beyond shared memory (int32 buckets: J~ > ~57k):
1024^3, J = 32768 (J~ = 98,302), D = 1 and 4: ms per call."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import json
import f32_cliff_time as T
print(json.dumps({f"J32768_D{D}": T.run((1024, 1024, 1024), 32768, D) for D in (1, 4)}))
