"""Config-3 rtpm wall time with and without the CUDA-graph inner loops
(ST_RTPM_GRAPH), each warm, median of 5; prints JSON."""
import json, os, statistics, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_13062_b200 as st  # noqa: E402
from paper_2106_13062_b200 import configs  # noqa: E402
c = configs.C3
t, lam, V = configs.c3_tensor(c)
dt = st.DenseTensor.from_array(t)
est = st.EstimatorConfig(c.hash_len, c.sketch_count, c.seed)
cfg = st.RtpmConfig(c.rank, configs.C3_INITS, configs.C3_ITERS, st.SketchBackend.FCS, est)
res = {}
for mode in ("0", "1", "0", "1"):
    os.environ["ST_RTPM_GRAPH"] = mode
    st.rtpm(dt, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        cp = st.rtpm(dt, cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    res.setdefault("graphs" if mode == "1" else "plain", []).append(round(statistics.median(ts) * 1e3, 3))
    res["weights_" + mode] = [round(float(x), 9) for x in cp.weights.cpu().numpy()[:3]]
print(json.dumps(res))
