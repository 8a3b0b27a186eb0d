"""bench.secondary() standalone (no CPU legs): ms of each config."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
r = bench.secondary(None, cpu=False)
print(os.environ.get("ST_IUV_CLUSTER_OFF"), json.dumps({"c1": r["c1_dense_fcs"]["ms"], "c2": r["c2_cp_fcs"]["ms"],
      "c3_step": r["c3_rtpm"]["iuv_step_ms"], "c3_pipe": r["c3_rtpm"]["pipelined_ms"]["iuv_step"],
      "c3_b1_pipe": r["c3_rtpm"]["pipelined_ms"]["iuv_batch1"], "rtpm": r["c3_rtpm"]["rtpm_total_s"],
      "c5": r["c5_kron"]["ms"]}))
