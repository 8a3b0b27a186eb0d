"""bench.secondary() standalone (no CPU legs): does the c3 pipelined step
match tools/c3_step_time.py?"""
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
r = bench.secondary(None, cpu=len(sys.argv) > 1)
print(json.dumps(r["c3_rtpm"]["pipelined_ms"]), r["c3_rtpm"]["rtpm_total_s"])
