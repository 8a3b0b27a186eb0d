import sys, os, runpy, torch
sys.argv = [sys.argv[0], "paper_2106_13062_b200/_lib/libfcs_b200.so", "4", "10"]
runpy.run_path("tools/k1_ab_raw.py", run_name="__main__")
sys.argv = ["c3"]
runpy.run_path("tools/c3_step_time.py", run_name="__main__")
