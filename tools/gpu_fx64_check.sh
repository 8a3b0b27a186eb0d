set -x
timeout 300 python tools/fp64_dense_time.py > gpurun_out/fx64_new.json; cat gpurun_out/fx64_new.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/fp64_dense_one.py 1024 1024 256 8192 1 2>/dev/null | grep -E "fx64|sample|scale|reduce" | awk -F'","' '{print $5, $NF}' | cut -c1-40,200-260 | tail -4
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/fp64_dense_one.py 100 100 100 1000 1 2>/dev/null | grep -E "fx64|sample|scale|reduce" | awk -F'","' '{print $5, $NF}' | cut -c1-40,200-260 | tail -4
