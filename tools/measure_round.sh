# One measurement pass for profiles/ (run on the GPU box, then
# `python tools/update_profiles.py TAG` here): the bench line first (no
# profiler), then the ncu launch list of a short bench, a full capture of K1
# (second launch of tools/prof_c4.py) and the DRAM traffic of 6 launches.
set -e
python bench.py > gpurun_out/bench_r01_final.json 2> gpurun_out/bench_r01_final.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 > gpurun_out/launches_final.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fcs_dense_fx_kernel -s 1 -c 1 \
  -o gpurun_out/fx_final -f python tools/prof_c4.py --reps 2 > gpurun_out/fx_final.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fcs_dense_fx_kernel \
  python tools/prof_c4.py --reps 6 > gpurun_out/ncu_traffic.log 2>&1
echo measured
