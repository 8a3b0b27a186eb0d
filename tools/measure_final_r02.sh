# Final round-2 pass: bench line + reference arm (no profiler), then the ncu
# launch list of a short bench (its command run plainly first).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_final.json 2>&1
python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 > gpurun_out/launches_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 > gpurun_out/launches_final.log 2>&1
echo measured
