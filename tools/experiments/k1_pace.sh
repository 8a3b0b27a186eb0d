# K1 with and without sibling pacing: bench kernel time and ncu DRAM bytes.
for e in "X=1" "ST_FX_NOPACE=1"; do
  env $e python bench.py --steps 30 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 2>&1 | grep -o '"kernel_ms": [0-9.]*' | sed "s/^/$e /"
  env $e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:fcs_dense_fx -s 1 -c 1 python tools/prof_c4.py --reps 2 2>&1 | grep -E "duration|dram__bytes" | sed "s/^/$e /"
done
python -m pytest tests/test_gpu_parity.py -q -k "dense or f32 or host" 2>&1 | tail -1
