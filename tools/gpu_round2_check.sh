set -x
nproc; free -g | head -2
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_a.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_a.json 2> gpurun_out/ref_a.err; echo ref rc=$?
cat gpurun_out/ref_a.json; tail -5 gpurun_out/ref_a.err
