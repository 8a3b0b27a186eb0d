# K1 time at config 4 (bench kernel_ms) and the dense parity tests.
python bench.py --steps 30 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4))
"
python -m pytest tests/test_gpu_parity.py -q -k "dense or f32 or host" 2>&1 | tail -2
