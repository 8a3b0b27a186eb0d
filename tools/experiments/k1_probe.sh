for v in 0 11 12; do
  ST_FX_PROBE=$v python bench.py --steps 20 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('probe $v', round(d['roofline']['kernel_ms'],4))
"
done
