for v in 1 4; do
ST_IUV_VARIANT=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/iuv_v$v.csv python tools/prof_spectral.py --reps 1 --which c3 > /dev/null 2>&1
python - <<PY
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/iuv_v$v.csv')) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split('(')[0][:40]; a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(',', ''))
print("v$v", {k: round(t / n / 1000, 2) for k, (n, t) in agg.items() if 'iuv' in k or 'median' in k or 'memset' in k.lower()})
PY
done
