# Kernel-time breakdown of the config-2 CP sketch and one config-3 iuv step (ncu launch list).
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/spec_launches.csv \
  python tools/prof_spectral.py --reps 1 > gpurun_out/ncu_spec.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/spec_launches.csv')) if len(r) > 10]
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split('(')[0][:48]; a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(',', ''))
for k, (n, t) in agg.items(): print(f"{n:5d} {t / n / 1000:9.2f} us  {k}")
PY
