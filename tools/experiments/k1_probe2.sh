for r in 1 2; do
for v in 0 1 2 3; do
  ST_FX_PROBE=$v K1_TAG=probe$v K1_LIB=paper_2106_13062_b200/_lib/libfcs_probe.so python tools/experiments/k1_ab.py 30 4
done; done
