# ncu of the K1 loads-only probe (ST_FX_PROBE=1) and of scatter_bench's loads-only kernel
ST_FX_PROBE=1 K1_TAG=p1 K1_LIB=paper_2106_13062_b200/_lib/libfcs_probe.so python tools/experiments/k1_ab.py 10 4
ST_FX_PROBE=1 K1_LIB=paper_2106_13062_b200/_lib/libfcs_probe.so ncu --set full --clock-control none -k regex:fcs_dense_fx_kernel -c 1 -o gpurun_out/k1_p1 python tools/experiments/k1_ab.py 2 4 > gpurun_out/k1_p1.log 2>&1
./tools/microbench/scatter_bench | head -3
ncu --set full --clock-control none -k regex:scatter -c 1 -o gpurun_out/sb_m3 ./tools/microbench/scatter_bench > gpurun_out/sb_m3.log 2>&1
echo done
