# K1 with greedy (fx_group_kernel) vs offline-annealed line groups (config 4)
P=paper_2106_13062_b200/_lib/libfcs_probe.so
for r in 1 2; do
K1_TAG=greedy K1_LIB=$P python tools/experiments/k1_ab.py 30 4
ST_FX_GROUPS_FILE=tools/experiments/groups_c4_annealed.bin K1_TAG=annealed K1_LIB=$P python tools/experiments/k1_ab.py 30 4
done
for v in greedy annealed; do
  if [ $v = annealed ]; then export ST_FX_GROUPS_FILE=tools/experiments/groups_c4_annealed.bin; fi
  K1_LIB=$P ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:fcs_dense_fx_kernel -c 3 python tools/experiments/k1_ab.py 2 4 2>&1 | grep -E "duration|wavefronts" | head -6 | sed "s/^/$v /"
done
