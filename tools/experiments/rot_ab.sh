# K1: searched groups (default) vs offline-annealed groups + rotations (rot2: {0,2}, rot4: {0..3})
P=paper_2106_13062_b200/_lib/libfcs_probe.so
for r in 1 2; do
K1_TAG=searched K1_LIB=$P python tools/experiments/k1_ab.py 30 4
ST_FX_ROT=1 ST_FX_GROUPS_FILE=tools/experiments/groups_c4_rot2.bin K1_TAG=rot2 K1_LIB=$P python tools/experiments/k1_ab.py 30 4
ST_FX_ROT=1 ST_FX_GROUPS_FILE=tools/experiments/groups_c4_rot4.bin K1_TAG=rot4 K1_LIB=$P python tools/experiments/k1_ab.py 30 4
done
for v in rot2 rot4; do
  ST_FX_ROT=1 ST_FX_GROUPS_FILE=tools/experiments/groups_c4_$v.bin K1_LIB=$P ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:fcs_dense_fx_kernel -c 2 python tools/experiments/k1_ab.py 2 4 2>&1 | grep -E "duration|wavefronts|issue|inst_exec" | head -5 | sed "s/^/$v /"
done
