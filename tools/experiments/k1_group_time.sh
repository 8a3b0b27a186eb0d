for r in 1 2; do K1_TAG=searched python tools/experiments/k1_ab.py 30 4; done
ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:"fcs_dense_fx_kernel|fx_group" -c 6 python tools/experiments/k1_ab.py 2 4 2>&1 | grep -E "fx_group|fcs_dense_fx|duration|wavefronts" | head -24
