# Round-2 full captures, one kernel each (the regex of measure_round2.sh
# matched the scatter's redo launch and repeated cp_rank1).
set -x
python tools/prof_c4.py --reps 3 > gpurun_out/p.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fcs_dense_fx_kernel -s 2 -c 1 \
  -o gpurun_out/c4_fx_r02 -f python tools/prof_c4.py --reps 3 > gpurun_out/c4_fx.log 2>&1
python tools/prof_spectral.py --reps 2 --which c2,c3,c5,coo > gpurun_out/p.log 2>&1
for k in cp_rank1_kernel iuv1_kernel conv_kernel fcs_coo_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 \
    -o gpurun_out/${k}_r02 -f python tools/prof_spectral.py --reps 2 --which c2,c3,c5,coo > gpurun_out/$k.log 2>&1
done
echo measured
