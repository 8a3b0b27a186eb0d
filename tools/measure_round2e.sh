# Round-2 captures of the direct estimator (correlate.cu) at config-3 geometry:
# the DMMA Hankel product (batch 15), the DFMA one (batch 1), the readout with
# its fused median tail; plus the warm launch list of both paths.
set -x
N="ncu --set full --import-source on --clock-control none"
python tools/corr_probe.py > gpurun_out/p.log 2>&1 && \
$N -k regex:corr_q_mma -s 1 -c 1 -o gpurun_out/corr_q_mma_c3 -f python tools/corr_probe.py > gpurun_out/q.log 2>&1
$N -k regex:corr_q_kernel -s 1 -c 1 -o gpurun_out/corr_q_b1_c3 -f python tools/corr_probe.py > gpurun_out/q1.log 2>&1
$N -k regex:corr_z -s 2 -c 1 -o gpurun_out/corr_z_c3 -f python tools/corr_probe.py > gpurun_out/z.log 2>&1
for r in corr_q_mma_c3 corr_q_b1_c3 corr_z_c3; do
  echo "== $r"; python tools/ncu_summary.py gpurun_out/$r.ncu-rep
done > gpurun_out/ncu_r02e.txt 2>&1
for p in direct spectral; do
  echo "== warm launch list ($p path), ns"
  ncu --metrics gpu__time_duration.sum,launch__grid_size --cache-control none --clock-control none --csv \
    python tools/corr_probe.py $p 2>/dev/null | python tools/ncu_parse.py /dev/stdin 8
done > gpurun_out/corr_launches_r02e.txt 2>&1
echo measured
