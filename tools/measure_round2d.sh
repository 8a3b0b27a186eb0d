# Round-2 captures of the last cluster-transform users: deflation (config 3),
# T(u,u,u) at batch 1 (cluster, mode 4), the CP sketch's per-family inverse (config 2).
set -x
N="ncu --set full --import-source on --clock-control none"
python tools/experiments/prof_defl.py > gpurun_out/p.log 2>&1 && \
$N -k regex:deflate_cluster -s 1 -c 1 -o gpurun_out/deflate_cluster_c3 -f python tools/experiments/prof_defl.py > gpurun_out/d.log 2>&1
$N -k regex:iuv_cluster -s 1 -c 1 -o gpurun_out/uvw_cluster_b1 -f python tools/experiments/prof_defl.py > gpurun_out/u.log 2>&1
python tools/prof_spectral.py --reps 2 --which c2 > gpurun_out/p.log 2>&1 && \
$N -k regex:spec_inverse_cluster -s 1 -c 1 -o gpurun_out/inv_cluster_c2 -f python tools/prof_spectral.py --reps 2 --which c2 > gpurun_out/i.log 2>&1
for r in deflate_cluster_c3 uvw_cluster_b1 inv_cluster_c2; do
  echo "== $r"; python tools/ncu_summary.py gpurun_out/$r.ncu-rep
done > gpurun_out/ncu_r02d.txt 2>&1
echo measured
