# Round-2 captures of the kernels added late in the round, one launch each:
# the cluster estimator (batch 1 with the fused median tail), the cluster
# convolution (config 5), the split batch-15 step's one-CTA part, the fp64
# fixed point over bucket ranges and over fiber segments.
set -x
N="ncu --set full --import-source on --clock-control none"
python tools/prof_iuv.py 1 3 > gpurun_out/p.log 2>&1 && \
$N -k regex:iuv_cluster -s 1 -c 1 -o gpurun_out/iuv_cluster_b1 -f python tools/prof_iuv.py 1 3 > gpurun_out/ic.log 2>&1
$N -k regex:iuv1_kernel -s 1 -c 1 -o gpurun_out/iuv1_split15 -f python tools/prof_iuv.py 15 3 > gpurun_out/i1.log 2>&1
python tools/prof_spectral.py --reps 2 --which c5 > gpurun_out/p.log 2>&1 && \
$N -k regex:conv_cluster -s 1 -c 1 -o gpurun_out/conv_cluster_c5 -f python tools/prof_spectral.py --reps 2 --which c5 > gpurun_out/cc.log 2>&1
python tools/fp64_dense_one.py 1024 1024 512 16384 1 > gpurun_out/p.log 2>&1 && \
$N -k regex:fcs_dense_fx64 -s 1 -c 1 -o gpurun_out/fx64_ranges -f python tools/fp64_dense_one.py 1024 1024 512 16384 1 > gpurun_out/fr.log 2>&1
python tools/fp64_dense_one.py 2048 1024 256 8192 1 > gpurun_out/p.log 2>&1 && \
$N -k regex:fcs_dense_fx64 -s 1 -c 1 -o gpurun_out/fx64_segments -f python tools/fp64_dense_one.py 2048 1024 256 8192 1 > gpurun_out/fs.log 2>&1
for r in iuv_cluster_b1 iuv1_split15 conv_cluster_c5 fx64_ranges fx64_segments; do
  echo "== $r"; python tools/ncu_summary.py gpurun_out/$r.ncu-rep
done > gpurun_out/ncu_r02c.txt 2>&1
echo measured
