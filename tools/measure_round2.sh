# Round-2 measurement pass for profiles/ (on the GPU box; summaries are made
# here afterwards): the bench line and the reference arm (no profiler), the
# ncu launch list of a short bench, and one full capture per key kernel, each
# command run plainly first (exit 0) and then under ncu.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_r02.json 2>&1
python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 > gpurun_out/launches_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 3 --warmup 3 --no-secondary --no-cpu --e2e-steps 1 > gpurun_out/launches_r02.log 2>&1
python tools/prof_c4.py --reps 2 > gpurun_out/p.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fcs_dense_fx_kernel -s 1 -c 1 \
  -o gpurun_out/c4_fx_r02 -f python tools/prof_c4.py --reps 2 > gpurun_out/c4_fx.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fcs_dense_fx_kernel \
  python tools/prof_c4.py --reps 6 > gpurun_out/ncu_traffic_r02.log 2>&1
python tools/fp64_dense_one.py 1024 1024 512 8192 1 > gpurun_out/p.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fcs_dense_fx64 -s 1 -c 1 \
  -o gpurun_out/fx64_r02 -f python tools/fp64_dense_one.py 1024 1024 512 8192 1 > gpurun_out/fx64.log 2>&1
python tools/fp64_dense_one.py 100 100 100 1000 1 > gpurun_out/p.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fcs_dense_smem -s 1 -c 1 \
  -o gpurun_out/c1_smem_r02 -f python tools/fp64_dense_one.py 100 100 100 1000 1 > gpurun_out/c1.log 2>&1
python tools/prof_spectral.py --reps 2 --which c2,c3,c5,coo > gpurun_out/p.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"cp_rank1_kernel|iuv1_kernel|conv_kernel|fcs_coo_kernel" -c 4 \
  -o gpurun_out/spectral_r02 -f python tools/prof_spectral.py --reps 1 --which c2,c3,c5,coo > gpurun_out/spec.log 2>&1
echo measured
